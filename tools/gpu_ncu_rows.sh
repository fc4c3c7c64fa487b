python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"conv_walk_kernel" -s 2 -c 1 \
    -o gpurun_out/rows_c2 python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/ncu_rows_c2.log 2>&1; echo ncu=$?
ncu --set full --clock-control none --import-source on -k regex:"conv_walk_kernel" -s 1 -c 1 \
    -o gpurun_out/rows_c4 python bench.py --workload c4 --steps 1 --warmup 1 --profile > gpurun_out/ncu_rows_c4.log 2>&1; echo ncu=$?
