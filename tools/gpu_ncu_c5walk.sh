python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"conv_walk_kernel|rf_sort_kernel" -s 60 -c 2 \
    -o gpurun_out/c5walk python bench.py --workload c5 --steps 1 --warmup 1 --profile > gpurun_out/ncu_c5walk.log 2>&1; echo ncu=$?
