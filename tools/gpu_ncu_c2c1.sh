python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"conv_walk_kernel" -s 2 -c 1 \
    -o gpurun_out/c2conv1 python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/ncu_c2conv1.log 2>&1; echo ncu=$?
ncu -i gpurun_out/c2conv1.ncu-rep --page source --csv --print-source sass > gpurun_out/c2conv1_sass.csv 2>&1; echo src=$?
