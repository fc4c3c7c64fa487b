# Baseline of the current HEAD: C2/C4 bench lines and an ncu source capture of C2's fused conv1 walk
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --workload c2 --no-cpu-baseline > gpurun_out/base_c2.json 2> gpurun_out/base_c2.err
python bench.py --workload c4 --no-cpu-baseline > gpurun_out/base_c4.json 2> gpurun_out/base_c4.err
ncu --set full --clock-control none --import-source on -k regex:"conv_walk_kernel<4, 4" -s 2 -c 1 \
    -o gpurun_out/c2conv1 python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/ncu_c2conv1.log 2>&1; echo ncu=$?
