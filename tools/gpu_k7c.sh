python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_nhwc.py -x -q -k "rows or in_nhwc" > gpurun_out/k7c_pytest.log 2>&1; echo pytest=$?
for g in 1 2 4; do SNN_SORT_ROWS=0 SNN_WALK_ROWS_G=$g python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/k7c_c2_g$g.json 2>/dev/null; done
for g in 1 2 4; do SNN_WALK_ROWS_G=$g python bench.py --workload c4 --no-cpu-baseline --no-e2e > gpurun_out/k7c_c4_g$g.json 2>/dev/null; done
for nx in 8 12; do SNN_SORT_ROWS_NX=$nx python bench.py --workload c5 --no-cpu-baseline --no-e2e > gpurun_out/srows${nx}_c5.json 2>/dev/null; done
