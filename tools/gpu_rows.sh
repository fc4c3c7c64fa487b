# K7 row tiles: parity + C2/C4 bench (rows on) vs SNN_WALK_ROWS=0 on the same box
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_nhwc.py -x -q -k "rows or in_nhwc" > gpurun_out/rows_pytest.log 2>&1; echo pytest=$?
python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/rows_c2.json 2> gpurun_out/rows_c2.err
SNN_WALK_ROWS=0 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/norows_c2.json 2>/dev/null
python bench.py --workload c4 --no-cpu-baseline --no-e2e > gpurun_out/rows_c4.json 2> gpurun_out/rows_c4.err
