python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_nhwc.py tests/test_gpu_kernels.py -q -m gpu -x -k "pool" > gpurun_out/pytest_i11.log 2>&1; echo t=$?
tail -1 gpurun_out/pytest_i11.log
timeout 600 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print(d['value'], d['stages_ms'])"
