python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_f1.py -q -m gpu -x > gpurun_out/pytest_f1.log 2>&1; echo f1=$?
tail -2 gpurun_out/pytest_f1.log
for i in 1 2; do timeout 600 python bench.py --workload c4 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?;
python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print(d['value'], d['stages_ms'], d['gpu_launches'])"; done
timeout 300 python tools/rstdp_stamps.py > gpurun_out/stamps.txt 2>&1; cat gpurun_out/stamps.txt | tail -4
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_bench_steps.py -q -m gpu -x -k c4 > gpurun_out/pytest_full.log 2>&1; echo full=$?
tail -2 gpurun_out/pytest_full.log
