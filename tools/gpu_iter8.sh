python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_f1.py tests/test_gpu_encode_large.py tests/test_gpu_nhwc.py -q -m gpu -x > gpurun_out/pytest_f1.log 2>&1; echo f1=$?
tail -2 gpurun_out/pytest_f1.log
for w in c4 c5; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$?;
python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print(d['value'], d['stages_ms'], d['gpu_launches'])"; done
bash tools/gpu_checked.sh
