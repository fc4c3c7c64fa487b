# K2e (kmin test-free prefix, unpadded prefix buckets): parity + same-box A/B by env
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_nhwc.py tests/test_gpu_large_rf.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/pytest_k2e.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_k2e.log
for w in ${WL:-c5}; do for v in 1 0 1; do
  SNN_KMIN=$v timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps ${STEPS:-5} > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "$w [kmin $v] $(python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['value'], d['stages_ms'], d['clocks'] and d['clocks']['sm_mhz'])")"
done; done
