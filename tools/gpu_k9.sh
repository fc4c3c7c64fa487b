# K9 (fully connected rewrite of theta = inf layers with H W < KH KW): parity + same-box A/B by env
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_nhwc.py tests/test_gpu_configs.py -q -m gpu -x -k "fc or inf or conv_fire or c2 or C2" > gpurun_out/pytest_k9.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_k9.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
for w in ${WL:-c2}; do for v in 1 0 1 0; do
  SNN_TC_FC=$v timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps ${STEPS:-10} > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "$w [fc $v] $(python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['value'], d['stages_ms'], d['clocks'] and d['clocks']['sm_mhz'])")"
done; done
