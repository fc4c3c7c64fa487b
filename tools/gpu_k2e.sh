# K2e (kmin test-free prefix) / K2f (K* cut with the sort's adaptive count guess): parity + same-box A/B by env
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_nhwc.py -q -m gpu -x -k "kmin or kstar or conv_fire" > gpurun_out/pytest_k2e.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_k2e.log
for w in ${WL:-c5 c2}; do for cfg in "0 0" "1 0" "0 1" "1 1"; do
  set -- $cfg
  SNN_KMIN=$1 SNN_KSTAR=$2 timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps ${STEPS:-5} > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "$w [kmin $1 kstar $2] $(python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['value'], d['stages_ms'], d['clocks'] and d['clocks']['sm_mhz'])")"
done; done
