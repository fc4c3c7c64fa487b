# same-box A/B of one environment switch: VAR=name, VALS="a b", WL workloads
for w in ${WL:-c5}; do for v in ${VALS:-1 0 1 0}; do
  env ${VAR}=$v timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps ${STEPS:-5} > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "$w [${VAR} $v] $(python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['value'], d['stages_ms'], d['clocks'] and d['clocks']['sm_mhz'])")"
done; done
