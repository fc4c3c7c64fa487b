# A/B of library builds in one GPU call: LIBS="path1 path2 ..." (built on the CPU side), WL workloads
for w in ${WL:-c2 c5}; do for L in ${LIBS}; do
  SNN_LIB=$L timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps ${STEPS:-10} > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "$w [$L] $(python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['value'], d['stages_ms'], d['clocks'] and d['clocks']['sm_mhz'])")"
done; done
