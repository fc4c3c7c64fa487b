# same-box A/B of library builds: WL workloads x LIBS (bench lines); then the parity tests on the current build
for w in ${WL:-c3 c5}; do for L in ${LIBS}; do
  SNN_LIB=$L timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "$w [$L] $(python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['value'], d['stages_ms'])")"
done; done
