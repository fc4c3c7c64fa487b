set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in 1 4; do
  SNN_SORT_PPW=$v timeout 300 python bench.py --workload c5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_sp$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/bench_c5_sp$v.json'));print('sp$v', d['value'], d['stages_ms'])"
done
for w in c3 c1; do timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench_$w.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print('$w', d['value'], d['stages_ms'])"; done
