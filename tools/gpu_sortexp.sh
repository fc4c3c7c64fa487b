# sort-kernel experiments: C2 with SNN_SORT_PPW = 1 / 2 / 4 (launch lists), plus the default bench lines
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in 1 2 4; do
  SNN_SORT_PPW=$v timeout 300 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_sp$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/bench_c2_sp$v.json'));print('sp$v', d['value'], d['stages_ms'])"
done
timeout 300 python bench.py --workload c4 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_c4.json'));print('c4', d['value'], d['stages_ms'])"
