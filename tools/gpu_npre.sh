# presorted-walk prefetch depth experiment (SNN_WALK_NPRE) on C2 and C5
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in 256 160 128 96 64; do
  for w in c2 c5; do
  SNN_WALK_NPRE=$v timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench_${w}_np$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/bench_${w}_np$v.json'));print('$w np$v', d['value'], d['stages_ms'])"
  done
done
