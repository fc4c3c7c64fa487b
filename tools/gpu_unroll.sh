# sort-pass unroll experiment (SNN_SORT_UNROLL via SNN_NVCC_EXTRA): C2 and C5 conv stages
for u in 4 8 16; do
  SNN_NVCC_EXTRA="-DSNN_SORT_UNROLL=$u" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$u.log 2>&1 || { echo build$u failed; continue; }
  for w in c2 c5; do
    timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench_${w}_u$u.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/bench_${w}_u$u.json'));print('u$u $w', d['value'], {k: d['stages_ms'][k] for k in d['stages_ms'] if k.startswith('conv')})"
  done
done
