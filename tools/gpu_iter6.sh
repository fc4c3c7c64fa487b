python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for nw in 32 28 24 20 16; do
  SNN_DEBUG_PLAN=1 SNN_WALK_PRE_WARPS=$nw timeout 600 python bench.py --workload c5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "c5 warps=$nw $(python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['value'], d['stages_ms']['conv1'])") $(grep 'walk plan' gpurun_out/ab.err | tail -1)"
done
