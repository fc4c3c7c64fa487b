# A/B timing of env settings: AB="VAR=val;VAR2=val" (';'-separated configurations, '-' = none), WL
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
IFS=';' read -ra CFGS <<< "${AB:--}"
for w in ${WL:-c2 c5}; do for c in "${CFGS[@]}"; do
  if [ "$c" = "-" ]; then envs=""; else envs="$c"; fi
  env $envs timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps ${STEPS:-10} > gpurun_out/ab.json 2>/dev/null
  echo "$w [$c] $(python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['value'], d['stages_ms'])")"
done; done
