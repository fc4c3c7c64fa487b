# theta=inf GEMM knobs on C2 conv3: pipeline stages (build-time) x feature chunks (SNN_TC_NCH)
for st in 4 6; do
  SNN_NVCC_EXTRA="-DSNN_TC_STAGES=$st" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$st.log 2>&1 || { echo build$st failed; continue; }
  for nch in 4 5 8; do
    SNN_TC_NCH=$nch timeout 300 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_tc.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/bench_tc.json'));print('st$st nch$nch', d['value'], d['stages_ms']['conv3'])"
  done
done
