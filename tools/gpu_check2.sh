# GPU check of a change: selected parity tests + bench lines (no cpu baseline), given as env:
#   TESTS="tests/test_gpu_nhwc.py ..."  WL="c2 c5"
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest ${TESTS:-tests} -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
for w in ${WL:-c2 c5}; do timeout 600 python bench.py --workload $w --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$?;
  python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['stages_ms'], d['roofline'] and d['roofline']['frac'], {k: v['frac'] for k, v in d.get('stage_rooflines', {}).items()})"; done
