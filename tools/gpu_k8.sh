python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_nhwc.py -x -q -k "implicit or in_nhwc" > gpurun_out/k8_pytest.log 2>&1; echo pytest=$?
python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/k8_c2.json 2>/dev/null
SNN_TC_IMPLICIT=0 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/nok8_c2.json 2>/dev/null
