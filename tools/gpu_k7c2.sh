python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_nhwc.py tests/test_gpu_kernels.py -x -q > gpurun_out/k7c2_pytest.log 2>&1; echo pytest=$?
python bench.py --workload c4 --no-cpu-baseline --no-e2e > gpurun_out/k7c2_c4.json 2>/dev/null
python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/k7c2_c2.json 2>/dev/null
