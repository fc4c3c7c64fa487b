python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_nhwc.py tests/test_gpu_configs.py -x -q -k "pool2 or rows or c2_parity" > gpurun_out/pool2_pytest.log 2>&1; echo pytest=$?
python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/pool2_c2.json 2>gpurun_out/pool2_c2.err
