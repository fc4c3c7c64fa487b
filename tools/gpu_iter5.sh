python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
LIBS="ab/libO.so ab/libA.so ab/libB.so" WL="c3 c5" bash tools/gpu_ab_lib.sh > gpurun_out/ab7.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_nhwc.py tests/test_gpu_large_rf.py tests/test_gpu_configs.py tests/test_gpu_encode_large.py -q -m gpu -x > gpurun_out/pytest_iter.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_iter.log
