python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
LIBS="ab/libA.so ab/libC.so" WL="c5" bash tools/gpu_ab_lib.sh > gpurun_out/ab8.txt 2>&1
SNN_SORT_TABLE=1 LIBS="ab/libC.so" WL="c5" bash tools/gpu_ab_lib.sh >> gpurun_out/ab8.txt 2>&1
for L in ab/libA.so ab/libC.so; do
SNN_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rf_sort|conv_walk|enc_" -c 30 --csv \
      --log-file gpurun_out/ab_l.csv python bench.py --workload c5 --steps 1 --warmup 1 --profile > /dev/null 2>&1
echo "== $L" >> gpurun_out/ab8.txt; python tools/launch_summary.py gpurun_out/ab_l.csv >> gpurun_out/ab8.txt
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_nhwc.py tests/test_gpu_configs.py tests/test_gpu_encode_large.py -q -m gpu -x > gpurun_out/pytest_iter.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_iter.log
