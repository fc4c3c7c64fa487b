# iteration pass: build, conv parity tests, C5/C2 bench lines, C5 launch list (sort vs walk split)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_nhwc.py tests/test_gpu_large_rf.py ${EXTRA_TESTS} -q -m gpu -x > gpurun_out/pytest_iter.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_iter.log
for w in ${WL:-c5 c2}; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$?; done
for w in ${LWL:-c5}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$w.csv \
      python bench.py --workload $w --steps 1 --warmup 1 --profile > gpurun_out/ncu_$w.log 2>&1; echo launches_$w=$?
done
