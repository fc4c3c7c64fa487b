set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_f1.py -q -m gpu -x > gpurun_out/pytest_f1.log 2>&1; echo f1=$?
tail -3 gpurun_out/pytest_f1.log
timeout 900 python -m pytest tests/test_gpu_encode_large.py tests/test_gpu_kernels.py tests/test_gpu_variants.py tests/test_gpu_nhwc.py -q -m gpu -x -k "encode" > gpurun_out/pytest_iter.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_iter.log
for w in c4 c5; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c5.csv \
      python bench.py --workload c5 --steps 1 --warmup 1 --profile > gpurun_out/ncu_c5.log 2>&1; echo launches_c5=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c4.csv \
      python bench.py --workload c4 --steps 1 --warmup 1 --profile > gpurun_out/ncu_c4.log 2>&1; echo launches_c4=$?
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k c4 > gpurun_out/pytest_full.log 2>&1; echo full=$?
tail -3 gpurun_out/pytest_full.log
