# full measurement pass: GPU tests, smoke, every bench line (with cpu_baseline + e2e), launch lists of
# every workload, ncu --set full traffic captures of the conv kernels (C2, C5)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
for w in c2 c5 c3 c4 c1; do timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$?; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
for w in c2 c5 c3 c4 c1; do
  python bench.py --workload $w --steps 2 --warmup 1 --profile > gpurun_out/plain_$w.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$w.csv \
      python bench.py --workload $w --steps 2 --warmup 1 --profile > gpurun_out/ncu_$w.log 2>&1; echo launches_$w=$?
done
timeout 1200 bash tools/gpu_traffic.sh
