set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"conv_tct" -s 2 -c 2 \
    -o gpurun_out/prof_tct python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/ncu_tct.log 2>&1; echo ncu=$?
