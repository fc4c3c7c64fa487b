# per-launch device times (ncu, cold-cache/serialised: compare shares) for one bench workload
# usage: bash tools/gpu_launches.sh <workload> [steps]
set -x
w=${1:-c2}; k=${2:-2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --workload $w --steps $k --warmup 1 --profile > gpurun_out/plain_$w.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$w.csv \
    python bench.py --workload $w --steps $k --warmup 1 --profile > gpurun_out/ncu_$w.log 2>&1; echo ncu=$?
