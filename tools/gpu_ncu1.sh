# one ncu --set full capture (with source) of the first launch of kernel regex $1 in bench workload $2
set -x
k=${1:-conv_walk}; w=${2:-c2}; skip=${3:-0}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --workload $w --steps 1 --warmup 1 --profile --no-cpu-baseline > gpurun_out/plain_$w.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$k" -s $skip -c 1 \
    -o gpurun_out/one_$w python bench.py --workload $w --steps 1 --warmup 1 --profile --no-cpu-baseline > gpurun_out/ncu1_$w.log 2>&1; echo ncu=$?
