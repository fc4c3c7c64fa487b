# ncu --set full capture (with source) of kernel regex $1 (skip $3 launches, capture $4) in bench workload $2
set -x
k=${1:-conv_walk}; w=${2:-c2}; skip=${3:-0}; cnt=${4:-1}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --workload $w --steps 1 --warmup 1 --profile --no-cpu-baseline > gpurun_out/plain_$w.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$k" -s $skip -c $cnt \
    -o gpurun_out/k_$w python bench.py --workload $w --steps 1 --warmup 1 --profile --no-cpu-baseline > gpurun_out/ncuk_$w.log 2>&1; echo ncu=$?
