# launch lists for c2 and c5 + full ncu capture of the walk/sort kernels
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for w in c2 c5; do
python bench.py --workload $w --steps 1 --warmup 1 --profile > gpurun_out/plain_$w.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 1 --profile > gpurun_out/ncu_$w.log 2>&1; echo ncu_$w=$?
done
ncu --set full --clock-control none --import-source on -k regex:"conv_walk|rf_sort" -s 8 -c 8 \
    -o gpurun_out/prof_c2 python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/ncu_full_c2.log 2>&1; echo full_c2=$?
ncu --set full --clock-control none --import-source on -k regex:"conv_walk|rf_sort" -s 20 -c 2 \
    -o gpurun_out/prof_c5 python bench.py --workload c5 --steps 1 --warmup 1 --profile > gpurun_out/ncu_full_c5.log 2>&1; echo full_c5=$?
