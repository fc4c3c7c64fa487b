# ncu --set full captures of the conv kernels (C2 all layers of one step, C5 conv walk)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --workload c2 --steps 2 --warmup 1 --profile > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"conv_walk|rf_sort|conv_tc|tc_prep|enc_small|pool" -s 12 -c 12 \
    -o gpurun_out/prof_c2 python bench.py --workload c2 --steps 2 --warmup 1 --profile > gpurun_out/ncu_c2.log 2>&1; echo c2=$?
python bench.py --workload c5 --steps 1 --warmup 1 --profile > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"conv_walk|enc_|kwta|inhibit|pool" -s 0 -c 8 \
    -o gpurun_out/prof_c5 python bench.py --workload c5 --steps 1 --warmup 1 --profile > gpurun_out/ncu_c5.log 2>&1; echo c5=$?
