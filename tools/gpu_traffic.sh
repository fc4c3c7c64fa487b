# ncu --set full captures of exactly one step's conv kernels (C2: conv1 fused walk + conv2 sort/walk
# chunks; C5: two of the 285 sort/walk chunk pairs), for bench.py's roofline "traffic"
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"conv_walk|rf_sort|conv_tc_kernel|tc_prep" -s 14 -c 14 \
    -o gpurun_out/traffic_c2 python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/ncu_t_c2.log 2>&1; echo c2=$?
python bench.py --workload c5 --steps 1 --warmup 1 --profile > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"conv_walk|rf_sort" -s 570 -c 4 \
    -o gpurun_out/traffic_c5 python bench.py --workload c5 --steps 1 --warmup 1 --profile > gpurun_out/ncu_t_c5.log 2>&1; echo c5=$?
