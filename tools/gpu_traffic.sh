# ncu --set full captures of one bench step's conv kernels, for bench.py's roofline "traffic":
# C2: step 2's conv1 (fused walk), conv2 (sort + walk, 1 list chunk), conv3 (K9: tc prep limbs / b / a + GEMM);
# C5: two of the sort/walk chunk pairs of step 2 (scaled by the chunk count in tools/traffic_json.py)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"conv_walk|rf_sort|conv_tc_kernel|tc_prep" -s 7 -c 7 \
    -o gpurun_out/traffic_c2 python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/ncu_t_c2.log 2>&1; echo c2=$?
python bench.py --workload c5 --steps 1 --warmup 1 --profile > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"conv_walk|rf_sort" -s 56 -c 4 \
    -o gpurun_out/traffic_c5 python bench.py --workload c5 --steps 1 --warmup 1 --profile > gpurun_out/ncu_t_c5.log 2>&1; echo c5=$?
