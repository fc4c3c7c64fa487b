python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
ncu --set full --clock-control none --import-source on -k regex:"enc_small|pool_nhwc" -s 3 -c 3 \
    -o gpurun_out/c2enc python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/ncu_c2enc.log 2>&1; echo ncu=$?
