python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv \
      python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/ncu_c2.log 2>&1; echo launches_c2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_walk" -s 2 -c 1 -o gpurun_out/walk_c2conv1 \
      python bench.py --workload c2 --steps 1 --warmup 1 --profile > gpurun_out/ncu_w.log 2>&1; echo walk=$?
