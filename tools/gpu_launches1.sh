# launch list (ncu gpu__time_duration) of one workload: WL, extra env passed through
python bench.py --workload ${WL:-c2} --steps 2 --warmup 1 --profile > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_one.csv \
   python bench.py --workload ${WL:-c2} --steps 2 --warmup 1 --profile > gpurun_out/ncu_one.log 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/launches_one.csv 2>/dev/null | head -40
