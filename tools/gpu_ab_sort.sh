# same-box A/B of library builds (ab/lib*.so, built on the CPU side): C5 bench line + sort/walk launch times
for L in ${LIBS:-ab/libA.so ab/libB.so ab/libC.so ab/libD.so}; do
  for V in ${VECS:-0}; do
    if [ "$V" = 1 ]; then export SNN_SORT_VEC=1; else unset SNN_SORT_VEC; fi
    SNN_LIB=$L timeout 600 python bench.py --workload c5 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/ab.json 2>gpurun_out/ab.err
    echo "c5 [$L vec=$V] $(python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['value'], d['stages_ms'])")"
    SNN_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rf_sort|conv_walk" -c 20 --csv \
      --log-file gpurun_out/ab_l.csv python bench.py --workload c5 --steps 1 --warmup 1 --profile > /dev/null 2>&1
    python tools/launch_summary.py gpurun_out/ab_l.csv
  done
done
