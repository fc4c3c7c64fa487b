# compute-sanitizer memcheck / racecheck / synccheck / initcheck over one shrunken step of every workload
# (tools/sanitize_run.py); logs under gpurun_out/sanitize/, summary in gpurun_out/sanitize/summary.txt
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for w in ${WL:-c1 c2 c3 c4 c5}; do
  for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
    timeout ${SAN_TIMEOUT:-900} $CS --tool $tool $extra --print-limit 50 \
        python tools/sanitize_run.py $w > gpurun_out/sanitize/${w}_${tool}.log 2>&1
    rc=$?
    echo "$w $tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize/${w}_${tool}.log | tail -1)" \
        | tee -a gpurun_out/sanitize/summary.txt
  done
done
