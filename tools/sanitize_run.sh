for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_step.py all > gpurun_out/san_$t.log 2>&1
  echo "$t: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$t.log | tail -1)"
done
