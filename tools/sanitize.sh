# compute-sanitizer over tools/sanitize_run.py: memcheck, racecheck, synccheck
# -> gpurun_out/sanitize_<tool>.log (summary lines: "ERROR SUMMARY: N errors")
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py \
    > gpurun_out/sanitize_$t.log 2>&1
  echo "$t exit $?" >> gpurun_out/sanitize_$t.log
done
