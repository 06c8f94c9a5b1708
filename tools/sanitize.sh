#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py -> gpurun_out/r2_sanitize_<tool>.log
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout ${TMO:-900} /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 50 \
    python tools/sanitize_cases.py > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'OK' gpurun_out/r2_sanitize_$tool.log) cases OK; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/r2_sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
