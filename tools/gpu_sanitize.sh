#!/bin/bash
# compute-sanitizer over the hot path (tools/sanitize_run.py): one tool after the other,
# each bounded by its own timeout; summaries in gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 3 \
      python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
