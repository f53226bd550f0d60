#!/bin/sh
# compute-sanitizer over every kernel of the library (tools/sanitize_driver.py
# on small inputs, results checked against the oracle).  Logs -> $1 (default
# gpurun_out/); the committed summaries live in profiles/.
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report analysis"
  JT_SAN_SMALL=1 timeout 900 $CS --tool $tool $extra --print-limit 50 \
    python tools/sanitize_driver.py > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/sanitize_$tool.log"
  tail -4 "$OUT/sanitize_$tool.log"
done
