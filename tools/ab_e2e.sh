#!/bin/sh
# e2e knob A/B (streamed jt_parse, pinned input): call times per setting
#   sh tools/ab_e2e.sh CONFIG
C=${1:-4}
for s in "" "JT_UP_PIECES=4" "JT_D2H_MIN_KB=16384" "JT_UP_PIECES=4 JT_D2H_MIN_KB=16384" "JT_CHUNK_KB=8192" "JT_CHUNK_KB=8192 JT_UP_PIECES=1" "JT_RANGE_PCTS=40,65,85" "JT_UP_PIECES=8 JT_D2H_MIN_KB=32768"; do
  echo "== $s"
  env $s python tools/trace_e2e.py --config $C --reps 4 2>&1 | grep "^call" | tail -n 3
done
