#!/bin/sh
# pageable-input e2e A/B of the staging knobs: sh tools/ab_e2e_pageable.sh CONFIG
C=${1:-4}
for s in "JT_UP_PIECES=2" "JT_UP_PIECES=4" "JT_UP_PIECES=4 JT_COPY_THREADS=16" "JT_UP_PIECES=2 JT_COPY_THREADS=16" "JT_UP_PIECES=1"; do
  echo "== $s"
  env $s python tools/trace_e2e.py --config $C --reps 4 --pageable 2>&1 | grep "^call" | tail -n 2
done
