#!/bin/sh
# e2e A/B of the streamed parse's stage-2 range cuts (JT_RANGE_PCTS, % of the
# pieces), pinned input:   sh tools/ab_e2e_ranges.sh [CONFIG]
C=${1:-4}
for s in "" "JT_RANGE_PCTS=30,55,80,93" "JT_RANGE_PCTS=30,60,85,96" "JT_RANGE_PCTS=40,70,90,97" "JT_RANGE_PCTS=50,80,93,98" "JT_RANGE_PCTS=35,65,88,95"; do
  echo "== $s"
  env $s python tools/trace_e2e.py --config $C --reps 5 2>&1 | grep "^call" | tail -n 4
done
