#!/bin/sh
# A/B of library builds on the GPU box: bench.py's headline (and other
# configs) per build, each build loaded through JT_B200_LIB.
#   sh tools/ab_bench.sh "libjsontape_b200 ab_variant ..." "4 1"
# (builds are paper_1902_08318_b200/<name>.so; results in gpurun_out/ab_*.json)
for v in $1; do
  for c in $2; do
    JT_B200_LIB=$PWD/paper_1902_08318_b200/$v.so timeout 300 python bench.py --no-table --no-cpu \
      --config $c --steps 10 > gpurun_out/ab_${v}_c$c.json 2> gpurun_out/ab_${v}_c$c.err
  done
done
for f in gpurun_out/ab_*.json; do
  python - "$f" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(sys.argv[1], round(d["value"], 1), "GB/s; jt_stage1", round(d["stage1_ms"], 4), "ms;",
          {k: round(v, 4) for k, v in d["kernel_ms"].items()})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
