#!/bin/sh
# bench.py's N > 1 paths (strong scaling: C4 byte-range shards, C3 records)
# as 2 and 3 processes sharing the one GPU with gloo collectives
# (JT_BENCH_GLOO=1): a functional check, not a scaling measurement.
for n in 2 3; do
  for c in 4 3; do
    JT_BENCH_GLOO=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29600 + n * 10 + c)) bench.py --gpus $n --config $c \
      --steps 3 --warmup 3 > gpurun_out/mr_n${n}_c$c.json 2> gpurun_out/mr_n${n}_c$c.err
    echo "n=$n c=$c rc=$?"
    python - gpurun_out/mr_n${n}_c$c.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("  value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "parity", d.get("parity"),
          "config", {k: d["config"][k] for k in d["config"] if k in ("shard_bytes_rank0", "resident_bytes_rank0", "records", "records_rank0", "first_record_rank0")})
except Exception as e:
    print("  failed", e)
PY
  done
done
