"""bench.py — JSON parse throughput on B200 (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[1] = C1, a 64 MiB pretty-printed
document (random tree, 30% non-ASCII string chars, escapes), seeded synthetic
(tools/jtgen.c) standing in for the paper's public datasets.  One step = one
full parse (stage 1 + stage 2, the jt_parse path) of that document.

  value  = input bytes / device time of the full parse, input resident in HBM
           (CUDA events on the parser's stream; L2 flushed before every step by
           a 256 MiB memset outside the events)
  e2e    = same metric through the public C ABI jt_parse with a pinned host
           input and the host document (tape + strings) read back every step
  roofline = dominant kernel: algorithmic bytes / its event-timed duration
  cpu_baseline = the unmodified reference (oracle/_ref) on 1 core

N > 1 (torchrun, one process per GPU): ONE document of N x 64 MiB, split
into N tile-aligned byte ranges; rank g parses shard g (paper_1902_08318_b200
.shard: four phases with an NCCL all_gather of a small summary after each:
carry functions, counts, open-container stacks, first error + bracket
patches).  Per-GPU work is fixed as N grows (weak scaling); value = document
bytes / max-over-ranks device time.  --shard runs this path at N = 1 too.

--impl reference: the reference's own CPU parser (oracle/_ref, jt_parse) on
the same document, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "JSON parsed GB/s (stage1 & full tape) at 1/2/4/8 B200; % of HBM roofline"
WORKLOAD = ("C1: 64 MiB single document, pretty-printed (2-space, LF), random tree "
            "branching 1-10 depth<=8, 30% non-ASCII string chars, 10% strings with escapes")
CONFIG = 1
PROFILE = "r01d_ncu_full_c1.json"  # ncu --set full capture of the current kernels (traffic)
SIZE = 64 << 20


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def wait_first(self, timeout=3.0):
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def max_over_ranks(value: float, dist=None, device="cpu") -> float:
    """Max of a per-rank scalar (device time of the timed region) over all
    ranks; identity without a process group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(bytes_per_rank: int, steps: int, world: int, max_total_ms: float) -> float:
    """Whole-job GB/s: every rank parses its own copy (replicas, weak
    scaling), so all ranks' bytes divided by the slowest rank's time."""
    return world * bytes_per_rank * steps / (max_total_ms / 1e3) / 1e9


def reference_all_threads(data: bytes, steps: int, warmup: int = 1):
    """The reference's parse on all host cores: one jt_parser per thread
    (thread-compatible, jsontape.h:1-4; the reference cannot split one
    document), every thread parsing `data` once per step.  Returns
    (aggregate GB/s, threads, one-thread GB/s, kind, step times)."""
    import threading
    from oracle.pyoracle import REF_SO, Oracle, Reference
    n = len(data)
    kind = "reference" if os.path.exists(REF_SO) else "port"

    def make():
        return Reference() if kind == "reference" else Oracle()

    def parse_once(obj):
        if kind == "reference":
            obj.parse_code(data)
        else:
            obj.parse(data)
    # bounded so the per-thread buffers (~7 x the document) stay within 24 GB
    threads = max(1, min(os.cpu_count() or 1, 64, (24 << 30) // max(1, 7 * n)))
    objs = [make() for _ in range(threads)]
    t0 = time.perf_counter()
    parse_once(objs[0])
    one = time.perf_counter() - t0

    def step():
        ths = [threading.Thread(target=parse_once, args=(o,)) for o in objs]
        t = time.perf_counter()
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        return time.perf_counter() - t
    times = []
    for i in range(warmup + steps):
        dt = step()
        if i >= warmup:
            times.append(dt)
    return threads * n * len(times) / sum(times) / 1e9, threads, n / one / 1e9, kind, times


def run_reference(args, rank: int, world: int):
    """The reference's own CPU parse (oracle/_ref: the unmodified sources) on
    this box's host cores, all threads (reference_all_threads); the
    one-thread rate is reported beside it."""
    if rank != 0:
        return
    from tools.gen import generate
    size = args.size or (SIZE if args.config == CONFIG else None)
    data = generate(args.config, size)
    n = len(data)
    v, threads, one, kind, times = reference_all_threads(data, args.steps, args.warmup)
    sample = (f"per step {threads} threads, each jt_parse of the full document (incl. its padded copy) "
              f"with its own parser; 1 thread alone: {one:.3f} GB/s")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(times) / len(times) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": WORKLOAD if args.config == CONFIG else f"config {args.config}", "bytes": n,
                   "parallelism": f"{threads} host threads (one document each)"},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": threads, "kind": kind, "sample": sample,
                         "one_thread_gbs": one},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_sharded(args, rank: int, world: int, local: int, torch, dist):
    """One document, world byte-range shards, NCCL exchanges (see header)."""
    from paper_1902_08318_b200 import Parser
    from paper_1902_08318_b200 import shard as SH
    from tools.gen import generate
    size = args.size or SIZE
    data = generate(args.config, size * world)
    n = len(data)
    begin, end = SH.layout(n, world)[rank]
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    p = Parser()
    p.set_stream(stream.cuda_stream)
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    p.copy_in(host.data_ptr(), n)  # whole document resident: the halo is everything
    torch.cuda.synchronize()
    if dist is None:  # --shard at N = 1: a one-rank NCCL group for the same exchanges
        import torch.distributed as D
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        D.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        dist = D
    ex = SH.nccl_exchange(dist, world)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    name, off = SH.run_shard(p, n, rank, world, ex)
    assert name == "OK", (name, off)
    ext = SH.extent(p)  # tape words ext[2], string bytes ext[4], tokens ext[6]
    launches = p.last_launches()
    for _ in range(args.warmup):
        flush.zero_()
        assert SH.run_shard(p, n, rank, world, ex)[0] == "OK"

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        clk.wait_first()
        for k in range(args.steps):
            flush.zero_()
            starts[k].record(stream)
            mark = (lambda ph, k=k: mids[k].record(stream) if ph == 1 else None)
            assert SH.run_shard(p, n, rank, world, ex, mark=mark)[0] == "OK"
            ends[k].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    s1_ms = statistics.median(s.elapsed_time(m) for s, m in zip(starts, mids))
    tot_ms = max_over_ranks(sum(step_ms), dist, "cuda")
    value = n * args.steps / (tot_ms / 1e3) / 1e9

    # e2e: pinned host bytes of this shard (+64 B before, 64 KiB after) -> device,
    # sharded parse, this shard's tape words and string bytes -> pinned host
    lo, hi = max(0, begin - 64), min(n, end + (64 << 10))
    tape_h = torch.empty(max(1, ext[2]) * 8, dtype=torch.uint8).pin_memory()
    str_h = torch.empty(max(1, ext[4]), dtype=torch.uint8).pin_memory()
    e2e_ms = []
    for k in range(args.warmup + args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        assert p._lib.jt_b200_copy_in_range(p._h, host.data_ptr(), lo, hi - lo) == 0
        assert SH.run_shard(p, n, rank, world, ex)[0] == "OK"
        assert p._lib.jt_b200_shard_download(p._h, tape_h.data_ptr(), str_h.data_ptr()) == 0
        e1.record(stream)
        e1.synchronize()
        if k >= args.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
    e2e_tot = max_over_ranks(sum(e2e_ms), dist, "cuda")
    e2e_v = n * args.steps / (e2e_tot / 1e3) / 1e9

    peak, peak_src = peaks()
    rn = end - begin
    B1 = rn + 4 * ext[6]
    B2 = rn + 8 * ext[2] + ext[4]
    per_step = tot_ms / args.steps
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": (WORKLOAD if args.config == CONFIG else f"config {args.config}")
                       + f"; one document of {world} x {size} bytes, {world} byte-range shards",
                       "bytes": n, "shard_bytes": rn,
                       "l2": "flushed before every step (256 MiB memset, outside the events)",
                       "parallelism": f"{world} shards (NCCL all_gather x4 per parse)"},
            "stage1_gbs": n / (s1_ms / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": "full parse of rank 0's shard",
                         "achieved": B2 / (per_step / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": B2 / (per_step / 1e3) / 1e9 / peak, "traffic": None,
                         "peak_source": peak_src},
            "roofline_stage1": {"achieved": B1 / (s1_ms / 1e3) / 1e9,
                                "frac": B1 / (s1_ms / 1e3) / 1e9 / peak, "bytes": B1},
            "cpu_baseline": None,
            "e2e": {"value": e2e_v, "unit": "GB/s", "h2d_bytes_per_step": hi - lo,
                    "d2h_bytes_per_step": 8 * ext[2] + ext[4]},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def record_ranges(data: bytes, world: int) -> list[tuple[int, int]]:
    """Split an NDJSON buffer on record boundaries: rank g starts after the
    first '\n' at or after g/world of the bytes."""
    n = len(data)
    cuts = [0]
    for g in range(1, world):
        k = data.find(b"\n", g * n // world)
        cuts.append(n if k < 0 else k + 1)
    cuts.append(n)
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


def run_records(args, rank: int, world: int, local: int, torch, dist):
    """C3: NDJSON records, each parsed as jt_parse(record) would, in one pass
    per GPU (jt_b200_parse_records).  N > 1: one buffer of N x size bytes cut
    on record boundaries; ranks need no exchange but an all_gather of their
    record counts (global record numbering)."""
    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    size = args.size or (64 << 20)
    data = generate(3, size * world)
    b, e = record_ranges(data, world)[rank]
    mine = data[b:e]
    n = len(mine)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    p = Parser()
    p.set_stream(stream.cuda_stream)
    host = torch.frombuffer(bytearray(mine), dtype=torch.uint8).pin_memory()
    p.copy_in(host.data_ptr(), n)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = p.parse_records(n, download=False)
    nrec = len(res)
    bad = sum(1 for r in res if r[0] != "OK")
    counts = torch.tensor([nrec], dtype=torch.int64, device="cuda")
    if dist:
        allc = torch.empty(world, dtype=torch.int64, device="cuda")
        dist.all_gather_into_tensor(allc, counts)
        first_record = int(allc[:rank].sum().item())
    else:
        first_record = 0
    cnt = C.c_size_t()
    for _ in range(args.warmup):
        flush.zero_()
        assert p._lib.jt_b200_parse_records(p._h, n, C.byref(cnt)) == 0
    launches = p.last_launches()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        clk.wait_first()
        for k in range(args.steps):
            flush.zero_()
            starts[k].record(stream)
            assert p._lib.jt_b200_parse_records(p._h, n, C.byref(cnt)) == 0  # one host sync inside
            ends[k].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    tot_ms = max_over_ranks(sum(s.elapsed_time(e) for s, e in zip(starts, ends)), dist, "cuda")
    total_bytes = len(data)
    value = total_bytes * args.steps / (tot_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    sz = (C.c_ulonglong * 2)()
    p._lib.jt_b200_records_size(p._h, sz)
    if rank == 0:
        cpu = None
        if not args.no_cpu and world == 1:
            try:
                from oracle.pyoracle import Reference
                ref = Reference()
                recs = mine.split(b"\n")[:20000]
                t0 = time.perf_counter()
                for r in recs:
                    ref.parse_code(r)
                dt = time.perf_counter() - t0
                sb = sum(len(r) + 1 for r in recs)
                cpu = {"value": sb / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference",
                       "sample": f"first {len(recs)} records, one reference jt_parse each, 1 thread"}
            except Exception as ex:
                cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "port", "sample": str(ex)}
        per_step = tot_ms / args.steps
        B2 = n + 8 * int(sz[0]) + int(sz[1])
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"C3: NDJSON, lognormal records (mean 256 B), {world} x {size} bytes, "
                                   "each record parsed as jt_parse(record)",
                       "bytes": total_bytes, "records_rank0": nrec, "failed_records_rank0": bad,
                       "first_record_rank0": first_record,
                       "l2": "flushed before every step (256 MiB memset, outside the events)",
                       "parallelism": f"{world} GPUs, record-boundary split" if world > 1 else "1 GPU"},
            "roofline": {"bound": "hbm", "kernel": "record-mode parse of rank 0's records",
                         "achieved": B2 / (per_step / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": B2 / (per_step / 1e3) / 1e9 / peak, "traffic": None,
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": None,
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_select(args, rank: int, world: int, local: int, torch, dist):
    """Parse + select (the paper's parse-then-query use):
    distinct_values at a key path that occurs in the document.  Device:
    resident parse + jt_b200_distinct (selection on the GPU, values and string
    bytes gathered, host sort of the selected values); the same text as
    jt_document_distinct on the downloaded document (checked).  CPU baseline:
    the reference's jt_parse + jt_document_distinct on one core.  Every rank
    runs its own replica (no collective)."""
    import re
    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    size = args.size or (SIZE if args.config == CONFIG else None)
    data = generate(args.config, size)
    n = len(data)
    keys = [m.group(1) for m in re.finditer(rb'"([^"\\.]{1,24})"\s*:', data[:1 << 20])]
    path = keys[0] if keys else b"a"
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    p = Parser()
    p.set_stream(stream.cuda_stream)
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    p.copy_in(host.data_ptr(), n)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    assert p.parse_resident(n).name == "OK"
    want = p.download().distinct(path)
    assert p.distinct(path) == want
    for _ in range(args.warmup):
        p.parse_resident(n)
        p.distinct(path)
    if dist:
        dist.barrier()
    ts = []
    with ClockSampler(local) as clk:
        clk.wait_first()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = p.parse_resident(n)
            out = p.distinct(path)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            assert r.name == "OK" and out == want
    tot_ms = max_over_ranks(sum(ts) * 1e3, dist, "cuda")
    value = job_throughput(n, args.steps, world, tot_ms)
    if rank == 0:
        cpu = None
        if not args.no_cpu:
            try:
                from oracle.pyoracle import Reference
                ref = Reference()
                best = None
                for _ in range(2):
                    t0 = time.perf_counter()
                    got = ref.distinct(data, [path])
                    dt = time.perf_counter() - t0
                    best = dt if best is None else min(best, dt)
                assert got is not None and got[0] == want
                cpu = {"value": n / best / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference",
                       "sample": "full document, reference jt_parse + jt_document_distinct, best of 2, 1 thread"}
            except Exception as e:
                cpu = {"unavailable": e.__class__.__name__}
        print(json.dumps({
            "metric": "JSON parse + select (distinct_values) GB/s", "value": value, "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"config {args.config} + distinct_values at path {path.decode('utf-8', 'replace')!r}",
                       "bytes": n, "distinct_values": want.count(b"\n"),
                       "timing": "host wall clock around resident parse + jt_b200_distinct (synchronous)",
                       "l2": "flushed before every step"},
            "cpu_baseline": cpu, "clocks": clk.summary()}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=CONFIG)
    ap.add_argument("--size", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--shard", action="store_true", help="byte-range shard path even at N = 1")
    ap.add_argument("--select", action="store_true",
                    help="parse + select: distinct_values at a key path (SURVEY.md §8f rank 4)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.select:
        return run_select(args, rank, world, local, torch, dist)
    if args.config == 3:
        return run_records(args, rank, world, local, torch, dist)
    if world > 1 or args.shard:
        return run_sharded(args, rank, world, local, torch, dist)

    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    size = args.size or (SIZE if args.config == CONFIG else None)
    data = generate(args.config, size)
    n = len(data)

    # a real (non-NULL) stream: torch's default stream is the legacy NULL
    # stream, which the C ABI treats as "use the parser's own stream"
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    p = Parser()
    p.set_stream(stream.cuda_stream)
    # device-resident input
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    p.copy_in(host.data_ptr(), n)
    torch.cuda.synchronize()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    r = p.parse_resident(n)
    assert r.name == "OK", (r.name, r.offset)
    S = p.device_index()[1]
    T = p.device_tape()[1]
    SB = p.device_strings()[1]
    launches = p.last_launches()

    # warm-up
    for _ in range(args.warmup):
        flush.zero_()
        p.parse_async(n)
        assert p.finish().code == 0

    # timed region: K full parses, events around each, L2 flush outside
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        clk.wait_first()
        for k in range(args.steps):
            flush.zero_()
            starts[k].record(stream)
            p.parse_async(n)
            ends[k].record(stream)
            assert p.finish().code == 0
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    tot_ms = max_over_ranks(sum(step_ms), dist, "cuda")
    value = job_throughput(n, args.steps, world, tot_ms)

    # per-kernel times (separate profiled passes) for the roofline
    p.profile(True)
    kt_runs = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.zero_()
        p.parse_async(n)
        p.finish()
        kt_runs.append(p.kernel_times())
    p.profile(False)
    kt = {k: statistics.median(r[k] for r in kt_runs) for k in kt_runs[0]}
    s1_ms = kt["stage1"]
    full_ms = sum(kt.values())
    peak, peak_src = peaks()
    # algorithmic bytes: stage 1 B1 = N + 4S; full B2 = N + 8T + strings
    B1 = n + 4 * S
    B2 = n + 8 * T + SB
    # token pass: reads the index (4S) and the input (N), writes token records
    # (4S), scalar tape words (8T) and the string buffer
    Btok = n + 4 * S + 4 * S + 8 * T + SB
    kern_bytes = {"stage1": B1, "tokens": Btok, "struct": 4 * S + 8 * T}
    dom = max(kern_bytes, key=lambda k: kt.get(k, 0.0))
    ach = kern_bytes[dom] / (kt[dom] / 1e3) / 1e9
    # DRAM traffic of the dominant kernel per launch, from the committed
    # `ncu --set full` capture of this workload (profiles/), when it matches
    traffic, traffic_src, alu_pct = None, None, None
    try:
        with open(os.path.join(ROOT, "profiles", PROFILE)) as f:
            prof = json.load(f)
        kname = {"stage1": "k_stage1<0>", "tokens": "k_scalars", "struct": "k_struct<0, 0>"}[dom]
        e = next(v for k, v in prof.items() if k.endswith(kname))
        if args.config == CONFIG and not args.size:
            traffic = (float(e["dram__bytes_read.sum"]) + float(e["dram__bytes_write.sum"])) * 1e6
            traffic_src = f"profiles/{PROFILE} {kname} dram read+write per launch"
        alu_pct = float(e["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"])
    except Exception:
        pass

    # jt_stage1 alone (the reference's stage 1: UTF-8 check + structural
    # index, k_index), device-resident input, L2 flushed before each call
    s1i_ms = []
    for k in range(args.warmup + args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        p.stage1_async(n)
        e1.record(stream)
        r1 = p.finish()
        assert r1.name == "OK" and p.device_index()[1] == S
        if k >= args.warmup:
            s1i_ms.append(e0.elapsed_time(e1))
    s1i = statistics.median(s1i_ms)

    # e2e through the public C ABI: pinned host input -> jt_parse -> host document
    e2e_ms = []
    for k in range(args.warmup + args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rr = p._lib.jt_parse(p._h, C.c_char_p(host.data_ptr()), n, C.byref(doc_ptr := C.c_void_p()),
                             None)
        e1.record(stream)
        e1.synchronize()
        assert rr == 0
        p._lib.jt_document_free(doc_ptr)
        if k >= args.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
    e2e_tot = max_over_ranks(sum(e2e_ms), dist, "cuda")
    e2e_v = job_throughput(n, args.steps, world, e2e_tot)

    if rank == 0:
        cpu = None
        if not args.no_cpu:
            v, threads, one, kind, _ = reference_all_threads(data, 3)
            cpu = {"value": v, "unit": "GB/s", "cores": threads, "kind": kind,
                   "sample": (f"the full document, 3 steps of {threads} threads each parsing it with "
                              f"its own parser (jt_parse incl. its padded copy); 1 thread alone: "
                              f"{one:.3f} GB/s"),
                   "one_thread_gbs": one}
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD if args.config == CONFIG else f"config {args.config}",
                       "bytes": n, "structurals": S, "tape_words": T, "string_bytes": SB,
                       "l2": "flushed before every step (256 MiB memset, outside the events)",
                       "parallelism": "replicas" if world > 1 else "1 GPU"},
            "stage1_gbs": n / (s1i / 1e3) / 1e9,
            "stage1_ms": s1i,
            "stage1_in_parse_ms": s1_ms,
            "kernel_ms": kt,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_bytes": kern_bytes[dom], "peak_source": peak_src,
                         # the integer ALU pipe (LOP3/SHF/IADD3/PRMT, 16 lanes per SMSP
                         # per clock) is what binds these kernels, not HBM
                         "alu_pipe_pct_of_peak": alu_pct},
            "roofline_stage1": {"achieved": B1 / (s1i / 1e3) / 1e9, "frac": B1 / (s1i / 1e3) / 1e9 / peak,
                                "bytes": B1, "path": "jt_stage1 (k_init, k_index, k_stage1_final)"},
            "roofline_full": {"achieved": B2 / (tot_ms / args.steps / 1e3) / 1e9,
                              "frac": B2 / (tot_ms / args.steps / 1e3) / 1e9 / peak, "bytes": B2},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_v, "unit": "GB/s", "h2d_bytes_per_step": n,
                    "d2h_bytes_per_step": 8 * T + SB + 64},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
