"""bench.py — JSON parse throughput on B200 (BASELINE.json metric).

Headline workload (N=1): BASELINE.json configs[4] = C4, the 1 GiB
adversarial single document (strings dense in backslash runs, depth up to
1024, mixed UTF-8) — the largest single-GPU config; seeded synthetic
(tools/jtgen.c) standing in for the paper's public datasets.  One step = one
full parse (stage 1 + stage 2, the jt_parse path) of that document.

  value  = input bytes / device time of the full parse, input resident in HBM
           (CUDA events on the parser's stream; L2 flushed before every step by
           a 256 MiB memset outside the events)
  e2e    = same metric through the public C ABI jt_parse with a pinned host
           input and the host document (tape + strings) read back every step;
           e2e_pageable = the same from an ordinary (pageable) host buffer
  parity = the timed document's structural index, tape and string buffer
           (sha256) equal what the UNMODIFIED reference produced for it
           (tests/golden/large_outputs.json); also the e2e document
  roofline = dominant kernel: algorithmic bytes / its event-timed duration
  cpu_baseline = the unmodified reference (oracle/_ref, jt_parse) on all host
           cores (oracle/ref_driver.c: one pthread + parser per core, each
           parsing the document) and on one core
  configs = the other BASELINE configs, one short measurement each (C0 1 MiB,
           C1 64 MiB, C2 256 MiB, C3 1 GiB NDJSON records), same keys.

N > 1 (torchrun, one process per GPU), strong scaling on the 1 GiB inputs:
  * --config 4 (default): ONE 1 GiB document split into N tile-aligned byte
    ranges; rank g uploads only [begin - 64, end + 64 KiB) of it and parses
    shard g (paper_1902_08318_b200.shard: four phases, an NCCL all_gather of a
    small summary after each).  value = document bytes / max-over-ranks time.
  * --config 3: the 1 GiB NDJSON buffer cut on record boundaries; rank g
    parses its records (no data exchange; an all_gather of record counts).

--impl reference: the reference's own CPU parser (oracle/_ref, jt_parse) on
the same workload on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
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
WORKLOADS = {
    0: "C0: 1 MiB minified document, ~5,000 flat 6-key objects",
    1: ("C1: 64 MiB single document, pretty-printed (2-space, LF), random tree branching 1-10 "
        "depth<=8, 30% non-ASCII string chars, 10% strings with escapes"),
    2: "C2: 256 MiB number-heavy document, 1M rows x 16 numbers (90% %.17g floats, 10% int64)",
    3: "C3: 1 GiB NDJSON, ~3.9M lognormal records (mean 256 B), each parsed as jt_parse(record)",
    4: ("C4: 1 GiB adversarial single document: strings up to 64 KiB dense in backslash runs 1-9 "
        "and embedded quotes, nesting up to 1024, mixed UTF-8"),
}
CONFIG = 4           # headline: the largest single-GPU config
TABLE = (0, 1, 2, 3)  # the other configs, one short line each inside the headline's JSON
# ncu --set full captures of the current kernels (DRAM traffic per launch)
PROFILES = {4: "r02d_ncu_full_c4.json"}
FIXTURE = os.path.join(ROOT, "tests", "golden", "large_outputs.json")
L2_NOTE = "flushed before every step (256 MiB memset, outside the events)"
# JT_BENCH_GLOO=1 runs the N > 1 paths with every rank on cuda:0 and gloo
# collectives over host tensors: a functional check of the multi-GPU code on a
# one-GPU box (ranks share the GPU; its times are not a scaling measurement)
GLOO_TEST = os.environ.get("JT_BENCH_GLOO") == "1"
COLL = "cpu" if GLOO_TEST else "cuda"  # device of the collectives' tensors


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
    """Whole-job GB/s when every rank parses its own copy (replicas)."""
    return world * bytes_per_rank * steps / (max_total_ms / 1e3) / 1e9


def sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def fixture(config: int, n: int):
    """The reference's results for the seeded config document of n bytes
    (tests/golden/large_outputs.json, made from oracle/_ref), or None."""
    try:
        with open(FIXTURE) as f:
            fx = json.load(f)
    except OSError:
        return None
    rows = [fx["records"]] if config == 3 else fx["clean"]
    return next((r for r in rows if r["config"] == config and r["bytes"] == n), None)


def generate(config: int, size=None) -> bytes:
    from tools.gen import generate as gen
    return gen(config, size)


# ---- CPU baseline: the unmodified reference on the host cores ---------------

def host_threads(n: int, bytes_per_input_byte: float) -> int:
    """All host cores, bounded so the reference's per-thread buffers (padded
    copy, index, tape, strings: ~7 bytes per input byte) fit in 60% of the
    available host memory."""
    cores = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 32 << 30
    return max(1, min(cores, 128, int(0.6 * avail // max(1, bytes_per_input_byte * n))))


def reference_document(data: bytes, reps: int = 2):
    """The reference's jt_parse of the whole document on all host cores (each
    thread its own parser, oracle/ref_driver.c) and on one core."""
    from oracle.pyoracle import REF_SO, RefDriver
    n = len(data)
    if not os.path.exists(REF_SO):
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built on this box"}
    d = RefDriver()
    t1, code = d.parse_many(data, 1, 1)
    threads = host_threads(n, 7.0)
    tn, code_n = d.parse_many(data, threads, reps)
    assert code == code_n == 0, (code, code_n)
    return {"value": threads * n * reps / tn / 1e9, "unit": "GB/s", "cores": threads, "kind": "reference",
            "sample": (f"the full document: {reps} passes of {threads} pthreads, each jt_parse()ing it with "
                       f"its own parser (the reference cannot split one document; oracle/ref_driver.c); "
                       f"1 thread alone: {n / t1 / 1e9:.3f} GB/s"),
            "one_thread_gbs": n / t1 / 1e9}


def reference_records(data: bytes, reps: int = 2):
    """The reference's jt_parse of every NDJSON record on all host cores
    (records dealt to the threads in contiguous slices) and on one core (a
    64 MiB prefix)."""
    from oracle.pyoracle import REF_SO, RefDriver
    n = len(data)
    if not os.path.exists(REF_SO):
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built on this box"}
    d = RefDriver()
    cut = data.find(b"\n", min(n, 64 << 20))
    head = data if cut < 0 else data[:cut + 1]
    t1, _, _ = d.parse_records(head, 1, 1)
    threads = host_threads(n, 0.2)
    tn, nr, ok = d.parse_records(data, threads, reps)
    return {"value": n * reps / tn / 1e9, "unit": "GB/s", "cores": threads, "kind": "reference",
            "sample": (f"all {nr} records, {reps} passes, dealt to {threads} pthreads in contiguous slices, "
                       f"each record jt_parse()d alone (oracle/ref_driver.c); {ok} OK; 1 thread on the "
                       f"first {len(head) >> 20} MiB: {len(head) / t1 / 1e9:.3f} GB/s"),
            "one_thread_gbs": len(head) / t1 / 1e9, "records": nr}


def run_reference(args, rank: int, world: int):
    """--impl reference: the reference's own CPU parse (oracle/_ref: the
    unmodified sources) of the same workload on this box's host cores."""
    if rank != 0:
        return
    data = generate(args.config, args.size)
    n = len(data)
    from oracle.pyoracle import REF_SO, RefDriver
    if not os.path.exists(REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}), flush=True)
        return
    d = RefDriver()
    if args.config == 3:
        d.parse_records(data[:1 << 20], 1, 1)
        threads = host_threads(n, 0.2)
        times = []
        for i in range(args.warmup + args.steps):
            dt, nr, ok = d.parse_records(data, threads, 1)
            if i >= args.warmup:
                times.append(dt)
        v = n * len(times) / sum(times) / 1e9
        sample = f"all {nr} records per step dealt to {threads} pthreads, each record jt_parse()d alone"
    else:
        threads = host_threads(n, 7.0)
        # a 1 GiB document takes seconds per thread: one untimed pass inside
        # the driver per call, then args.steps timed passes (bounded)
        reps = max(1, min(args.steps, 3 if n >= (256 << 20) else args.steps))
        dt, code = d.parse_many(data, threads, reps)
        assert code == 0, code
        times = [dt / reps] * reps
        v = threads * n * reps / dt / 1e9
        sample = (f"{reps} passes of {threads} pthreads, each jt_parse()ing the whole document with its "
                  f"own parser (the reference cannot split one document)")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": sum(times) / len(times) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "bytes": n,
                   "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- one GPU: single documents -------------------------------------------------

def kernel_profile(p, n, flush, reps):
    """per-kernel event times (ms) of the full parse, median of `reps`"""
    p.profile(True)
    runs = []
    for _ in range(reps):
        flush.zero_()
        p.parse_async(n)
        p.finish()
        runs.append(p.kernel_times())
    p.profile(False)
    return {k: statistics.median(r[k] for r in runs) for k in runs[0]}


def e2e_loop(torch, p, stream, ptr, n, steps, warmup):
    """jt_parse through the C ABI from host memory at `ptr`, host document
    back; returns (ms per call list, the last document handle)."""
    ms, last = [], None
    for k in range(warmup + steps):
        doc = C.c_void_p()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rr = p._lib.jt_parse(p._h, C.c_char_p(ptr), n, C.byref(doc), None)
        e1.record(stream)
        e1.synchronize()
        assert rr == 0, rr
        if k >= warmup:
            ms.append(e0.elapsed_time(e1))
        if last is not None:
            p._lib.jt_document_free(last)
        last = doc
    return ms, last


def measure_document(torch, config, steps, warmup, flush, full, clk_index=None, size=None):
    """Device-resident full parse, jt_stage1, e2e (pinned; + pageable when
    `full`) and parity against the reference's fixture for one config."""
    from paper_1902_08318_b200 import Parser
    from paper_1902_08318_b200.jsontape import Document
    data = generate(config, size)
    n = len(data)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    # a real (non-NULL) stream: torch's default stream is the legacy NULL
    # stream, which the C ABI treats as "use the parser's own stream"
    p = Parser()
    p.set_stream(stream.cuda_stream)
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    p.copy_in(host.data_ptr(), n)
    torch.cuda.synchronize()
    r = p.parse_resident(n)
    assert r.name == "OK", (r.name, r.offset)
    S = p.device_index()[1]
    T = p.device_tape()[1]
    SB = p.device_strings()[1]
    launches = p.last_launches()
    for _ in range(warmup):
        flush.zero_()
        p.parse_async(n)
        assert p.finish().code == 0
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    torch.cuda.synchronize()
    clk = ClockSampler(clk_index) if clk_index is not None else None
    if clk:
        clk.__enter__()
        clk.wait_first()
    for k in range(steps):
        flush.zero_()
        starts[k].record(stream)
        p.parse_async(n)
        ends[k].record(stream)
        assert p.finish().code == 0
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    out = {"bytes": n, "S": S, "T": T, "SB": SB, "launches": launches, "steps": steps,
           "tot_ms": sum(step_ms), "ms_per_step": sum(step_ms) / steps,
           "value": n * steps / (sum(step_ms) / 1e3) / 1e9,
           "clocks": clk.summary() if clk else None}

    # parity of the timed document: the last timed parse is what is on the device
    fx = fixture(config, n)
    par = {"checked": False}
    if fx is not None:
        assert sha(data) == fx["input_sha"], "generator drifted"
        idx = p.index()
        doc = p.download()
        got = {"index_sha": sha(idx.tobytes()), "tape_sha": sha(doc.tape.tobytes()),
               "strings_sha": sha(doc.strings), "S": len(idx), "T": len(doc.tape),
               "string_bytes": len(doc.strings)}
        bad = [k for k, v in got.items() if v != fx[k]]
        assert not bad, f"parity: config {config} timed document differs from the reference in {bad}"
        par = {"checked": True, "against": "tests/golden/large_outputs.json (oracle/_ref)",
               "index": True, "tape": True, "strings": True}
        del idx, doc

    # per-kernel event times (separate profiled passes) for the roofline
    out["kernel_ms"] = kernel_profile(p, n, flush, max(3, min(steps, 10)))

    # jt_stage1 alone (k_index), device-resident input
    s1 = []
    for k in range(warmup + steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        p.stage1_async(n)
        e1.record(stream)
        r1 = p.finish()
        assert r1.name == "OK" and p.device_index()[1] == S
        if k >= warmup:
            s1.append(e0.elapsed_time(e1))
    out["stage1_ms"] = statistics.median(s1)

    # e2e through the public C ABI: host input -> jt_parse -> host document
    ms, last = e2e_loop(torch, p, stream, host.data_ptr(), n, steps, warmup)
    out["e2e_ms"] = ms
    if fx is not None:
        d = Document(last.value)
        assert sha(d.tape.tobytes()) == fx["tape_sha"] and sha(d.strings) == fx["strings_sha"], \
            "parity: e2e document differs from the reference"
        par["e2e_document"] = True
        del d
    else:
        p._lib.jt_document_free(last)
    if full:
        buf = C.create_string_buffer(data, n)  # ordinary malloc'd (pageable) host memory
        msp, lastp = e2e_loop(torch, p, stream, C.addressof(buf), n, steps, warmup)
        p._lib.jt_document_free(lastp)
        out["e2e_pageable_ms"] = msp
        del buf
    out["parity"] = par
    out["data"] = data if full else None
    p.close()
    del host
    return out


def measure_records(torch, steps, warmup, flush, size=None, with_cpu=True):
    """C3 on one GPU: device-resident record-mode parse, e2e (pinned input up,
    per-record results + tape + strings down) and parity of every record."""
    import numpy as np
    from paper_1902_08318_b200 import Parser
    data = generate(3, size)
    n = len(data)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    p = Parser()
    p.set_stream(stream.cuda_stream)
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    p.copy_in(host.data_ptr(), n)
    torch.cuda.synchronize()
    cnt = C.c_size_t()
    for _ in range(warmup):
        flush.zero_()
        assert p._lib.jt_b200_parse_records(p._h, n, C.byref(cnt)) == 0
    launches = p.last_launches()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    torch.cuda.synchronize()
    for k in range(steps):
        flush.zero_()
        starts[k].record(stream)
        assert p._lib.jt_b200_parse_records(p._h, n, C.byref(cnt)) == 0  # one host sync inside
        ends[k].record(stream)
    torch.cuda.synchronize()
    tot = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    sz = (C.c_ulonglong * 2)()
    p._lib.jt_b200_records_size(p._h, sz)
    nrec = cnt.value
    # e2e: pinned host buffer -> device, record parse, per-record results
    # (jt_b200_records) + all records' tape words and strings -> host
    tape_h = torch.empty(max(1, int(sz[0])) * 8, dtype=torch.uint8).pin_memory()
    str_h = torch.empty(max(1, int(sz[1])), dtype=torch.uint8).pin_memory()
    e2e = []
    for k in range(warmup + steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        p.copy_in(host.data_ptr(), n)
        assert p._lib.jt_b200_parse_records(p._h, n, C.byref(cnt)) == 0
        assert p._lib.jt_b200_records(p._h)
        assert p._lib.jt_b200_records_download(p._h, tape_h.data_ptr(), str_h.data_ptr()) == 0
        e1.record(stream)
        e1.synchronize()
        if k >= warmup:
            e2e.append(e0.elapsed_time(e1))
    # parity: every record's code / offset, and the OK records' tape words and strings
    arr, tape, strings = p.parse_records_arrays(n)
    fx = fixture(3, n)
    par = {"checked": False}
    if fx is not None:
        assert sha(data) == fx["input_sha"], "generator drifted"
        ok = arr["code"] == 0
        got = {"records": int(len(arr)), "ok": int(ok.sum()),
               "codes_sha": sha(np.ascontiguousarray(arr["code"], dtype=np.int32).tobytes()),
               "offsets_sha": sha(np.ascontiguousarray(arr["offset"], dtype=np.int64).tobytes()),
               "tape_sha": sha(gather(tape, arr["tape_begin"][ok], arr["tape_words"][ok]).tobytes()),
               "strings_sha": sha(gather(strings, arr["string_begin"][ok], arr["string_bytes"][ok]).tobytes())}
        bad = [k for k, v in got.items() if v != fx[k]]
        assert not bad, f"parity: C3 records differ from the reference in {bad}"
        par = {"checked": True, "against": "tests/golden/large_outputs.json (oracle/_ref, per record)",
               "records": got["records"]}
    out = {"bytes": n, "records": nrec, "tape_words": int(sz[0]), "string_bytes": int(sz[1]),
           "steps": steps, "ms_per_step": tot / steps, "value": n * steps / (tot / 1e3) / 1e9,
           "launches": launches, "parity": par,
           "e2e": {"value": n * steps / (sum(e2e) / 1e3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": n,
                   "d2h_bytes_per_step": 8 * int(sz[0]) + int(sz[1]) + 48 * nrec}}
    if with_cpu:
        out["cpu_baseline"] = reference_records(data)
    p.close()
    return out


def gather(buf, begin, count):
    """Concatenate buf[begin[k]:begin[k]+count[k]] (vectorised)."""
    import numpy as np
    count = count.astype(np.int64)
    total = int(count.sum())
    if total == 0:
        return buf[:0]
    starts = np.repeat(begin.astype(np.int64) - np.concatenate(([0], np.cumsum(count)[:-1])), count)
    return buf[starts + np.arange(total, dtype=np.int64)]


def roofline_of(out, config, n):
    """Dominant kernel of the full parse: algorithmic bytes
    over its event-timed duration; DRAM traffic from the committed ncu
    capture of this workload when there is one."""
    peak, peak_src = peaks()
    kt = out["kernel_ms"]
    S, T, SB = out["S"], out["T"], out["SB"]
    B1 = n + 4 * S               # stage 1: input read, index written
    B2 = n + 8 * T + SB          # full parse: input read, tape + string buffer written
    # token pass: reads the index (4S) and the input (N), writes token
    # records (4S), scalar tape words (8T) and the string buffer
    kern_bytes = {"stage1": B1, "tokens": n + 8 * S + 8 * T + SB, "struct": 4 * S + 8 * T}
    dom = max(kern_bytes, key=lambda k: kt.get(k, 0.0))
    ach = kern_bytes[dom] / (kt[dom] / 1e3) / 1e9
    traffic, traffic_src, alu = None, None, None
    prof = PROFILES.get(config)
    if prof:
        try:
            with open(os.path.join(ROOT, "profiles", prof)) as f:
                pr = json.load(f)
            kname = {"stage1": ("k_carry_fn<0>", "k_carry_scan", "k_stage1<0>"), "tokens": ("k_scalars",),
                     "struct": ("k_struct<0, 0>",)}[dom]
            es = [v for k, v in pr.items() if k != "units" and k.endswith(kname)]
            if "units" in pr and pr.get("input_bytes", n) == n and len(es) == len(kname):
                traffic = sum(float(e["dram__bytes_read.sum"]) + float(e["dram__bytes_write.sum"]) for e in es)
                traffic_src = f"profiles/{prof}: {'+'.join(kname)} DRAM read+write per launch (ncu --set full)"
            alu = float(es[-1]["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"])
        except Exception:
            pass
    per_step_s = out["ms_per_step"] / 1e3
    return {
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes": kern_bytes[dom], "peak_source": peak_src,
                     # the integer ALU pipe is what binds these kernels
                     "alu_pipe_pct_of_peak": alu},
        "roofline_stage1": {"achieved": B1 / (out["stage1_ms"] / 1e3) / 1e9,
                            "frac": B1 / (out["stage1_ms"] / 1e3) / 1e9 / peak, "bytes": B1,
                            "path": "jt_stage1 (k_index)"},
        "roofline_full": {"achieved": B2 / per_step_s / 1e9, "frac": B2 / per_step_s / 1e9 / peak,
                          "bytes": B2, "path": "full parse (all kernels)"},
    }


def doc_line(out, config, steps):
    n = out["bytes"]
    e2e_v = n * steps / (sum(out["e2e_ms"]) / 1e3) / 1e9
    line = {"value": out["value"], "unit": "GB/s", "ms_per_step": out["ms_per_step"],
            "config": {"workload": WORKLOADS[config], "bytes": n, "structurals": out["S"],
                       "tape_words": out["T"], "string_bytes": out["SB"], "l2": L2_NOTE},
            "stage1_gbs": n / (out["stage1_ms"] / 1e3) / 1e9, "stage1_ms": out["stage1_ms"],
            "kernel_ms": out["kernel_ms"],
            "e2e": {"value": e2e_v, "unit": "GB/s", "h2d_bytes_per_step": n,
                    "d2h_bytes_per_step": 8 * out["T"] + out["SB"]},
            "parity": out["parity"]}
    if "e2e_pageable_ms" in out:
        line["e2e_pageable"] = {"value": n * steps / (sum(out["e2e_pageable_ms"]) / 1e3) / 1e9, "unit": "GB/s",
                                "h2d_bytes_per_step": n, "d2h_bytes_per_step": 8 * out["T"] + out["SB"],
                                "input": "ordinary malloc'd host buffer"}
    line.update(roofline_of(out, config, n))
    return line


def run_single(args, torch, local):
    """N = 1: the headline config, then one short line per other config."""
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    head = measure_document(torch, args.config, args.steps, args.warmup, flush, True, clk_index=local,
                            size=args.size)
    data = head.pop("data")
    line = {"metric": METRIC, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (tools/jtgen.c, seeded; BASELINE.json config shapes)"}
    line.update(doc_line(head, args.config, args.steps))
    line["config"]["parallelism"] = "1 GPU"
    line["gpu_launches"] = head["launches"] * args.steps
    line["clocks"] = head["clocks"]
    line["cpu_baseline"] = None if args.no_cpu else reference_document(data)
    del data
    if not args.no_table:
        table = {}
        ksteps = max(3, min(args.steps, 10))
        for c in TABLE:
            if c == args.config:
                continue
            if c == 3:
                r = measure_records(torch, ksteps, args.warmup, flush, with_cpu=not args.no_cpu)
                table["C3"] = {"value": r["value"], "unit": "GB/s", "ms_per_step": r["ms_per_step"],
                               "config": {"workload": WORKLOADS[3], "bytes": r["bytes"], "records": r["records"],
                                          "tape_words": r["tape_words"], "string_bytes": r["string_bytes"],
                                          "l2": L2_NOTE},
                               "e2e": r["e2e"], "parity": r["parity"], "cpu_baseline": r.get("cpu_baseline"),
                               "gpu_launches": r["launches"] * ksteps}
                continue
            o = measure_document(torch, c, ksteps, args.warmup, flush, False)
            t = doc_line(o, c, ksteps)
            t["gpu_launches"] = o["launches"] * ksteps
            if not args.no_cpu:
                t["cpu_baseline"] = reference_document(generate(c), reps=1)
            table[f"C{c}"] = t
        line["configs"] = table
    print(json.dumps(line), flush=True)


# ---- N > 1: byte-range shards of one document (strong scaling) -----------------

HALO = 64 << 10  # bytes after a shard's end resident on its GPU (tokens crossing the cut)


def run_sharded(args, rank: int, world: int, local: int, torch, dist):
    """ONE document, world byte-range shards, NCCL exchanges; each rank holds
    only its halo range [begin - 64, end + HALO) (see header)."""
    from paper_1902_08318_b200 import Parser
    from paper_1902_08318_b200 import shard as SH
    data = generate(args.config, args.size)
    n = len(data)
    begin, end = SH.layout(n, world)[rank]
    lo, hi = max(0, begin - 64), min(n, end + HALO)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    p = Parser()
    p.set_stream(stream.cuda_stream)
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    p.input_buffer(n)  # document-sized address space, zero tail; only [lo, hi) is uploaded
    assert p._lib.jt_b200_copy_in_range(p._h, host.data_ptr(), lo, hi - lo) == 0
    SH.set_resident(p, lo, hi)
    torch.cuda.synchronize()
    if dist is None:  # --shard at N = 1: a one-rank NCCL group for the same exchanges
        import torch.distributed as D
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        D.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        dist = D
    ex = SH.host_exchange(dist, world) if GLOO_TEST else SH.nccl_exchange(dist, world)
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
    tot_ms = max_over_ranks(sum(step_ms), dist, COLL)
    value = n * args.steps / (tot_ms / 1e3) / 1e9

    # parity: the shards' tape and string parts, concatenated in rank order on
    # rank 0, are the reference's document (sha256 against the fixture)
    fx = fixture(args.config, n)
    par = {"checked": False}
    if fx is not None:
        _, tape_part, _, str_part = SH.download(p)
        parts = [None] * world if rank == 0 else None
        dist.gather_object((tape_part.tobytes(), str_part), parts, dst=0)
        del tape_part, str_part
        if rank == 0:
            h_t, h_s = hashlib.sha256(), hashlib.sha256()
            nt = ns = 0
            for t, st in parts:
                h_t.update(t)
                h_s.update(st)
                nt += len(t) // 8
                ns += len(st)
            ok = (name == fx["code"] and h_t.hexdigest() == fx["tape_sha"] and h_s.hexdigest() == fx["strings_sha"]
                  and nt == fx["T"] and ns == fx["string_bytes"])
            assert ok, "parity: the sharded document differs from the reference's"
            par = {"checked": True, "against": "tests/golden/large_outputs.json (oracle/_ref)",
                   "tape": True, "strings": True, "shards": world}
        del parts

    # e2e: pinned host bytes of this shard's halo range -> device, sharded
    # parse, this shard's tape words and string bytes -> pinned host
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
    e2e_tot = max_over_ranks(sum(e2e_ms), dist, COLL)
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
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config] + f"; {world} byte-range shards of the one document",
                       "bytes": n, "shard_bytes_rank0": rn, "resident_bytes_rank0": hi - lo,
                       "l2": L2_NOTE, "parallelism": f"{world} shards (NCCL all_gather x4 per parse)"},
            "stage1_gbs": n / (s1_ms / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": "full parse of rank 0's shard",
                         "achieved": B2 / (per_step / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": B2 / (per_step / 1e3) / 1e9 / peak, "traffic": None,
                         "peak_source": peak_src},
            "roofline_stage1": {"achieved": B1 / (s1_ms / 1e3) / 1e9,
                                "frac": B1 / (s1_ms / 1e3) / 1e9 / peak, "bytes": B1},
            "parity": par,
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
    first '\\n' at or after g/world of the bytes."""
    n = len(data)
    cuts = [0]
    for g in range(1, world):
        k = data.find(b"\n", g * n // world)
        cuts.append(n if k < 0 else k + 1)
    cuts.append(n)
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


def record_numbering(dist, world: int, rank: int, count: int, device="cpu") -> tuple[int, int]:
    """Global numbering of the ranks' records: (first record of this rank,
    total records) from an all_gather of the per-rank counts."""
    import torch
    counts = torch.tensor([count], dtype=torch.int64, device=device)
    allc = torch.empty(world, dtype=torch.int64, device=device)
    try:
        dist.all_gather_into_tensor(allc, counts)
    except (RuntimeError, NotImplementedError, AttributeError):  # backends without it (gloo)
        parts = [torch.empty_like(counts) for _ in range(world)]
        dist.all_gather(parts, counts)
        allc = torch.cat(parts)
    return int(allc[:rank].sum().item()), int(allc.sum().item())


def run_records(args, rank: int, world: int, local: int, torch, dist):
    """C3 at N > 1: the 1 GiB NDJSON buffer cut on record boundaries, each
    rank parses its records (jt_b200_parse_records); the only exchange is an
    all_gather of record counts (global record numbering)."""
    from paper_1902_08318_b200 import Parser
    data = generate(3, args.size)
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
    cnt = C.c_size_t()
    assert p._lib.jt_b200_parse_records(p._h, n, C.byref(cnt)) == 0
    first_record, total_records = record_numbering(dist, world, rank, cnt.value, COLL)
    for _ in range(args.warmup):
        flush.zero_()
        assert p._lib.jt_b200_parse_records(p._h, n, C.byref(cnt)) == 0
    launches = p.last_launches()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
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
    dist.barrier()
    tot_ms = max_over_ranks(sum(s.elapsed_time(e) for s, e in zip(starts, ends)), dist, COLL)
    value = len(data) * args.steps / (tot_ms / 1e3) / 1e9
    # e2e: this rank's records up, results + tape + strings down
    sz = (C.c_ulonglong * 2)()
    p._lib.jt_b200_records_size(p._h, sz)
    tape_h = torch.empty(max(1, int(sz[0])) * 8, dtype=torch.uint8).pin_memory()
    str_h = torch.empty(max(1, int(sz[1])), dtype=torch.uint8).pin_memory()
    e2e = []
    for k in range(args.warmup + args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        p.copy_in(host.data_ptr(), n)
        assert p._lib.jt_b200_parse_records(p._h, n, C.byref(cnt)) == 0
        assert p._lib.jt_b200_records(p._h)
        assert p._lib.jt_b200_records_download(p._h, tape_h.data_ptr(), str_h.data_ptr()) == 0
        e1.record(stream)
        e1.synchronize()
        if k >= args.warmup:
            e2e.append(e0.elapsed_time(e1))
    e2e_tot = max_over_ranks(sum(e2e), dist, COLL)
    # parity: every rank's per-record results and OK records' tape words and
    # strings, concatenated in rank order on rank 0, digest to the reference's
    fx = fixture(3, len(data))
    par = {"checked": False}
    if fx is not None:
        import numpy as np
        arr, tape, strings = p.parse_records_arrays(n)
        ok = arr["code"] == 0
        mine_part = (np.ascontiguousarray(arr["code"], dtype=np.int32).tobytes(),
                     np.ascontiguousarray(arr["offset"], dtype=np.int64).tobytes(),
                     gather(tape, arr["tape_begin"][ok], arr["tape_words"][ok]).tobytes(),
                     gather(strings, arr["string_begin"][ok], arr["string_bytes"][ok]).tobytes())
        del arr, tape, strings
        parts = [None] * world if rank == 0 else None
        dist.gather_object(mine_part, parts, dst=0)
        del mine_part
        if rank == 0:
            hs = [hashlib.sha256() for _ in range(4)]
            for part in parts:
                for h, b in zip(hs, part):
                    h.update(b)
            got = [h.hexdigest() for h in hs]
            want = [fx["codes_sha"], fx["offsets_sha"], fx["tape_sha"], fx["strings_sha"]]
            assert got == want and total_records == fx["records"], "parity: records differ from the reference's"
            par = {"checked": True, "against": "tests/golden/large_outputs.json (oracle/_ref, per record)",
                   "records": total_records, "ranks": world}
        del parts
    if rank == 0:
        peak, peak_src = peaks()
        per_step = tot_ms / args.steps
        B2 = n + 8 * int(sz[0]) + int(sz[1])
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOADS[3] + f"; cut on record boundaries into {world} parts",
                       "bytes": len(data), "records": total_records, "records_rank0": cnt.value,
                       "first_record_rank0": first_record, "l2": L2_NOTE,
                       "parallelism": f"{world} GPUs, record-boundary split"},
            "roofline": {"bound": "hbm", "kernel": "record-mode parse of rank 0's records",
                         "achieved": B2 / (per_step / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": B2 / (per_step / 1e3) / 1e9 / peak, "traffic": None, "peak_source": peak_src},
            "parity": par,
            "cpu_baseline": None,
            "e2e": {"value": len(data) * args.steps / (e2e_tot / 1e3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": n, "d2h_bytes_per_step": 8 * int(sz[0]) + int(sz[1]) + 48 * cnt.value},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_select(args, torch, local):
    """Parse + select (the paper's parse-then-query use):
    distinct_values at a key path that occurs in the document, one GPU."""
    import re
    from paper_1902_08318_b200 import Parser
    config = 1 if args.config == CONFIG else args.config
    data = generate(config, args.size)
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
    tot_ms = sum(ts) * 1e3
    cpu = None
    if not args.no_cpu:
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
    print(json.dumps({
        "metric": "JSON parse + select (distinct_values) GB/s", "value": n * args.steps / (tot_ms / 1e3) / 1e9,
        "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"config {config} + distinct_values at path {path.decode('utf-8', 'replace')!r}",
                   "bytes": n, "distinct_values": want.count(b"\n"),
                   "timing": "host wall clock around resident parse + jt_b200_distinct (synchronous)",
                   "l2": "flushed before every step"},
        "cpu_baseline": cpu, "clocks": clk.summary()}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=CONFIG)
    ap.add_argument("--size", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-table", action="store_true", help="headline config only")
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
    torch.cuda.set_device(0 if GLOO_TEST else local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if GLOO_TEST:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.select:
        return run_select(args, torch, local)
    if world > 1:
        if args.config == 3:
            return run_records(args, rank, world, local, torch, dist)
        return run_sharded(args, rank, world, local, torch, dist)
    if args.shard:
        return run_sharded(args, rank, world, local, torch, None)
    if args.config == 3:
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        r = measure_records(torch, args.steps, args.warmup, flush, size=args.size, with_cpu=not args.no_cpu)
        line = {"metric": METRIC, "value": r["value"], "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": {"workload": WORKLOADS[3], "bytes": r["bytes"], "records": r["records"],
                           "l2": L2_NOTE, "parallelism": "1 GPU"},
                "parity": r["parity"], "cpu_baseline": r.get("cpu_baseline"), "e2e": r["e2e"],
                "gpu_launches": r["launches"] * args.steps}
        print(json.dumps(line), flush=True)
        return
    run_single(args, torch, local)


if __name__ == "__main__":
    main()
