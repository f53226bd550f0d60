"""Byte-range shards as separate processes (the bench's N > 1 path) on the
one GPU of this environment: every rank has its own parser holding only its
halo range of the document (jt_b200_copy_in_range, as bench.py's e2e leg),
phases exchanged by torch.distributed all_gather over gloo with host
staging (the bench uses NCCL on device tensors; same fixed-size summaries).
The ranks' kernels never wait on one another — exchanges are between phases
on the host — so this checks the per-rank logic, not multi-GPU performance.
Result vs the oracle: code, offset, and the concatenated shard tapes/strings.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, docs, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_1902_08318_b200 import Parser
        from paper_1902_08318_b200 import shard as SH

        def ex(phase, local):  # all_gather over gloo, host staging
            h = local.cpu()
            parts = [torch.empty_like(h) for _ in range(world)]
            dist.all_gather(parts, h)
            return torch.cat(parts).to(local.device)

        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        p = Parser()
        p.set_stream(stream.cuda_stream)  # the copy and the phases on one stream
        out = []
        for item in docs:
            d, halo = item if isinstance(item, tuple) else (item, 64 << 10)
            n = len(d)
            begin, end = SH.layout(n, world)[rank]
            lo, hi = max(0, begin - 64), min(n, end + halo)
            host = torch.frombuffer(bytearray(d), dtype=torch.uint8)
            assert p._lib.jt_b200_input_buffer(p._h, n)
            assert p._lib.jt_b200_copy_in_range(p._h, host.data_ptr(), lo, hi - lo) == 0
            SH.set_resident(p, lo, hi)
            name, off = SH.run_shard(p, n, rank, world, ex)
            part = SH.download(p) if name == "OK" else None
            if part is not None:
                part = (part[0], part[1].tobytes(), part[2], part[3])
            gathered = [None] * world
            dist.all_gather_object(gathered, (name, off, part))
            out.append(gathered)
        if rank == 0:
            q.put(("ok", out))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # report, do not hang the parent
        import traceback
        q.put(("err", f"rank {rank}: {e!r}\n{traceback.format_exc()}"))


def _run(world, docs):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, docs, q)) for r in range(world)]
    for p in ps:
        p.start()
    kind, res = q.get(timeout=600)
    for p in ps:
        p.join(timeout=120)
    assert kind == "ok", res
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_shards(oracle, world):
    from tools.gen import generate
    docs = [generate(1, 3 << 20, seed=41), generate(4, 2 << 20, seed=42), generate(2, 1 << 20, seed=43),
            generate(4, 1 << 20, seed=44, err=3), generate(0, 1 << 20, seed=45)]
    res = _run(world, docs)
    for d, gathered in zip(docs, res):
        r = oracle.parse(d)
        for name, off, _ in gathered:  # every rank reports the document's result
            assert (name, off) == (r.name, r.offset), (world, len(d), name, off, r.name, r.offset)
        if r.code == 0:
            parts = [g[2] for g in gathered]
            at = 0
            for t0, t, _, _ in parts:
                assert t0 == at
                at += len(t) // 8
            tape = np.frombuffer(b"".join(t for _, t, _, _ in parts), dtype=np.uint64)
            assert np.array_equal(tape, r.tape_array())
            assert b"".join(s for _, _, _, s in parts) == r.strings


def _long_number_doc(world):
    """A document whose ~100 KB number starts 50 bytes before the cut after
    shard 0 and ends past that shard's 64 KiB halo."""
    from paper_1902_08318_b200 import shard as SH
    n = 400_000
    cut = SH.layout(n, world)[0][1]
    head = b"[" + b" " * (cut - 50 - 1 - 5) + b"1, 0."
    num = b"0" * 100_000 + b"1"
    body = head + num + b", 2"
    tail = b", 3" * ((n - len(body) - 1) // 3)
    d = body + tail + b" " * (n - len(body) - len(tail) - 1) + b"]"
    assert len(d) == n and d.index(b"0.") < cut < d.index(b"0.") + len(num) - (64 << 10)
    return d


@pytest.mark.parametrize("world", [2])
def test_multirank_number_longer_than_halo(oracle, world):
    """A number crossing the shard cut by more than the resident halo: the
    shard holding its start fails loudly (CAPACITY, -1) rather than reading
    bytes its GPU does not have; with a halo that covers it the parse equals
    the reference's (reference: numbers.cpp accepts unbounded digit runs)."""
    d = _long_number_doc(world)
    r = oracle.parse(d)
    assert r.code == 0
    res = _run(world, [(d, 64 << 10), (d, 256 << 10)])
    for name, off, _ in res[0]:
        assert (name, off) == ("CAPACITY", -1)
    for name, off, _ in res[1]:
        assert (name, off) == (r.name, r.offset)
    tape = np.frombuffer(b"".join(g[2][1] for g in res[1]), dtype=np.uint64)
    assert np.array_equal(tape, r.tape_array())


def _records_rank(rank, world, port, data, q):
    """bench.py run_records at N > 1 on the one GPU: rank g parses its
    record-boundary slice in one record-mode pass, numbers its records from
    an all_gather of the counts, and sends its per-record results to rank 0."""
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import bench
        from paper_1902_08318_b200 import Parser
        b, e = bench.record_ranges(data, world)[rank]
        mine = data[b:e]
        p = Parser()
        host = torch.frombuffer(bytearray(mine), dtype=torch.uint8) if mine else torch.zeros(1, dtype=torch.uint8)
        p.copy_in(host.data_ptr(), len(mine))
        got = p.parse_records(len(mine))
        first, total = bench.record_numbering(dist, world, rank, len(got))
        rows = [(g[0], g[1], None if g[2] is None else g[2].tobytes(), g[3]) for g in got]
        gathered = [None] * world
        dist.all_gather_object(gathered, (first, total, rows))
        if rank == 0:
            q.put(("ok", gathered))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:
        import traceback
        q.put(("err", f"rank {rank}: {ex!r}\n{traceback.format_exc()}"))


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_records(oracle, world):
    """C3 split across ranks (each its own parser and records): every record
    equals jt_parse(record) (oracle), global numbering contiguous."""
    import multiprocessing as mp
    from tools.gen import generate
    data = generate(3, 2 << 20, seed=11)
    mid = data.index(b"\n", len(data) // 3) + 1
    data = data[:mid] + b'{"a":[1,2}\n"\\q"\n\n' + data[mid:]  # failing and empty records
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_records_rank, args=(r, world, port, data, q)) for r in range(world)]
    for p in ps:
        p.start()
    kind, res = q.get(timeout=600)
    for p in ps:
        p.join(timeout=120)
    assert kind == "ok", res
    recs = data.split(b"\n")
    if data.endswith(b"\n"):
        recs = recs[:-1]
    rows = []
    for first, total, rr in res:
        assert first == len(rows) and total == len(recs)
        rows += rr
    assert len(rows) == len(recs)
    for k, (rec, g) in enumerate(zip(recs, rows)):
        o = oracle.parse(rec)
        assert (g[0], g[1]) == (o.name, o.offset), (k, rec[:80])
        if o.code == 0:
            assert np.frombuffer(g[2], dtype=np.uint64).tolist() == o.tape_array().tolist(), k
            assert g[3] == o.strings, k
