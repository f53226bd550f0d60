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
        for d in docs:
            n = len(d)
            begin, end = SH.layout(n, world)[rank]
            lo, hi = max(0, begin - 64), min(n, end + (64 << 10))
            host = torch.frombuffer(bytearray(d), dtype=torch.uint8)
            assert p._lib.jt_b200_input_buffer(p._h, n)
            assert p._lib.jt_b200_copy_in_range(p._h, host.data_ptr(), lo, hi - lo) == 0
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
