"""N>1 path of bench.py on CPU: world_size-2 gloo process group, the same
reduction helpers the GPU run uses (replicas, max-over-ranks timing)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r pretends its timed region took 10*(r+1) ms
    mx = bench.max_over_ranks(10.0 * (rank + 1), dist)
    gbs = bench.job_throughput(64 << 20, 5, world, mx)
    q.put((rank, mx, gbs))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, gbs in res:
        assert mx == 20.0  # every rank sees the slowest rank's time
        assert gbs == pytest.approx(2 * (64 << 20) * 5 / 0.020 / 1e9)


def test_single_process_identity():
    import bench
    assert bench.max_over_ranks(3.5) == 3.5


def _shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_1902_08318_b200 import shard as SH
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ex = SH.nccl_exchange(dist, world)
    out = []
    for phase, nb in enumerate((16, 80, 16400, 32800)):  # Sum0..Sum3 sizes (shard.h)
        local = torch.full((nb,), rank + 1 + 10 * phase, dtype=torch.uint8)
        local[0] = rank
        g = ex(phase, local)
        out.append([(int(g[k * nb]), int(g[k * nb + 1])) for k in range(world)])
    q.put((rank, out, SH.layout(5 * SH.TILE + 123, world)))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_exchange_gloo():
    """bench.py --gpus N shards one document; every phase all-gathers a fixed
    size summary that must arrive in rank order on every rank (the shard
    bases are prefix sums over it)."""
    world, port = 3, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    layouts = {tuple(r[2]) for r in res}
    assert len(layouts) == 1  # every rank derives the same byte ranges
    for rank, out, _ in res:
        for phase, slots in enumerate(out):
            assert slots == [(k, k + 1 + 10 * phase) for k in range(world)]


def test_shard_summary_sizes():
    """the sizes the gloo test assumes are the library's (shard.h)"""
    from paper_1902_08318_b200 import shard as SH
    assert [SH.summary_bytes(k) for k in range(4)] == [16, 80, 16400, 32800]


def test_shard_layout_cpu():
    from paper_1902_08318_b200.shard import TILE, layout
    for n, G in [(TILE, 1), (5 * TILE + 7, 3), (64 * TILE, 8), (100 * TILE - 1, 7)]:
        lo = layout(n, G)
        assert lo[0][0] == 0 and lo[-1][1] == n
        assert all(b % TILE == 0 and b < e for b, e in lo)
        assert all(lo[k][1] == lo[k + 1][0] for k in range(G - 1))
    with pytest.raises(ValueError):
        layout(TILE, 2)


def test_record_ranges():
    """C3 across ranks: cuts fall right after a '\\n', cover the buffer, and
    every record lands on exactly one rank"""
    import bench
    data = b"\n".join(b"[%d]" % k * (k % 7 + 1) for k in range(5000)) + b"\n"
    for world in (1, 2, 3, 8):
        rr = bench.record_ranges(data, world)
        assert rr[0][0] == 0 and rr[-1][1] == len(data)
        assert all(rr[k][1] == rr[k + 1][0] for k in range(world - 1))
        assert all(b == 0 or data[b - 1:b] == b"\n" for b, _ in rr)
        assert sum(data[b:e].count(b"\n") for b, e in rr) == data.count(b"\n")


def _records_worker(rank, world, port, data, q):
    """bench.py run_records' host logic: the record-boundary split and the
    global numbering; each rank parses its records with the oracle standing
    in for jt_b200_parse_records (one jt_parse per record)."""
    import torch.distributed as dist
    import bench
    from oracle.pyoracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = bench.record_ranges(data, world)[rank]
    recs = data[b:e].split(b"\n")
    if data[b:e].endswith(b"\n"):
        recs = recs[:-1]  # a trailing newline ends the last record
    o = Oracle()
    res = [(o.parse(r).code, o.parse(r).offset) for r in recs]
    first, total = bench.record_numbering(dist, world, rank, len(res))
    q.put((rank, b, e, first, total, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_record_split_gloo(world):
    """C3 at N > 1 (bench.py run_records): ranks cut the NDJSON buffer after
    the first newline at each g/N point and number their records from an
    all_gather of the counts.  Every record lands on exactly one rank, in
    order, and the per-record results equal jt_parse(record) over the whole
    buffer; also a cut point that falls on a newline, and a last record
    without a trailing newline."""
    from tools.gen import generate
    data = generate(3, 256 << 10, seed=7)
    mid = data.index(b"\n", len(data) // 2) + 1
    data = data[:mid] + b"\n" + data[mid:]  # an empty record mid-buffer
    data = data.rstrip(b"\n")  # last record unterminated
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_records_worker, args=(r, world, port, data, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle.pyoracle import Oracle
    o = Oracle()
    want = [(o.parse(r).code, o.parse(r).offset) for r in data.split(b"\n")]
    got = []
    at = 0
    for rank, b, e, first, total, rr in res:
        assert b == (res[rank - 1][2] if rank else 0) and first == len(got) and total == len(want)
        got += rr
        at = e
    assert at == len(data)
    assert got == want
    assert any(c == 7 for c, _ in want)  # the empty record: EMPTY
