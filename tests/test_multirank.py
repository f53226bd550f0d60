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
