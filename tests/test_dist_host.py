"""Host side of the multi-GPU path, on CPU with gloo (world_size 2).

The NCCL data path needs one GPU per rank; here we check what can be checked
without GPUs: the shard / batch-split rules cover every row exactly once, and
the NCCL unique id rank 0 creates reaches every rank intact over
torch.distributed (the bootstrap the sharded solve uses).
"""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2605_00837_b200 import dist as D


def test_shard_bounds_partition():
    for n in (1, 7, 64, 1000, 65536):
        for P in (1, 2, 3, 4, 8):
            if P > n:
                continue
            spans = [D.shard_bounds(n, P, r) for r in range(P)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_split_batch_c5():
    spans = [D.split_batch(256, 8, r) for r in range(8)]
    assert all(hi - lo == 32 for lo, hi in spans)


def test_bad_rank():
    with pytest.raises(ValueError):
        D.shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = D.broadcast_unique_id()
        q.put((rank, uid))
    finally:
        dist.destroy_process_group()


def test_unique_id_broadcast_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got[0]) == 128 and got[0] == got[1] and any(got[0])
