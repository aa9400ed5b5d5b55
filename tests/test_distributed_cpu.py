"""World-size-2/4 gloo test of the batch-sharded driver's host logic (shard ranges +
ragged output gather).  The per-shard compute is the CPU oracle (test infrastructure);
on the GPU box the same gather runs over NCCL (bench.py --gpus N)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_2512_08888_b200 import distributed as D
        from paper_2512_08888_b200.rotconv import Desc
        rng = np.random.default_rng(77)  # identical inputs on every rank (seeded host init)
        x = (rng.integers(-4, 5, (n, 3, 8, 8)) / 4).astype(np.float32)
        fx = (rng.integers(-4, 5, (5, 3, 3, 3)) / 4).astype(np.float32)
        fy = (rng.integers(-4, 5, (5, 3, 3, 3)) / 4).astype(np.float32)
        gdesc = Desc(n, 3, 8, 8, 5, 3, "steer", 8, "subgroup", 4)
        ld, b, e = D.local_desc(gdesc, world, rank)
        od = O.Desc(ld.n, 3, 8, 8, 5, 3, "steer", 8, "subgroup", 4)
        y_loc, a_loc = O.ri_forward(od, x[b:e], fx, fy)
        y = D.gather_shards(torch.from_numpy(y_loc), n)
        a = D.gather_shards(torch.from_numpy(a_loc), n, to_all=False)
        if rank == 0:
            y_full, a_full = O.ri_forward(O.Desc(n, 3, 8, 8, 5, 3, "steer", 8, "subgroup", 4), x, fx, fy)
            q.put((np.array_equal(y.numpy(), y_full), np.array_equal(a.numpy(), a_full), (b, e)))
        else:
            q.put((a is None, True, (b, e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 6), (2, 5), (4, 6)])  # even, ragged, and a 4-rank split
def test_rank_shard_and_gather(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[0] and r[1] for r in res), res
    spans = sorted(r[2] for r in res)
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))  # contiguous cover
    assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1   # balanced
