"""The batch-sharded driver with the CUDA kernels on >= 2 ranks.

Two (or three) processes share the one leased GPU, each running the product kernels on its
contiguous shard (paper_2512_08888_b200.distributed.sharded_forward); the shards are gathered
over gloo (the on-request gather; NCCL on a multi-GPU node) and must be BIT-IDENTICAL to one
full-batch launch -- values and argmax, ragged splits included.  Every image is computed by
the same kernel code whichever launch or CTA runs it, so sharding cannot change a bit.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_08888_b200 import distributed as D
        from paper_2512_08888_b200.rotconv import Desc, bank_precompute, ri_conv_forward
        n, cin, h, w, cout, g, R, pool, pg = cfg
        dev = torch.device("cuda", 0)
        gen = torch.Generator().manual_seed(2024)  # identical host-side init on every rank
        x = torch.rand((n, cin, h, w), generator=gen) * 2 - 1
        s = 1 / np.sqrt(cin * 9)
        fx = (torch.rand((cout, cin, 3, 3), generator=gen) * 2 - 1) * s
        fy = (torch.rand((cout, cin, 3, 3), generator=gen) * 2 - 1) * s
        bias = torch.rand(cout, generator=gen) * 0.2 - 0.1
        gdesc = Desc(n, cin, h, w, cout, 3, g, R, pool, pg)  # precision auto: the tcgen05 kernels
        ld, b, e = D.local_desc(gdesc, world, rank)
        y_loc, a_loc = D.sharded_forward(gdesc, x[b:e].contiguous().to(dev), fx.to(dev), fy.to(dev),
                                         bias.to(dev), world=world, rank=rank)
        torch.cuda.synchronize()
        y = D.gather_shards(y_loc.cpu(), n, to_all=False)
        a = D.gather_shards(a_loc.cpu(), n, to_all=False) if a_loc is not None else None
        if rank == 0:
            bank = bank_precompute(gdesc, fx.to(dev), fy.to(dev))
            y_full, a_full = ri_conv_forward(gdesc, x.to(dev), bank, bias.to(dev))
            ok_y = torch.equal(y, y_full.cpu())
            ok_a = a is None or torch.equal(a, a_full.cpu())
            q.put((ok_y, ok_a, (b, e), gdesc.kernel_name()))
        else:
            q.put((y is None, True, (b, e), ld.kernel_name()))
    finally:
        dist.destroy_process_group()


CASES = [
    # (world, (n, cin, h, w, cout, group, R, pool, g))
    (2, (64, 64, 16, 16, 256, "steer", 8, "subgroup", 4)),   # the C3 layer type, even split
    (2, (37, 32, 32, 32, 128, "steer", 16, "subgroup", 4)),  # the C4 layer type, ragged split
    (3, (10, 16, 8, 8, 128, "p4m", 8, "max", 8)),            # 3 ranks, ragged, small images
]


@pytest.mark.parametrize("world,cfg", CASES, ids=lambda c: "-".join(map(str, c)) if isinstance(c, tuple) else str(c))
def test_sharded_cuda_forward_equals_full_batch(world, cfg):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(r[0] and r[1] for r in res), res
    assert all(r[3].startswith("tc_") for r in res), res  # the tensor-core kernels ran on every rank
    spans = sorted(r[2] for r in res)
    assert spans[0][0] == 0 and spans[-1][1] == cfg[0]
    assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))
