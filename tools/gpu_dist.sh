#!/bin/bash
# torchrun code path on the single GPU the pool gives us (world size 1, NCCL backend),
# plus the sharded driver + NCCL gather helper
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/dist
mkdir -p $O
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/torchrun_c3.json 2> $O/torchrun_c3.err
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --impl reference --steps 1 --warmup 0 > $O/torchrun_ref.json 2> $O/torchrun_ref.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 - > $O/gather.log 2>&1 <<'PY'
import os, torch, torch.distributed as dist
import paper_2512_08888_b200 as P
from paper_2512_08888_b200 import distributed as D
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
desc = P.Desc(6, 16, 16, 16, 128, 3, "steer", 8, "subgroup", 4, "scatter", "auto")
g = torch.Generator(device="cuda").manual_seed(0)
fx = torch.rand((128, 16, 3, 3), generator=g, device="cuda"); fy = torch.rand_like(fx)
x = torch.rand((6, 16, 16, 16), generator=g, device="cuda")
y, a = D.sharded_forward(desc, x, fx, fy)
full = D.gather_shards(y, 6)
bank = P.bank_precompute(desc, fx, fy)
ref, _ = P.ri_conv_forward(desc, x, bank)
print("gather ok", torch.equal(full, ref), full.shape)
dist.destroy_process_group()
PY
