#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/pair
mkdir -p $O
timeout -s KILL 300 python - > $O/smoke_pair.log 2>&1 <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, "oracle")
import oracle as O, paper_2512_08888_b200 as P
rng = np.random.default_rng(0)
for (n, cin, h, cout, g, R, pool, pg) in [(1, 64, 16, 256, "p4", 4, "none", 4), (2, 128, 16, 256, "p4m", 8, "subgroup", 4)]:
    x = (rng.integers(-4, 5, (n, cin, h, 16)) / 4).astype(np.float32)
    w = (rng.integers(-4, 5, (cout, cin, 3, 3)) / 4).astype(np.float32)
    d = O.Desc(n, cin, h, 16, cout, 3, g, R, pool, pg)
    yr, ar = O.ri_forward(d, x, w)
    desc = P.Desc(n, cin, h, 16, cout, 3, g, R, pool, pg, "scatter", "bf16x3")
    bank = P.bank_precompute(desc, torch.from_numpy(w).cuda())
    y, a = P.ri_conv_forward(desc, torch.from_numpy(x).cuda(), bank)
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    print(n, cin, cout, g, "equal", np.array_equal(y.reshape(yr.shape), yr), "maxdiff", np.abs(y.reshape(yr.shape) - yr).max(), flush=True)
PY
echo "rc=$?" >> $O/smoke_pair.log
timeout -s KILL 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_stack.py -q -x --timeout 200 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in 1 0; do
RC_TC_PAIR=$v timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/bench_c3_pair$v.json 2> $O/bench_c3_pair$v.err
RC_TC_PAIR=$v timeout -s KILL 300 python bench.py --precision bf16 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/bench_c3_bf16_pair$v.json 2> $O/bench_c3_bf16_pair$v.err
done
