#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 120 python - > gpurun_out/tc_quick.log 2>&1 <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import oracle as O, paper_2512_08888_b200 as P
dev = torch.device('cuda:0')
rng = np.random.default_rng(0)
for prec in ('bf16', 'bf16x3'):
    n, cin, h, cout = 1, 64, 16, 128
    x = (rng.integers(-4, 5, (n, cin, h, 16)) / 4).astype(np.float32)
    w = (rng.integers(-4, 5, (cout, cin, 3, 3)) / 4).astype(np.float32)
    d = O.Desc(n, cin, h, 16, cout, 3, 'p4', 4, 'none', 4)
    yr, _ = O.ri_forward(d, x, w)
    pd = P.Desc(n, cin, h, 16, cout, 3, 'p4', 4, 'none', 4, 'scatter', prec)
    print(prec, pd.kernel_name(), pd.workspace_bytes(), flush=True)
    bank = P.bank_precompute(pd, torch.from_numpy(w).to(dev))
    y, _ = P.ri_conv_forward(pd, torch.from_numpy(x).to(dev), bank)
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    print(prec, 'equal', np.array_equal(y, yr), 'maxdiff', np.abs(y - yr).max(), flush=True)
    bad = np.argwhere(y != yr)
    print('first bad', bad[:10].tolist(), flush=True)
    if len(bad):
        i = tuple(bad[0]); print('got', y[i], 'want', yr[i])
PY
echo "quick rc=$?" >> gpurun_out/tc_quick.log
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x --timeout 120 > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --precision bf16x3 --e2e-steps 1 > gpurun_out/bench_bf16x3.json 2> gpurun_out/bench_bf16x3.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --precision bf16 --e2e-steps 1 > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
echo done
