#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/ablc4
mkdir -p $O
for w in c4 c3; do for a in 0 5 2 4; do
RC_TC_ABLATE=$a timeout -s KILL 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w ablate=$a', r['kernel'], round(r['kernel_ms'],3))" >> $O/res.txt
done; done
