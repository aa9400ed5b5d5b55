#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/pair3
mkdir -p $O
for v in 1 0; do for a in 0 4 5 2; do
RC_TC_PAIR=$v RC_TC_ABLATE=$a timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('pair=$v ablate=$a', round(r['kernel_ms'],3))" >> $O/res.txt
done; done
