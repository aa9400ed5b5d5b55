#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/pair2
mkdir -p $O
for v in 1 0; do for st in 2 4 6; do for p in auto bf16; do
RC_TC_PAIR=$v RC_TC_MIN_STAGES=$st timeout -s KILL 300 python bench.py --precision $p --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('pair=$v stages=$st $p', round(r['kernel_ms'],3), round(d['ms_per_step'],3))" >> $O/res.txt
done; done; done
