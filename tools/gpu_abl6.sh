#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/abl6
mkdir -p $O
for w in c3 c4; do for a in 0 6; do for p in auto bf16; do
RC_TC_ABLATE=$a timeout -s KILL 300 python bench.py --workload $w --precision $p --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w $p ablate=$a', r['kernel'], round(r['kernel_ms'],3), d['clocks'])" >> $O/res.txt
done; done; done
