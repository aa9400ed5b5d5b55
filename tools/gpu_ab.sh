#!/bin/bash
# A/B an env switch on the C3/C4 kernels: gpu_ab.sh VAR "v1 v2" [workloads] [precisions]
cd "${GRAFT_REPO_ROOT:-.}"
VAR=$1; VALS=$2; WLS=${3:-c3}; PRECS=${4:-"auto bf16"}
O=gpurun_out/ab_$VAR
mkdir -p $O
: > $O/summary.txt
for rep in 1 2 3; do for w in $WLS; do for p in $PRECS; do for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-cudnn \
    --precision $p --e2e-steps 1 > $O/b.json 2> $O/b.err
  python -c "import json,sys; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$rep $w $p $VAR=$v kernel_ms=%s step_ms=%.4f layers=%s' % (d['roofline'].get('kernel_ms'), d['ms_per_step'], d.get('layer_ms')))" >> $O/summary.txt 2>&1
done; done; done; done
