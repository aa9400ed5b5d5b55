#!/bin/bash
# same-box A/B of library builds: gpu_ab_lib.sh "libA.so libB.so" [workloads] [precisions]
cd "${GRAFT_REPO_ROOT:-.}"
LIBS=$1; WLS=${2:-c3}; PRECS=${3:-"auto bf16"}
O=gpurun_out/ab_lib; mkdir -p $O; : > $O/summary.txt
for rep in 1 2 3; do for w in $WLS; do for p in $PRECS; do for l in $LIBS; do
  RC_LIB_VARIANT=$PWD/$l timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-cudnn \
    --precision $p --e2e-steps 1 > $O/b.json 2> $O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$rep $w $p $l kernel_ms=%s step_ms=%.4f layers=%s' % (d['roofline'].get('kernel_ms'), d['ms_per_step'], d.get('layer_ms')))" >> $O/summary.txt 2>&1
done; done; done; done
