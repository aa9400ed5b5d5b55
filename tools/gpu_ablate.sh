#!/bin/bash
# C3 main-kernel time per RC_TC_ABLATE mode (see TcParams::ablate); LIBS = library builds to compare
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/ablate; mkdir -p $O; : > $O/summary.txt
for l in ${LIBS:-paper_2512_08888_b200/librotconv_b200.so}; do
for p in ${PRECS:-auto bf16}; do for a in ${MODES:-0 6 7 8 9}; do
  RC_LIB_VARIANT=$PWD/$l RC_TC_ABLATE=$a timeout 300 python bench.py --workload ${WL:-c3} --steps 10 --warmup 3 \
    --no-cpu-baseline --no-cudnn --precision $p --e2e-steps 1 > $O/b.json 2> $O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$l $p ablate=$a kernel_ms=%.4f' % d['roofline']['kernel_ms'])" >> $O/summary.txt 2>&1
done; done; done
