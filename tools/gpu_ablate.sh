#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for a in 0 1 3; do
  for p in bf16 bf16x3; do
    RC_TC_ABLATE=$a timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision $p --e2e-steps 1 > gpurun_out/abl_${a}_$p.json 2>/dev/null
  done
done
echo done
