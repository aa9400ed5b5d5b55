#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
RC_TC_ABLATE=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ri_tc_kernel -s 1 -c 1 -o gpurun_out/prof_tc_abl3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --precision bf16 --e2e-steps 0 > gpurun_out/ncu_abl3.log 2>&1
echo done
