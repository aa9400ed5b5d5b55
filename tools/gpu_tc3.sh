#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x --timeout 120 > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
for p in bf16 bf16x3; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --precision $p --e2e-steps 1 > gpurun_out/bench_$p.json 2> gpurun_out/bench_$p.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ri_tc_kernel -s 1 -c 1 -o gpurun_out/prof_tc_bf16_v7 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --precision bf16 --e2e-steps 0 > gpurun_out/ncu_tc_bf16.log 2>&1
echo done
