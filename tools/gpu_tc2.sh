#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -q --timeout 120 > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ri_tc_kernel -s 1 -c 1 -o gpurun_out/prof_tc_bf16 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --precision bf16 --e2e-steps 0 > gpurun_out/ncu_tc_bf16.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ri_tc_kernel -s 1 -c 1 -o gpurun_out/prof_tc_bf16x3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --precision bf16x3 --e2e-steps 0 > gpurun_out/ncu_tc_bf16x3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --precision bf16x3 --e2e-steps 1 > /dev/null 2>&1
echo done
