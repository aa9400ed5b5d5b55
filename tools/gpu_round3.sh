#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 ./tools/l2_microbench > gpurun_out/l2_microbench.jsonl 2>&1; echo "rc=$?" >> gpurun_out/l2_microbench.jsonl
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
