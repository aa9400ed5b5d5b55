#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/cpp
mkdir -p $O
timeout 600 ./tests/cpp/test_cpp_api --gpu > $O/cpp_gpu.log 2>&1; echo "rc=$?" >> $O/cpp_gpu.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
