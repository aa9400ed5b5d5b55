#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
RC_LIB_VARIANT=$PWD/tools/variants/cat.so timeout 900 python -m pytest tests/test_gpu_tc.py -q -x --timeout 300 > gpurun_out/cat_tests.log 2>&1; tail -1 gpurun_out/cat_tests.log
bash tools/gpu_ab_lib.sh "tools/variants/nocat.so tools/variants/cat.so" "c3" "auto bf16"
