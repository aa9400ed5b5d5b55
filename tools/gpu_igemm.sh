#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/igemm; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_igemm.py -q -x --timeout 300 > $O/pytest_igemm.log 2>&1; echo "rc=$?" >> $O/pytest_igemm.log
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_stack.py tests/test_gpu_backward.py -q --timeout 300 > $O/pytest_rest.log 2>&1; echo "rc=$?" >> $O/pytest_rest.log
bash tools/gpu_ab.sh RC_TC_IGEMM "0 1" "c5 c1" auto
cp gpurun_out/ab_RC_TC_IGEMM/summary.txt $O/ab.txt
