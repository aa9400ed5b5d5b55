timeout 120 python -m pytest tests/test_gpu_tc.py -x -q -k "strip or w32" > gpurun_out/q.log 2>&1; rc=$?; echo "quick rc=$rc"; tail -3 gpurun_out/q.log; [ $rc -eq 124 ] && exit 1
timeout 400 python -m pytest tests/test_gpu_tc.py tests/test_gpu_shipped_default.py tests/test_gpu_stack.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_tc.log
VARIANTS="t_base t_strip" bash tools/gpu_r2_ab2.sh
