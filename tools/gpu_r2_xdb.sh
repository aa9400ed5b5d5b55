# double-buffered X bands on carry strips: hang-guarded strip test, TC tests, A/B on C4 and C3
timeout 120 python -m pytest tests/test_gpu_tc.py -x -q -k "strip" > gpurun_out/q.log 2>&1; rc=$?; echo "quick rc=$rc"; tail -2 gpurun_out/q.log; grep -E "^E  " gpurun_out/q.log | head -3; [ $rc -ne 0 ] && exit 1
timeout 500 python -m pytest tests/test_gpu_tc.py tests/test_gpu_carry.py tests/test_gpu_shipped_default.py tests/test_gpu_stack.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_tc.log; grep -E "^E  " gpurun_out/pytest_tc.log | head -3
for r in 1 2; do for v in t_base t_xdb; do
timeout 90 python tools/tc_kernel_profile.py run --lib $v 112 128 32 32 512 steer 16 subgroup 4 auto
done; done
for v in t_base t_xdb; do timeout 60 python tools/tc_kernel_profile.py run --lib $v 256 256 16 16 1024 steer 8 subgroup 4 auto; done
