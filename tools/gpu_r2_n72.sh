# strips with N = 72 (multiple of 8): strip / carry tests (hang-guarded), then A/B on the C4 proxy
timeout 120 python -m pytest tests/test_gpu_tc.py -x -q -k "strip" > gpurun_out/q.log 2>&1; rc=$?; echo "quick rc=$rc"; tail -3 gpurun_out/q.log; grep -E "^E  " gpurun_out/q.log | head -5; [ $rc -ne 0 ] && exit 1
timeout 400 python -m pytest tests/test_gpu_tc.py tests/test_gpu_carry.py tests/test_gpu_shipped_default.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_tc.log
for v in t_base t_n72 t_base t_n72; do timeout 90 python tools/tc_kernel_profile.py run --lib $v 112 128 32 32 512 steer 16 subgroup 4 auto; done
