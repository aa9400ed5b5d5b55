# 16 KB hi / lo weight stages on CAT bands: hang-guarded quick test, TC tests, A/B on C3
timeout 120 python -m pytest tests/test_gpu_tc.py -x -q -k "dyadic_bitexact and 2-64-16-128-p4-4-subgroup" > gpurun_out/q.log 2>&1; rc=$?; echo "quick rc=$rc"; tail -2 gpurun_out/q.log; [ $rc -ne 0 ] && exit 1
timeout 400 python -m pytest tests/test_gpu_tc.py tests/test_gpu_carry.py tests/test_gpu_shipped_default.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_tc.log
for r in 1 2; do for v in t_base t_split; do
timeout 60 python tools/tc_kernel_profile.py run --lib $v 256 256 16 16 1024 steer 8 subgroup 4 auto
done; done
