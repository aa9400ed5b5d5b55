# carry tests + A/B of timing-only variants on the C3 and C4 shapes
timeout 400 python -m pytest tests/test_gpu_carry.py tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_tc.log
for r in 1 2; do for v in ${VARIANTS}; do
timeout 60 python tools/tc_kernel_profile.py run --lib $v 256 256 16 16 1024 steer 8 subgroup 4 auto
timeout 90 python tools/tc_kernel_profile.py run --lib $v 112 128 32 32 512 steer 16 subgroup 4 auto
done; done
