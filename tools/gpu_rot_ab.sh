cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stack.py -q -x --timeout 300 > gpurun_out/rot_tests.log 2>&1; tail -1 gpurun_out/rot_tests.log
bash tools/gpu_ab_lib.sh "tools/variants/norot.so tools/variants/rot.so" "c5" "auto"
cp gpurun_out/ab_lib/summary.txt gpurun_out/rot_c5.txt
bash tools/gpu_ab_lib.sh "tools/variants/norot.so tools/variants/rot.so" "c3" "fp32"
