set -x
timeout 600 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -3 gpurun_out/pytest_dist.log
# bench under torchrun with 2 ranks on the one GPU (NCCL needs distinct GPUs: expect failure) -> skip
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -12 gpurun_out/sanitize_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -12 gpurun_out/sanitize_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -6 gpurun_out/sanitize_synccheck.log
