# compute-sanitizer memcheck / racecheck / synccheck of every kernel family (current code)
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/sanitize_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/sanitize_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -4 gpurun_out/sanitize_synccheck.log
