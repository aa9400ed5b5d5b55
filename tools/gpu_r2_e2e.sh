# e2e (C-ABI host path) of C3 / C4 with 16 pipeline chunks, plus the C++ / distributed tests that use it
timeout 600 python -m pytest tests/test_cpp_api.py tests/test_gpu_distributed.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_e2e.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_e2e.log
for w in c3 c4; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-cpu-baseline --no-cudnn --no-backward --e2e-steps 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$w.json").read().strip().splitlines()[-1])
print("$w e2e", d["e2e"], "match", d["timed_output_matches_e2e"])
PY
done
