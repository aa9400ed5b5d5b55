# new GPU tests (FD verifier, bench_cli) and the C2 grid bench line
timeout 900 python -m pytest tests/test_fd_verifier.py tests/test_gpu_bench_cli.py -x -q > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_new.log
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"; tail -3 gpurun_out/bench_c2.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_c2.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value","ms_per_step","e2e","clocks","gpu_launches")})
print(d["roofline"]); print("wins", d["cells_vs_cudnn"]["cells_at_or_above_cudnn_fp32"], "of", len(d["cells_vs_cudnn"]["rows"]))
for r in d["cells_vs_cudnn"]["rows"]: print(r)
PY
