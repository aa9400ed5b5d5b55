# implicit-GEMM tests + C2 grid after the small-layer N-tile change
timeout 600 python -m pytest tests/test_gpu_igemm.py tests/test_gpu_shipped_default.py tests/test_gpu_backward.py -x -q > gpurun_out/pytest_ig.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ig.log; grep -E "^E  |FAILED" gpurun_out/pytest_ig.log | head -5
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_auto.json 2> gpurun_out/bench_c2_auto.err; echo "c2 rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c2_auto.json").read().strip().splitlines()[-1])
print("value", round(d["value"],2), "ms", round(d["ms_per_step"],4), "wins", d["cells_vs_cudnn"]["cells_at_or_above_cudnn_fp32"])
for r in d["cells_vs_cudnn"]["rows"]:
    if r[0] == 16 or r[7] < 1: print(r)
PY
