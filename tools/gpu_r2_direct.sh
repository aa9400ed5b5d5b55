# GPU tests, then the C2 grid (auto)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; grep -E "^E|FAILED" gpurun_out/pytest_gpu.log | head
for pr in auto; do
timeout 600 python bench.py --workload c2 --precision $pr --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_$pr.json 2> gpurun_out/bench_c2_$pr.err; echo "c2 $pr rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c2_$pr.json").read().strip().splitlines()[-1])
print("$pr value", round(d["value"],2), "ms", round(d["ms_per_step"],4), "wins", d["cells_vs_cudnn"]["cells_at_or_above_cudnn_fp32"])
for r in d["cells_vs_cudnn"]["rows"]:
    if r[1] <= 8 or r[7] < 1: print(r)
PY
done
