# A/B of the band kernel: tests of the tensor-core path, then C3 / C4 benches (kernel ms)
set -x
timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_shipped_default.py tests/test_gpu_stack.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_tc.log
for w in ${WL:-c3 c4}; do
  for pr in ${PR:-auto bf16}; do
    timeout 120 python bench.py --workload $w --precision $pr --steps 10 --warmup 3 --no-cpu-baseline --no-cudnn --no-backward --e2e-steps 1 > gpurun_out/bench_${w}_${pr}.json 2> gpurun_out/bench_${w}_${pr}.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/bench_${w}_${pr}.json").read().strip().splitlines()[-1])
r=d["roofline"]
print("$w $pr", d.get("kernel"), "step_ms", round(d["ms_per_step"],4), "kernel_ms", round(r["kernel_ms"],4), "frac", round(r["frac"],4), d.get("clocks"))
PY
  done
done
