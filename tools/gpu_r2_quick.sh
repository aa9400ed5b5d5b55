# quick loop: TC tests (hang-guarded), C3 bench (auto), profile variants
set -x
timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_shipped_default.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_tc.log
for w in ${WL:-c3}; do
timeout 120 python bench.py --workload $w --precision auto --steps 10 --warmup 3 --no-cpu-baseline --no-cudnn --no-backward --e2e-steps 1 > gpurun_out/bench_${w}_auto.json 2> gpurun_out/bench_${w}_auto.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_${w}_auto.json").read().strip().splitlines()[-1])
r=d["roofline"]
print("$w auto", d.get("kernel"), "step_ms", round(d["ms_per_step"],4), "kernel_ms", round(r["kernel_ms"],4), "frac", round(r["frac"],4), d.get("clocks"), "match", d.get("timed_output_matches_e2e"))
PY
done
for v in ${VARIANTS:-}; do
timeout 120 python tools/tc_kernel_profile.py run --lib $v 256 256 16 16 1024 steer 8 subgroup 4 auto
done
