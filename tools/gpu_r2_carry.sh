# carry-band kernel: a quick tensor-core case first (hang guard), the TC tests, then C3 bench
set -x
timeout 90 python -m pytest "tests/test_gpu_tc.py::test_tc_dyadic_bitexact" -x -q -k "2-64-16-128-p4-4-subgroup-4-scatter" > gpurun_out/pytest_quick.log 2>&1; rc=$?; echo "quick rc=$rc"; tail -5 gpurun_out/pytest_quick.log
[ $rc -eq 124 ] && exit 1
timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_shipped_default.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_tc.log
for pr in auto bf16; do
  timeout 120 python bench.py --workload c3 --precision $pr --steps 10 --warmup 3 --no-cpu-baseline --no-cudnn --no-backward --e2e-steps 1 > gpurun_out/bench_c3_${pr}.json 2> gpurun_out/bench_c3_${pr}.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c3_${pr}.json").read().strip().splitlines()[-1])
r=d["roofline"]
print("c3 ${pr}", d.get("kernel"), "step_ms", round(d["ms_per_step"],4), "kernel_ms", round(r["kernel_ms"],4), "frac", round(r["frac"],4), d.get("clocks"), "match", d.get("timed_output_matches_e2e"))
PY
done
