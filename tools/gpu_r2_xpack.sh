# tests + C3 / C4 bench step vs kernel time (x_pack via cp.async)
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_carry.py tests/test_gpu_shipped_default.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_tc.log
for w in c3 c4; do
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-cudnn --no-backward --e2e-steps 1 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$w.json").read().strip().splitlines()[-1])
r=d["roofline"]; print("$w step", round(d["ms_per_step"],4), "kernel", round(r["kernel_ms"],4), "frac", round(r["frac"],4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:x_pack python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-cudnn --no-backward --e2e-steps 1 2>/dev/null | grep x_pack | tail -2 | cut -c1-300
