# C5 stack bench (layer ms) + stack / parity tests
timeout 400 python -m pytest tests/test_gpu_stack.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_c5.json").read().strip().splitlines()[-1])
print("c5 ms", round(d["ms_per_step"],4), "layers", d["layer_ms"], d["kernels"][0], d["clocks"])
PY
