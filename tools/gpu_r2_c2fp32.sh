# C2 grid with precision fp32 (direct FP32 kernel up to Cin = 32 on small images) vs auto
for pr in fp32; do
timeout 600 python bench.py --workload c2 --precision $pr --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c2_$pr.json 2> gpurun_out/bench_c2_$pr.err; echo "c2 $pr rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_c2_$pr.json").read().strip().splitlines()[-1])
for r in d["cells_vs_cudnn"]["rows"]:
    if 8 < r[1] <= 32: print(r)
PY
done
