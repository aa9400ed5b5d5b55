# the driver's torchrun launch path at world size 1 (C3 default, C4, C2)
for w in c3 c4 c2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-cudnn --no-backward --e2e-steps 1 > gpurun_out/tr_$w.json 2> gpurun_out/tr_$w.err; echo "$w rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/tr_$w.json").read().strip().splitlines()[-1])
print("$w", d["n_gpus"], d["value"], d["ms_per_step"], d["per_rank_ms"], d["config"].get("parallelism"))
PY
done
