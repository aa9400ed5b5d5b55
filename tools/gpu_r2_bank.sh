# launch times of one bank precompute at the C3 shape (ncu launch list)
cat > gpurun_out/bank_probe.py <<'PY'
import sys; sys.path.insert(0, "."); import torch, paper_2512_08888_b200 as P
d = P.Desc(256, 256, 16, 16, 1024, 3, "steer", 8, "subgroup", 4, "scatter", "auto")
fx = torch.rand((1024, 256, 3, 3), device="cuda"); fy = torch.rand_like(fx)
for _ in range(3): P.bank_precompute(d, fx, fy)
torch.cuda.synchronize()
PY
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python gpurun_out/bank_probe.py > gpurun_out/bank_launches.csv 2>&1; echo "rc=$?"
grep -E "bank|w_pack" gpurun_out/bank_launches.csv | cut -c1-400 | tail -12
