#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench lines (all precisions), ncu launch list
# and one full ncu capture of the tensor-core kernel.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r1full
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for p in bf16x3 bf16 fp32; do
  timeout 600 python bench.py --steps 20 --warmup 5 --precision $p --no-cpu-baseline > $O/bench_c3_$p.json 2> $O/bench_c3_$p.err
done
timeout 900 python bench.py --steps 10 --warmup 3 --precision fp32 --workload c4 --no-cpu-baseline > $O/bench_c4_fp32.json 2> $O/bench_c4_fp32.err
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bf16x3.csv \
  python bench.py --steps 2 --warmup 3 --precision bf16x3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ri_tc_kernel -s 3 -c 1 -o $O/tc_bf16x3 \
  python bench.py --steps 1 --warmup 3 --precision bf16x3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_full.log 2>&1
echo done > $O/DONE
