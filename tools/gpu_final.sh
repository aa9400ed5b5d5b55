#!/bin/bash
# round-1 evidence pass: tests, smoke, C++ API, bench lines C1/C3/C4/C5 (+fp32/bf16 rows),
# reference arm, C2 sweep, ncu launch lists and full captures of the dominant kernels
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${FINAL_DIR:-final3}
mkdir -p $O/c2
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout -s KILL 600 ./tests/cpp/test_cpp_api --gpu > $O/cpp_gpu.log 2>&1; echo "rc=$?" >> $O/cpp_gpu.log
timeout -s KILL 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout -s KILL 600 python bench.py --precision fp32 --no-cpu-baseline > $O/bench_c3_fp32.json 2> $O/bench_c3_fp32.err
timeout -s KILL 600 python bench.py --precision bf16 --no-cpu-baseline > $O/bench_c3_bf16.json 2> $O/bench_c3_bf16.err
timeout -s KILL 900 python bench.py --workload c4 --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout -s KILL 900 python bench.py --workload c5 --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout -s KILL 300 python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err
timeout -s KILL 1500 python tools/appendix_sweep.py --out $O/c2 > $O/c2/sweep.log 2>&1; echo rc=$? >> $O/c2/sweep.log
timeout -s KILL 1500 python tools/bench_cli.py --sizes 8 16 32 --cin 64 256 --cout 256 1024 --orientations 8 --group steer --batch 32 --out $O/bench_cli_r8.md --format md > $O/bench_cli_r8.log 2>&1; echo rc=$? >> $O/bench_cli_r8.log
NCU=/usr/local/cuda/bin/ncu
for w in c3 c4 c1; do
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_$w.csv \
  python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch_$w.log 2>&1
done
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"simt_k3|igemm|ig_pack|x_pack|ri_tc|maxpool|gap_linear" -c 40 --csv \
  --log-file $O/launches_c5.csv python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch_c5.log 2>&1
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:ri_tc_kernel -s 3 -c 1 -o $O/tc_c3 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_full_c3.log 2>&1
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:ri_tc_kernel -s 3 -c 1 -o $O/tc_c4 \
  python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_full_c4.log 2>&1
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:igemm_kernel -c 1 -o $O/igemm_c5l2 \
  python tools/layer_probe.py 1024 128 64 64 64 single 1 none 1 auto relu 1 > $O/ncu_full_igemm.log 2>&1
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:simt_k3 -c 1 -o $O/simt_c5l1 \
  python tools/layer_probe.py 1024 3 64 64 64 steer 8 subgroup 4 auto relu 1 > $O/ncu_full_simt.log 2>&1
echo done > $O/DONE
