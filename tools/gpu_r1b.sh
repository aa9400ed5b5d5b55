#!/bin/bash
# round-1 full GPU pass: tests, smoke, C++ API, bench lines for C1/C3/C4/C5, launch lists
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r1b
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c3_default.json 2> $O/bench_c3_default.err
timeout 600 python bench.py --precision fp32 --no-cpu-baseline > $O/bench_c3_fp32.json 2> $O/bench_c3_fp32.err
timeout 600 python bench.py --precision bf16 --no-cpu-baseline > $O/bench_c3_bf16.json 2> $O/bench_c3_bf16.err
timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 300 python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch_c3.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c4.csv \
  python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch_c4.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ri_tc_kernel -s 3 -c 1 -o $O/tc_c4 \
  python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_full_c4.log 2>&1
echo done > $O/DONE
