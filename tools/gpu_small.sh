#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/small
mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_tc.py -q -x --timeout 200 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout -s KILL 300 python bench.py --workload c1 --steps 20 --warmup 5 --e2e-steps 3 > $O/bench_c1.json 2> $O/bench_c1.err
timeout -s KILL 300 python bench.py --workload c1 --precision fp32 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > $O/bench_c1_fp32.json 2> $O/bench_c1_fp32.err
