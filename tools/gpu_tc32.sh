#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/tc32
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x --timeout 300 > $O/pytest_tc.log 2>&1; echo "rc=$?" >> $O/pytest_tc.log
for p in bf16x3 bf16; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision $p --e2e-steps 1 > $O/bench_c3_$p.json 2> $O/bench_c3_$p.err
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --precision $p --e2e-steps 1 > $O/bench_c4_$p.json 2> $O/bench_c4_$p.err
done
