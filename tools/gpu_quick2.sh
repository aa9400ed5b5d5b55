#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/quick2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_stack.py -q -x --timeout 300 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/bench_c3.json 2> $O/bench_c3.err
