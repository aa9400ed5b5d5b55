#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/quick3
mkdir -p $O/c2
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 1400 python tools/appendix_sweep.py --out $O/c2 > $O/c2/sweep.log 2>&1; echo rc=$? >> $O/c2/sweep.log
