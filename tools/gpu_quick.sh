#!/bin/bash
# quick perf check: tc tests + C3/C4 bench lines
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/quick
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_stack.py -q -x --timeout 300 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for w in c3 c4; do for p in auto bf16; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --precision $p --e2e-steps 1 > $O/bench_${w}_$p.json 2> $O/bench_${w}_$p.err
done; done
