#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/strip32
mkdir -p $O
RC_TC_STRIP32=1 timeout -s KILL 600 python -m pytest tests/test_gpu_tc.py -q -x --timeout 200 -k "w32" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in 0 1; do for p in auto bf16; do
RC_TC_STRIP32=$v timeout -s KILL 300 python bench.py --workload c4 --precision $p --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('strip32=$v $p', r['kernel'], round(r['kernel_ms'],3))" >> $O/res.txt
done; done
