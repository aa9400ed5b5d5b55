#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/simtsw
mkdir -p $O
RC_SIMT_SW=4 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stack.py -q -x --timeout 300 > $O/pytest_sw4.log 2>&1; echo "rc=$?" >> $O/pytest_sw4.log
for sw in 8 4; do
RC_SIMT_SW=$sw timeout -s KILL 300 python bench.py --precision fp32 --steps 5 --warmup 2 --no-cpu-baseline --no-cudnn --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c3 fp32 sw=$sw', r['kernel'], round(r['kernel_ms'],3))" >> $O/res.txt
RC_SIMT_SW=$sw timeout -s KILL 300 python bench.py --workload c4 --precision fp32 --steps 3 --warmup 1 --no-cpu-baseline --no-cudnn --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4 fp32 sw=$sw', r['kernel'], round(r['kernel_ms'],3))" >> $O/res.txt
RC_SIMT_SW=$sw timeout -s KILL 600 python bench.py --workload c5 --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 sw=$sw', round(d['ms_per_step'],3), d['layer_ms'])" >> $O/res.txt
RC_SIMT_SW=$sw timeout -s KILL 300 python bench.py --workload c1 --precision fp32 --steps 10 --warmup 3 --no-cpu-baseline --no-cudnn --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c1 fp32 sw=$sw', r['kernel'], round(r['kernel_ms'],4))" >> $O/res.txt
done
