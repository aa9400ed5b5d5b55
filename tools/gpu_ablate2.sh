#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/abl
mkdir -p $O
for a in 0 1 2 3 4 5; do
  for p in bf16 bf16x3; do
    RC_TC_ABLATE=$a timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision $p --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a $p', round(d['ms_per_step'],3))" >> $O/abl.txt
  done
done
timeout 600 ./tests/cpp/test_cpp_api --gpu > $O/cpp_gpu.log 2>&1; echo "rc=$?" >> $O/cpp_gpu.log
