#!/bin/bash
# SIMT occupancy A/B: library built with __launch_bounds__(256, MINB) x RC_SIMT_SW
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/simt_occ; mkdir -p $O; : > $O/summary.txt
for rep in 1 2; do for cfg in "minb1 8" "minb2 4" "minb1 4"; do set -- $cfg
  RC_LIB_VARIANT=$PWD/tools/variants/$1.so RC_SIMT_SW=$2 timeout 300 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$rep c5 $1 sw=$2', round(d['ms_per_step'],3), d['layer_ms'])" >> $O/summary.txt
  RC_LIB_VARIANT=$PWD/tools/variants/$1.so RC_SIMT_SW=$2 timeout 300 python bench.py --workload c3 --precision fp32 --steps 5 --warmup 3 --no-cpu-baseline --no-cudnn --no-backward --e2e-steps 1 > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$rep c3fp32 $1 sw=$2', round(d['ms_per_step'],3))" >> $O/summary.txt
done; done
