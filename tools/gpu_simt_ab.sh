cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stack.py tests/test_gpu_backward.py -q -x --timeout 300 > gpurun_out/simt_f2_tests.log 2>&1; echo rc=$? >> gpurun_out/simt_f2_tests.log
O=gpurun_out/ab_simt; mkdir -p $O; : > $O/summary.txt
for rep in 1 2; do for l in scalar f2; do
 RC_LIB_VARIANT=$PWD/tools/variants/$l.so timeout 300 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline --no-cudnn --e2e-steps 1 > $O/b.json 2>$O/b.err
 python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$rep c5 $l', d['ms_per_step'], d['layer_ms'])" >> $O/summary.txt
 RC_LIB_VARIANT=$PWD/tools/variants/$l.so timeout 300 python bench.py --workload c3 --precision fp32 --steps 5 --warmup 3 --no-cpu-baseline --no-cudnn --e2e-steps 1 > $O/b.json 2>$O/b.err
 python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$rep c3fp32 $l', d['ms_per_step'])" >> $O/summary.txt
done; done
