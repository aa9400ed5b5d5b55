#!/bin/bash
# short evidence pass (no ncu): tests, smoke, C++ API, bench lines
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${FINAL_DIR:-final5}
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout -s KILL 600 ./tests/cpp/test_cpp_api --gpu > $O/cpp_gpu.log 2>&1; echo "rc=$?" >> $O/cpp_gpu.log
timeout -s KILL 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout -s KILL 600 python bench.py --precision bf16 --no-cpu-baseline > $O/bench_c3_bf16.json 2> $O/bench_c3_bf16.err
timeout -s KILL 600 python bench.py --precision fp32 --no-cpu-baseline > $O/bench_c3_fp32.json 2> $O/bench_c3_fp32.err
timeout -s KILL 900 python bench.py --workload c4 --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout -s KILL 900 python bench.py --workload c5 --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout -s KILL 300 python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err
echo done > $O/DONE
