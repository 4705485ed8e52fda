#!/bin/bash
# round 2 (f): full GPU suite, default bench (c4 fast), c4 exact bench, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/r2f_tests.log
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2f_bench.log
timeout 900 python bench.py --mode exact --no-cpu-baseline > gpurun_out/r2f_bench_exact.log 2>&1; echo "bench exact rc=$?"
tail -c 1500 gpurun_out/r2f_bench_exact.log
cmd="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/r2f_launches.csv $cmd > gpurun_out/r2f_ncu1.log 2>&1; echo "ncu rc=$?"
