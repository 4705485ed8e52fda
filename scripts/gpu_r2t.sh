#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export AFD_LIB_PATH=paper_1711_08604_b200/lib/ab/pr.so
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2t_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2t_tests.log
for a in "1048576 2048 1 1" "65536 4096 1 1" "1048576 16384 1 1"; do timeout 300 python scripts/probe_fast.py $a 3 | tail -1; done
timeout 120 python scripts/probe_power.py 1048576 16384 1 6 | tail -1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2t_bench.log 2>&1; echo "bench rc=$?"; tail -c 1200 gpurun_out/r2t_bench.log
