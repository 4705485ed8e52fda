#!/bin/bash
# round 2 (d): plain run of the sanitizer workload, then memcheck
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/sanitize_smoke.py > gpurun_out/r2d_plain.log 2>&1; echo "plain rc=$?"
tail -3 gpurun_out/r2d_plain.log
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --print-limit 50 python scripts/sanitize_smoke.py > gpurun_out/r2d_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -15 gpurun_out/r2d_memcheck.log
