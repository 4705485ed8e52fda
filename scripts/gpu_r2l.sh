#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2l_bench.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/r2l_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"big_field_a|col_tma" -s 2 -c 2 -o gpurun_out/r2l_big_c4_fast -f python scripts/probe_fast.py 1048576 2048 1 1 2 > gpurun_out/r2l_ncu1.log 2>&1; echo "ncu1 rc=$?"
