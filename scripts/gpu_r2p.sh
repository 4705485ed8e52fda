#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AFD_LIB_PATH=paper_1711_08604_b200/lib/ab/r4.so timeout 900 python -m pytest tests -m gpu -q -x -k "fast" > gpurun_out/r2p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2p_tests.log
bash scripts/ab_big.sh r2p g2 r4 2>&1 | grep "fast=1"
for lib in g2 r4; do for a in "4096 1024 64 1" "4096 512 1 1"; do echo -n "$lib "; AFD_LIB_PATH=paper_1711_08604_b200/lib/ab/$lib.so python scripts/probe_fast.py $a 10 | tail -1; done; done
bash scripts/ab_power.sh r2p "1048576 2048 1" g2 r4
