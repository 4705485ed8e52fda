#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5w
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "small_pruned" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -15 $O/tests.log
