#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export AFD_LIB_PATH=paper_1711_08604_b200/lib/ab/g2.so
AFD_COL_GROUPS=2 timeout 900 python -m pytest tests -m gpu -q -x -k "big or large or c2 or c4 or n65536 or fast" > gpurun_out/r2k_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2k_tests.log
for g in 1 2; do for a in "1048576 2048 1 1" "65536 4096 1 1" "1048576 1024 1 0" "65536 4096 1 0"; do
  echo -n "groups=$g "; AFD_COL_GROUPS=$g timeout 300 python scripts/probe_fast.py $a 5 | tail -1; done
  echo -n "groups=$g colonly "; AFD_BIG_SKIP=1 AFD_COL_GROUPS=$g timeout 300 python scripts/probe_fast.py 1048576 2048 1 1 5 | tail -1
done 2>&1 | tee gpurun_out/r2k_probe.log
