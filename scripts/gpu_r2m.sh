#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for e in "AFD_COL_GROUPS=1" "AFD_COL_GROUPS=2" "AFD_COL_GROUPS=1 AFD_BIG_SKIP=1" "AFD_COL_GROUPS=2 AFD_BIG_SKIP=1" "AFD_BIG_SKIP=2"; do
  echo -n "[$e] "; env $e timeout 120 python scripts/probe_power.py 1048576 2048 1 4 | tail -1
done 2>&1 | tee gpurun_out/r2m_power.log
