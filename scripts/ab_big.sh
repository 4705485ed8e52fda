#!/bin/bash
# A/B of large-N field variants: scripts/ab_big.sh TAG LIB[:ENV=V]...
# probes c4 (N=2^20, 2048 radii) and c2 (N=2^16, M=4096) field times, fast and exact
tag=$1; shift
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for spec in "$@"; do
  lib=${spec%%:*}; env=""; [ "$spec" != "$lib" ] && env=${spec#*:}
  for a in "1048576 2048 1 1" "65536 4096 1 1" "1048576 1024 1 0" "65536 4096 1 0"; do
    echo -n "$spec  "; env $env AFD_LIB_PATH=paper_1711_08604_b200/lib/ab/$lib.so timeout 300 python scripts/probe_fast.py $a 5 2>&1 | tail -1
  done
done; done 2>&1 | tee gpurun_out/${tag}_ab.log
