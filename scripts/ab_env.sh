#!/bin/bash
# scripts/ab_env.sh TAG LIB "N M B FAST" ENV...   (ENV "-" = none), twice each
tag=$1; lib=$2; args=$3; shift 3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do for e in "$@"; do
  [ "$e" == "-" ] && e=""
  echo -n "[$e]  "; env $e AFD_LIB_PATH=paper_1711_08604_b200/lib/ab/$lib.so timeout 300 python scripts/probe_fast.py $args 5 2>&1 | tail -1
done; done 2>&1 | tee -a gpurun_out/${tag}_env.log
