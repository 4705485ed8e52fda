#!/bin/bash
# scripts/ab_power.sh TAG "N M FAST" LIB[:ENV=V]...  sustained (power-capped) field A/B, twice
tag=$1; args=$2; shift 2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do for spec in "$@"; do
  lib=${spec%%:*}; env=""; [ "$spec" != "$lib" ] && env=${spec#*:}
  echo -n "$spec  "; env $env AFD_LIB_PATH=paper_1711_08604_b200/lib/ab/$lib.so timeout 120 python scripts/probe_power.py $args 4 2>&1 | tail -1
done; done 2>&1 | tee -a gpurun_out/${tag}_power.log
