#!/bin/bash
# round 2 (c): tests after the screened argmax + exact pow table; probes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r2c_tests.log
for a in "4096 1024 64 1" "4096 1024 64 0" "4096 512 1 1" "65536 4096 1 1" "1048576 2048 1 1"; do
  timeout 300 python scripts/probe_fast.py $a 5; done 2>&1 | tee gpurun_out/r2c_probe.log
