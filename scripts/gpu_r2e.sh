#!/bin/bash
# round 2 (e): TMEM twiddles in the TMA column pass; pass A direct stores A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "big or large or c2 or c4_length or fused or sharded or n65536" > gpurun_out/r2e_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2e_tests.log
for d in 0 1; do for a in "65536 4096 1 1" "1048576 2048 1 1" "65536 4096 1 0" "1048576 1024 1 0"; do
  AFD_PASSA_DIRECT=$d timeout 300 python scripts/probe_fast.py $a 5 | sed "s/^/direct=$d /"; done; done 2>&1 | tee gpurun_out/r2e_probe.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"big_field_a|col_tma" -s 2 -c 2 -o gpurun_out/r2e_big_c4_fast -f python scripts/probe_fast.py 1048576 2048 1 1 2 > gpurun_out/r2e_ncu.log 2>&1; echo "ncu rc=$?"
