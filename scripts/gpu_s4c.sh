#!/bin/bash
# round 2, session 4 (c): ncu --set full of the warp-per-row tier kernel and of field_kernel<10> (old tier 0)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s4c
mkdir -p $O
cmd="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:field_warp_kernel -s 2 -c 1 \
   -o $O/field_warp_c4 $cmd > $O/ncu1.log 2>&1; echo "ncu warp rc=$?"
AFD_WARP_FIELD=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:field_kernel -s 4 -c 1 \
   -o $O/field10_c4 $cmd > $O/ncu2.log 2>&1; echo "ncu field10 rc=$?"
ls -la $O
