#!/bin/bash
# round 2, session 4 (d): ncu --set full of the warp-per-row tier kernel + launch list of one c4 bench step
cd $GRAFT_REPO_ROOT
O=gpurun_out/s4d
mkdir -p $O
cmd="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:field_warp_kernel -s 2 -c 1 \
   -o $O/field_warp_c4 $cmd > $O/ncu1.log 2>&1; echo "ncu warp rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
   --log-file $O/launches_c4.csv $cmd > $O/ncu2.log 2>&1; echo "ncu list rc=$?"
ls -la $O
