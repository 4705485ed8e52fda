#!/bin/bash
# round 2, session 5 (u): launch list of one c2 fast decomposition
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5u
mkdir -p $O
cmd="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
   --log-file $O/launches_c2.csv $cmd > $O/ncu1.log 2>&1; echo "ncu list rc=$?"
python profiles/launch_summary.py $O/launches_c2.csv | head -40
