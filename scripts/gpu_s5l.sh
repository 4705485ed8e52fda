#!/bin/bash
# round 2, session 5 (l): per-kernel times of one c3 AFD step with the batched tiers
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5l
mkdir -p $O
cmd="python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:"field_reg_kernel|field_kernel|field_warp|prune_small|step_kernel" -s 24 -c 7 --csv \
   --log-file $O/c3_kernels.csv $cmd > $O/ncu2.log 2>&1; echo "ncu rc=$?"
grep -v "^==" $O/c3_kernels.csv | python -c "
import csv,sys
for r in csv.DictReader(sys.stdin):
    print(r['Kernel Name'][:44], r['Metric Name'], r['Metric Value'])
"
