#!/bin/bash
# round 2, session 5 (h): c3 with the batched register tiers: bench line with the tier split, per-kernel times
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5h
mkdir -p $O
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3_fast.json 2> $O/bench_c3_fast.err; echo "c3 rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/s5h/bench_c3_fast.json").read())
print("%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["roofline"].get("split"))
PY
cmd="python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:"field_reg_kernel|field_kernel|prune_small|step_kernel" -s 20 -c 12 --csv \
   --log-file $O/c3_kernels.csv $cmd > $O/ncu2.log 2>&1; echo "ncu rc=$?"
grep -v "^==" $O/c3_kernels.csv | python -c "
import csv,sys
for r in csv.DictReader(sys.stdin):
    print(r['Kernel Name'][:44], r['Metric Name'], r['Metric Value'])
"
