#!/bin/bash
# round 2, session 5 (r): sub tiers chosen by expected work: default-choice test, c4 / c2 / c3 lines
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5r
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "default_tier or reg_tier or small_pruned or pruned" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for c in c4 c2 c3; do
st=3; [ $c = c2 ] && st=5
timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > $O/bench_${c}.json 2> $O/bench_${c}.err; echo "$c rc=$?"
done
python - <<'PY'
import json
for c in ("c4","c2","c3"):
    try:
        d=json.loads(open("gpurun_out/s5r/bench_%s.json"%c).read())
        print(c, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), {k:v for k,v in d["roofline"].get("split",{}).items() if k.startswith("rows_")})
    except Exception as e: print(c, "ERR", e)
PY
cmd="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:"field_reg_kernel|field_warp_kernel|field_kernel|field_sub" -s 16 -c 7 --csv \
   --log-file $O/tier_kernels.csv $cmd > $O/ncu2.log 2>&1; echo "ncu rc=$?"
grep -v "^==" $O/tier_kernels.csv | python -c "
import csv,sys
for r in csv.DictReader(sys.stdin):
    print(r['Kernel Name'][:44], r['Metric Name'], r['Metric Value'])
"
