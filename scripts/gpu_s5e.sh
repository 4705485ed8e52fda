#!/bin/bash
# round 2, session 5 (e): tier grids sized by expected rows (tier_ncta) vs 37 row splits everywhere
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5e
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "reg_tier or pruned or margins or fast" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for c in c4 c2; do
st=3; [ $c = c2 ] && st=5
timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > $O/bench_${c}_pol.json 2> $O/bench_${c}_pol.err; echo "$c rc=$?"
AFD_TIER_NCTA=37 timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-parity > $O/bench_${c}_nc37.json 2> $O/bench_${c}_nc37.err; echo "$c nc37 rc=$?"
done
python - <<'PY'
import json
for f in ("c4_pol","c4_nc37","c2_pol","c2_nc37"):
    try:
        d=json.loads(open("gpurun_out/s5e/bench_%s.json"%f).read())
        print(f, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"])
    except Exception as e: print(f, "ERR", e)
PY
cmd="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:"field_reg_kernel|field_warp_kernel|field_kernel" -s 12 -c 5 --csv \
   --log-file $O/tier_kernels.csv $cmd > $O/ncu2.log 2>&1; echo "ncu rc=$?"
grep -v "^==" $O/tier_kernels.csv | python -c "
import csv,sys
for r in csv.DictReader(sys.stdin):
    print(r['Kernel Name'][:40], r['Metric Name'], r['Metric Value'])
"
