#!/bin/bash
# round 2, session 5 (d): hints across tiers (4096-point tier first) + row splits of the warp tier
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5d
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "reg_tier or pruned or margins or fast" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_nc0.json 2> $O/bench_c4_nc0.err; echo "c4 rc=$?"
for nc in 20 12 8; do
AFD_WARP_NCTA=$nc timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > $O/bench_c4_nc$nc.json 2> $O/bench_c4_nc$nc.err; echo "c4 nc=$nc rc=$?"
done
python - <<'PY'
import json
for f in ("nc0","nc20","nc12","nc8"):
    try:
        d=json.loads(open("gpurun_out/s5d/bench_c4_%s.json"%f).read())
        print(f, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"])
    except Exception as e: print(f, "ERR", e)
PY
cmd="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"field_reg_kernel|field_warp_kernel|field_kernel" -s 12 -c 5 --csv \
   --log-file $O/tier_kernels.csv $cmd > $O/ncu2.log 2>&1; echo "ncu rc=$?"
grep -v "^==" $O/tier_kernels.csv | python -c "
import csv,sys
for r in csv.DictReader(sys.stdin):
    print(r['Kernel Name'][:40], r['Metric Name'], r['Metric Value'])
"
