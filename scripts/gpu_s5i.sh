#!/bin/bash
# round 2, session 5 (i): D = 4 register kernel with three shared-memory-fed warps (A/B vs four warps), faster prune_small
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5i
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "reg_tier or small_pruned or pruned or margins or fast or bench_line" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for c in c4 c3; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_${c}_sm3.json 2> $O/bench_${c}_sm3.err; echo "$c rc=$?"
AFD_LIB_PATH=$PWD/paper_1711_08604_b200/lib/ab/sm0.so timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-parity > $O/bench_${c}_sm0.json 2> $O/bench_${c}_sm0.err; echo "$c sm0 rc=$?"
done
python - <<'PY'
import json
for f in ("c4_sm3","c4_sm0","c3_sm3","c3_sm0"):
    try:
        d=json.loads(open("gpurun_out/s5i/bench_%s.json"%f).read())
        print(f, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"])
    except Exception as e: print(f, "ERR", e)
PY
cmd="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:"field_reg_kernel<4" -s 4 -c 1 --csv \
   --log-file $O/reg4.csv $cmd > $O/ncu2.log 2>&1; echo "ncu rc=$?"
grep -v "^==" $O/reg4.csv | python -c "
import csv,sys
for r in csv.DictReader(sys.stdin):
    print(r['Kernel Name'][:44], r['Metric Name'], r['Metric Value'])
"
