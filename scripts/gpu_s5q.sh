#!/bin/bash
# round 2, session 5 (q): 256- / 512-point sub-warp tiers: tests, c4 / c2 / c3 A/B (AFD_SUB_TIERS=0)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5q
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "reg_tier or small_pruned or pruned or margins or fast or bench_line" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -12 $O/tests.log
for c in c4 c2 c3; do
st=3; [ $c = c2 ] && st=5
timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > $O/bench_${c}_sub.json 2> $O/bench_${c}_sub.err; echo "$c rc=$?"
AFD_SUB_TIERS=0 timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-parity > $O/bench_${c}_nosub.json 2> $O/bench_${c}_nosub.err; echo "$c nosub rc=$?"
done
python - <<'PY'
import json
for c in ("c4","c2","c3"):
  for v in ("sub","nosub"):
    try:
        d=json.loads(open("gpurun_out/s5q/bench_%s_%s.json"%(c,v)).read())
        print(c, v, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), {k:v for k,v in d["roofline"].get("split",{}).items() if k.startswith("rows_")})
    except Exception as e: print(c, v, "ERR", e)
PY
tail -c 300 $O/bench_c4_sub.err
