#!/bin/bash
# round 2, session 5 (g): register tiers for batches of on-chip fields (pruned_small): tests, c3 bench A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5g
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "small_pruned or c3 or bench_line or batch" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -25 $O/tests.log
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3_sp.json 2> $O/bench_c3_sp.err; echo "c3 rc=$?"
AFD_SMALL_PRUNED=0 timeout 600 python bench.py --config c3 --no-cpu-baseline --no-parity > $O/bench_c3_nosp.json 2> $O/bench_c3_nosp.err; echo "c3 nosp rc=$?"
python - <<'PY'
import json
for f in ("c3_sp","c3_nosp"):
    try:
        d=json.loads(open("gpurun_out/s5g/bench_%s.json"%f).read())
        print(f, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"], d["roofline"].get("split"))
    except Exception as e: print(f, "ERR", e)
PY
tail -c 600 $O/bench_c3_sp.err
