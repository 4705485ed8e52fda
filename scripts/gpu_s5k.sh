#!/bin/bash
# round 2, session 5 (k): 1024-point warp tier inside batches of on-chip fields (c3): tests, A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5k
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "small_pruned or c3 or batch or margins" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -4 $O/tests.log
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3_w1k.json 2> $O/bench_c3_w1k.err; echo "c3 rc=$?"
AFD_SMALL_WARP_TIER=0 timeout 600 python bench.py --config c3 --no-cpu-baseline --no-parity > $O/bench_c3_now1k.json 2> $O/bench_c3_now1k.err; echo "c3 now1k rc=$?"
python - <<'PY'
import json
for f in ("c3_w1k","c3_now1k"):
    try:
        d=json.loads(open("gpurun_out/s5k/bench_%s.json"%f).read())
        print(f, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"], {k:v for k,v in d["roofline"].get("split",{}).items() if k.startswith("rows_")})
    except Exception as e: print(f, "ERR", e)
PY
tail -c 400 $O/bench_c3_w1k.err
