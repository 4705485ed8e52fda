#!/bin/bash
# round 2, session 4 (b): warp-per-row 1024-point tier: fast/pruned parity tests, c4 bench A/B, TMEM bandwidth
cd $GRAFT_REPO_ROOT
O=gpurun_out/s4b
mkdir -p $O
timeout 120 scripts/micro/tmem_bw > $O/tmem_bw.txt 2>&1; echo "tmem_bw rc=$?"; cat $O/tmem_bw.txt
timeout 1200 python -m pytest tests -m gpu -x -q -k "fast or pruned or margins" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -5 $O/tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_warp.json 2> $O/bench_c4_warp.err; echo "c4 warp rc=$?"
AFD_WARP_FIELD=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > $O/bench_c4_old.json 2> $O/bench_c4_old.err; echo "c4 old rc=$?"
python - <<'PY'
import json
for f in ("warp","old"):
    try:
        d=json.loads(open("gpurun_out/s4b/bench_c4_%s.json"%f).read())
        print(f, "%.4e"%d["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"])
    except Exception as e: print(f, "ERR", e)
PY
