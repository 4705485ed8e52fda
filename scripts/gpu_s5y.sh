#!/bin/bash
# round 2, session 5 (y): pruning tests from one log2 table and tabulated radius logs: tests + c2 / c4 lines
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5y
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "default_tier or reg_tier or pruned or margins or fast or sharded" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for c in c4 c2; do
st=3; [ $c = c2 ] && st=5
timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > $O/bench_${c}.json 2> $O/bench_${c}.err; echo "$c rc=$?"
done
python - <<'PY'
import json
for c in ("c4","c2"):
    try:
        d=json.loads(open("gpurun_out/s5y/bench_%s.json"%c).read())
        print(c, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["gpu_launches"])
    except Exception as e: print(c, "ERR", e)
PY
