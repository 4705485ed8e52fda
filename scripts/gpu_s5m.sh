#!/bin/bash
# round 2, session 5 (m): faster prune_small (early exit on the first passing tier, 4 chains): c3 tests + bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5m
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "small_pruned or c3 or batch or margins" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3_fast.json 2> $O/bench_c3_fast.err; echo "c3 rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/s5m/bench_c3_fast.json").read())
print("%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"])
PY
cmd="python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prune_small" -s 3 -c 1 --csv --log-file $O/ps.csv $cmd > $O/ncu2.log 2>&1; echo "ncu rc=$?"
grep -v "^==" $O/ps.csv | tail -1
