#!/bin/bash
# round 2, session 5 (z): two-pass limit read back by the host (empty row batches not launched): tests, c4 / c2 A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5z
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "default_tier or reg_tier or pruned or margins or fast or sharded or c4 or c2 or bench_line" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for c in c4 c2; do
st=3; [ $c = c2 ] && st=5
timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > $O/bench_${c}_rb.json 2> $O/bench_${c}_rb.err; echo "$c rc=$?"
AFD_LIM_READBACK=0 timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-parity > $O/bench_${c}_norb.json 2> $O/bench_${c}_norb.err; echo "$c norb rc=$?"
done
python - <<'PY'
import json
for c in ("c4","c2"):
  for v in ("rb","norb"):
    try:
        d=json.loads(open("gpurun_out/s5z/bench_%s_%s.json"%(c,v)).read())
        print(c, v, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["gpu_launches"])
    except Exception as e: print(c, v, "ERR", e)
PY
