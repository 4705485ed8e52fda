#!/bin/bash
# round 2, session 5 (o): two row sets sharing tensor memory in the 128-term register kernel (8 warps; A/B vs 4)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5o
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "reg_tier or small_pruned or pruned or margins" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for c in c4 c3; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_${c}_sh2.json 2> $O/bench_${c}_sh2.err; echo "$c rc=$?"
AFD_LIB_PATH=$PWD/paper_1711_08604_b200/lib/ab/share1.so timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-parity > $O/bench_${c}_sh1.json 2> $O/bench_${c}_sh1.err; echo "$c sh1 rc=$?"
done
python - <<'PY'
import json
for f in ("c4_sh2","c4_sh1","c3_sh2","c3_sh1"):
    try:
        d=json.loads(open("gpurun_out/s5o/bench_%s.json"%f).read())
        print(f, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"])
    except Exception as e: print(f, "ERR", e)
PY
