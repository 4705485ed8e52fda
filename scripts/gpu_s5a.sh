#!/bin/bash
# round 2, session 5 (a): register tiers (32 / 64 spectrum terms) of the pruned field: tests, c4 and c2 bench A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5a
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "reg_tier or pruned or margins or fast" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -15 $O/tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_reg.json 2> $O/bench_c4_reg.err; echo "c4 reg rc=$?"
AFD_REG_TIERS=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > $O/bench_c4_noreg.json 2> $O/bench_c4_noreg.err; echo "c4 noreg rc=$?"
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c2_reg.json 2> $O/bench_c2_reg.err; echo "c2 reg rc=$?"
AFD_REG_TIERS=0 timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --no-parity > $O/bench_c2_noreg.json 2> $O/bench_c2_noreg.err; echo "c2 noreg rc=$?"
python - <<'PY'
import json
for f in ("c4_reg","c4_noreg","c2_reg","c2_noreg"):
    try:
        d=json.loads(open("gpurun_out/s5a/bench_%s.json"%f).read())
        print(f, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"], {k:v for k,v in d["roofline"].get("split",{}).items() if k.startswith("rows")})
    except Exception as e: print(f, "ERR", e)
PY
tail -5 $O/*.err
