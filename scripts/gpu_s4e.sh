#!/bin/bash
# round 2, session 4 (e): warp kernel with CTA threshold + scheduler phase offset; A/B against each switched off
cd $GRAFT_REPO_ROOT
O=gpurun_out/s4e
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "fast or pruned or margins" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_main.json 2> $O/bench_c4_main.err; echo "c4 main rc=$?"
for v in fw_nooffset fw_noctathr; do
AFD_LIB_PATH=$PWD/paper_1711_08604_b200/lib/ab/$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > $O/bench_c4_$v.json 2> $O/bench_c4_$v.err; echo "c4 $v rc=$?"
done
python - <<'PY'
import json
for f in ("main","fw_nooffset","fw_noctathr"):
    try:
        d=json.loads(open("gpurun_out/s4e/bench_c4_%s.json"%f).read())
        print(f, "%.4e"%d["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"])
    except Exception as e: print(f, "ERR", e)
PY
