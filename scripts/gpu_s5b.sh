#!/bin/bash
# round 2, session 5 (b): register tier D = 1 with 12 warps per CTA (A/B) + ncu --set full of both register kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5b
mkdir -p $O
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > $O/bench_c4_main.json 2> $O/bench_c4_main.err; echo "c4 main rc=$?"
AFD_LIB_PATH=$PWD/paper_1711_08604_b200/lib/ab/fr12.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_fr12.json 2> $O/bench_c4_fr12.err; echo "c4 fr12 rc=$?"
python - <<'PY'
import json
for f in ("c4_main","c4_fr12"):
    try:
        d=json.loads(open("gpurun_out/s5b/bench_%s.json"%f).read())
        print(f, "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d.get("parity_vs_oracle"), d["clocks"])
    except Exception as e: print(f, "ERR", e)
PY
cmd="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:field_reg_kernel -s 2 -c 2 \
   -o $O/field_reg_c4 $cmd > $O/ncu1.log 2>&1; echo "ncu reg rc=$?"
ls -la $O
