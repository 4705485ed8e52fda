#!/bin/bash
# round 2, session 5 (ab): full GPU suite on the five-tier pruned field, bench lines for every
# config/engine (v15), reference arm, launch list of the default bench, ncu of the tier kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5ab
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -3 $O/gpu_tests.log
timeout 600 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_c4_fast.json 2> $O/bench_c4_fast.err; echo "c4 fast rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err; echo "ref rc=$?"
for c in c2 c3; do for m in fast exact; do
timeout 600 python bench.py --config $c --mode $m --no-cpu-baseline > $O/bench_${c}_${m}.json 2> $O/bench_${c}_${m}.err; echo "$c $m rc=$?"
done; done
timeout 600 python bench.py --mode exact --no-cpu-baseline > $O/bench_c4_exact.json 2> $O/bench_c4_exact.err; echo "c4 exact rc=$?"
for c in c0 c1; do for m in fast exact; do
timeout 300 python bench.py --config $c --mode $m --steps 100 --warmup 10 --no-cpu-baseline > $O/bench_${c}_${m}.json 2> $O/bench_${c}_${m}.err; echo "$c $m rc=$?"
done; done
cmd="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
   --log-file $O/launches_c4.csv $cmd > $O/ncu1.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'field_kernel<12' -s 0 -c 1 \
   -o $O/field12_c4 $cmd > $O/ncu2.log 2>&1; echo "ncu warp/reg4 rc=$?"
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/s5ab/bench_*.json")):
    try:
        d=json.loads(open(f).read())
        print(f.split("/")[-1], "%.4e"%d["value"], "e2e %.4e"%d["e2e"]["value"], d["roofline"]["bound"], "%.3f"%d["roofline"]["frac"], d["roofline"].get("launch_ms"), d.get("parity_vs_oracle"), d.get("clocks"))
    except Exception as e: print(f, "ERR", e)
PY
