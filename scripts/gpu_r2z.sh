#!/bin/bash
# round 2 (z): final state — full GPU suite, smoke, every bench line, reference arm,
# launch list of the default bench command
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2z_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2z_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2z_smoke.log
timeout 900 python bench.py > gpurun_out/r2z_c4_fast.json 2> gpurun_out/r2z_c4_fast.err; echo "c4 fast rc=$?"
timeout 900 python bench.py --mode exact --no-cpu-baseline > gpurun_out/r2z_c4_exact.json 2> gpurun_out/r2z_c4_exact.err; echo "c4 exact rc=$?"
for c in c0 c1 c3 c2; do for m in fast exact; do
  st=30; [ $c == c2 ] && st=5; [ $c == c3 ] && st=5
  timeout 600 python bench.py --config $c --mode $m --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/r2z_${c}_${m}.json 2> gpurun_out/r2z_${c}_${m}.err; echo "$c $m rc=$?"
done; done
timeout 600 python bench.py --impl reference > gpurun_out/r2z_ref_c4.json 2> gpurun_out/r2z_ref_c4.err; echo "ref rc=$?"
cmd="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2z_launches.csv $cmd > gpurun_out/r2z_ncu.log 2>&1; echo "ncu rc=$?"
