#!/bin/bash
# round 2 (x): full GPU suite and every bench line with the pruned fast field
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2x_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2x_tests.log
timeout 900 python bench.py > gpurun_out/r2x_c4_fast.json 2> gpurun_out/r2x_c4_fast.err; echo "c4 fast rc=$?"
timeout 900 python bench.py --mode exact --no-cpu-baseline > gpurun_out/r2x_c4_exact.json 2> gpurun_out/r2x_c4_exact.err; echo "c4 exact rc=$?"
for c in c0 c1 c3 c2; do for m in fast exact; do
  st=30; [ $c == c2 ] && st=5; [ $c == c3 ] && st=5
  timeout 600 python bench.py --config $c --mode $m --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/r2x_${c}_${m}.json 2> gpurun_out/r2x_${c}_${m}.err; echo "$c $m rc=$?"
done; done
timeout 600 python bench.py --impl reference > gpurun_out/r2x_ref_c4.json 2> gpurun_out/r2x_ref_c4.err; echo "ref rc=$?"
