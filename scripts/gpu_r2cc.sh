#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2cc_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2cc_tests.log
for c in c1 c3 c4 c2; do
  st=30; [ $c == c2 ] && st=5; [ $c == c3 ] && st=5; [ $c == c4 ] && st=5
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/r2cc_${c}.json 2> gpurun_out/r2cc_${c}.err; echo "$c rc=$?"
done
