#!/bin/bash
# round 2, session 4 (a): sanity after the container was re-created (smoke, short default bench)
# and ncu --set full of the two on-chip tiers of the pruned c4 field
cd $GRAFT_REPO_ROOT
O=gpurun_out/s4a
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_fast.json 2> $O/bench_c4_fast.err; echo "c4 fast rc=$?"
cmd="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'field_kernel<10' -s 2 -c 1 \
   -o $O/field10_c4 $cmd > $O/ncu2.log 2>&1; echo "ncu field10 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'field_kernel<12' -s 2 -c 1 \
   -o $O/field12_c4 $cmd > $O/ncu3.log 2>&1; echo "ncu field12 rc=$?"
ls -la $O
