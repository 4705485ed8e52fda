#!/bin/bash
# round 2 (g): bench lines c0-c3 both modes, field probes, ncu of the fast
# kernels (c4 pass A + column pass, c3 field), then compute-sanitizer memcheck
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c0 c1 c3 c2; do for m in fast exact; do
  st=30; [ $c == c2 ] && st=5; [ $c == c3 ] && st=5
  timeout 600 python bench.py --config $c --mode $m --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/r2g_${c}_${m}.json 2> gpurun_out/r2g_${c}_${m}.err; echo "$c $m rc=$?"
  tail -c 400 gpurun_out/r2g_${c}_${m}.json; echo
done; done
for a in "4096 1024 64 0" "4096 1024 64 1" "4096 512 1 1" "65536 4096 1 1" "1048576 2048 1 1"; do
  timeout 300 python scripts/probe_fast.py $a 5; done 2>&1 | tee gpurun_out/r2g_probe.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"big_field_a|col_tma" -s 2 -c 2 -o gpurun_out/r2g_big_c4_fast -f python scripts/probe_fast.py 1048576 2048 1 1 2 > gpurun_out/r2g_ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:field_kernel -s 2 -c 1 -o gpurun_out/r2g_field_c3_fast -f python scripts/probe_fast.py 4096 1024 64 1 2 > gpurun_out/r2g_ncu2.log 2>&1; echo "ncu2 rc=$?"
timeout 300 python scripts/sanitize_smoke.py > gpurun_out/r2g_plain.log 2>&1; echo "plain rc=$?"
tail -3 gpurun_out/r2g_plain.log
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --print-limit 50 python scripts/sanitize_smoke.py > gpurun_out/r2g_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -8 gpurun_out/r2g_memcheck.log
