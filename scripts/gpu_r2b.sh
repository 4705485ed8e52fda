#!/bin/bash
# round 2 (b): fast + sharded tests, fast benches, field probes, ncu of fast kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -k "fast or sharded" > gpurun_out/r2b_tests.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/r2b_tests.log
for a in "4096 1024 64 0" "4096 1024 64 1" "4096 512 1 1" "1024 100 1 1" "8192 1024 16 1" "65536 4096 1 0" "65536 4096 1 1" "1048576 2048 1 1"; do
  timeout 300 python scripts/probe_fast.py $a 5; done 2>&1 | tee gpurun_out/r2b_probe.log
python bench.py --mode fast > gpurun_out/r2b_c4_fast.json 2> gpurun_out/r2b_c4_fast.err; echo "c4 fast rc=$?"
python bench.py --config c2 --mode fast --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2b_c2_fast.json 2> gpurun_out/r2b_c2_fast.err; echo "c2 fast rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:field_kernel -s 2 -c 1 -o gpurun_out/r2b_field_c3_fast -f python scripts/probe_fast.py 4096 1024 64 1 2 > gpurun_out/r2b_ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"big_field_a|col_tma" -s 2 -c 2 -o gpurun_out/r2b_big_c4_fast -f python scripts/probe_fast.py 1048576 2048 1 1 2 > gpurun_out/r2b_ncu2.log 2>&1; echo "ncu2 rc=$?"
