#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2u_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2u_tests.log
timeout 900 python bench.py > gpurun_out/r2u_c4_fast.json 2> gpurun_out/r2u_c4_fast.err; echo "c4 rc=$?"; tail -c 1600 gpurun_out/r2u_c4_fast.json
timeout 600 python bench.py --config c2 --steps 5 --no-cpu-baseline > gpurun_out/r2u_c2_fast.json 2> gpurun_out/r2u_c2_fast.err; echo "c2 rc=$?"
AFD_PRUNED=0 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2u_c4_fast_unpruned.json 2> gpurun_out/r2u_c4_fast_unpruned.err; echo "c4 unpruned rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"field_kernel|big_field_a|col_tma|prune_rows|pretwiddle" -c 6 -o gpurun_out/r2u_pruned_c4 -f python scripts/probe_fast.py 1048576 16384 1 1 1 > gpurun_out/r2u_ncu1.log 2>&1; echo "ncu1 rc=$?"
cmd="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2u_launches.csv $cmd > gpurun_out/r2u_ncu2.log 2>&1; echo "ncu2 rc=$?"
