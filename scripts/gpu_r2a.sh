#!/bin/bash
# round 2: fast-mode tests, full GPU suite, c4 default bench, c3/c1 fast benches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k fast > gpurun_out/r2a_fast_tests.log 2>&1; echo "fast tests rc=$?"
tail -5 gpurun_out/r2a_fast_tests.log
python bench.py --config c3 --mode fast --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2a_c3_fast.json 2> gpurun_out/r2a_c3_fast.err; echo "c3 fast rc=$?"
python bench.py --config c1 --mode fast --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_c1_fast.json 2> gpurun_out/r2a_c1_fast.err; echo "c1 fast rc=$?"
python bench.py > gpurun_out/r2a_c4_exact.json 2> gpurun_out/r2a_c4_exact.err; echo "c4 rc=$?"
python -m pytest tests -m gpu -q -x > gpurun_out/r2a_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/r2a_gpu_tests.log
