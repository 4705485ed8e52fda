#!/bin/bash
# Usage (on the GPU box via gpurun): scripts/gpu_check.sh [tag] [ncu]
# Runs the GPU parity tests, the bench, and optionally an ncu launch list +
# full captures of the field and step kernels, writing into gpurun_out/.
tag=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_tests.log
tail -3 gpurun_out/${tag}_tests.log
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/${tag}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${tag}_bench.log
tail -2 gpurun_out/${tag}_bench.log
if [ "$2" == "ncu" ]; then
  cmd="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
  $cmd > gpurun_out/${tag}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/${tag}_launches.csv $cmd > gpurun_out/${tag}_ncu1.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:field_kernel -s 3 -c 1 \
      -o gpurun_out/${tag}_field $cmd > gpurun_out/${tag}_ncu2.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"step_cluster_kernel|step_kernel" -s 3 -c 1 \
      -o gpurun_out/${tag}_step $cmd > gpurun_out/${tag}_ncu3.log 2>&1
fi
