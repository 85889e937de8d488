#!/bin/bash
# GPU test pass: each test file in its own process so one hang cannot take the rest down
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
: > gpurun_out/summary.txt
for f in ${@:-test_gpu_kernels test_gpu_engine test_gpu_dist test_gpu_wide test_gpu_fullsize}; do
  timeout -k 10 900 python -m pytest tests/$f.py -q -m gpu --tb=short -p no:cacheprovider > gpurun_out/$f.log 2>&1
  echo "$f exit $?" >> gpurun_out/summary.txt
  tail -n 3 gpurun_out/$f.log
done
cat gpurun_out/summary.txt
