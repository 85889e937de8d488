#!/bin/bash
# compute-sanitizer passes over the operator-step tests (memcheck, then racecheck on shared memory)
mkdir -p gpurun_out
K='operator_run_equals_three_steps'
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "$K or merge or clifford or split" -p no:cacheprovider > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?"; grep -c "Invalid\|out of bounds" gpurun_out/memcheck.log; tail -3 gpurun_out/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "$K and (8-3000 or 12-60 or 7-400 or 9-500)" -p no:cacheprovider > gpurun_out/racecheck.log 2>&1
echo "racecheck rc=$?"; grep -i "hazard\|race" gpurun_out/racecheck.log | sort | uniq -c | head -10; tail -3 gpurun_out/racecheck.log
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_engine.py tests/test_gpu_dist.py -q -m gpu -x -k "ladder or slot_partition or streamed or collapse or narrow_and_packed" -p no:cacheprovider > gpurun_out/memcheck_engine.log 2>&1
echo "memcheck engine rc=$?"; tail -3 gpurun_out/memcheck_engine.log
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --error-exitcode 9 python -m pytest tests/test_gpu_engine.py -q -m gpu -x -k "(ladder and (8_4 or 10_3) and v3) or narrow_and_packed" -p no:cacheprovider > gpurun_out/racecheck_engine.log 2>&1
echo "racecheck engine rc=$?"; tail -3 gpurun_out/racecheck_engine.log
