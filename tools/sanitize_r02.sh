#!/bin/bash
# compute-sanitizer over the round-2 kernels: the one-launch circuit kernel (csrc/program.cuh), the
# bucketed operator step (csrc/bucket.cuh), the support compaction above 32 qubits (csrc/wide.cu)
mkdir -p gpurun_out
out=gpurun_out/r02q_sanitizer.txt
: > $out
run() {  # tool, extra flags, pytest args...
  tool=$1; shift; flags=$1; shift
  echo "## compute-sanitizer --tool $tool $flags  pytest $*" >> $out
  timeout 1800 compute-sanitizer --tool $tool $flags --error-exitcode 9 python -m pytest "$@" -q -m gpu -x -p no:cacheprovider > gpurun_out/san_tmp.log 2>&1
  echo "rc=$?" >> $out
  grep -i "hazard\|Invalid\|out of bounds\|ERROR SUMMARY\|passed\|failed" gpurun_out/san_tmp.log | sort | uniq -c | tail -8 >> $out
}
run memcheck "" tests/test_gpu_program.py -k "random_circuits or baseline_configs or collapse or initial or outgrows"
run racecheck "--racecheck-report analysis" tests/test_gpu_program.py -k "baseline_configs or (random_circuits and v3)"
run memcheck "" tests/test_gpu_bucket.py
run racecheck "--racecheck-report analysis" tests/test_gpu_bucket.py
run memcheck "" tests/test_gpu_wide.py -k "compact or support or embedded or idle or leaves_alone"
cat $out
