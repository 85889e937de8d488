#!/bin/bash
# Round evidence in one call: tools/r02_evidence.sh <tag>  -> gpurun_out/<tag>_*
R=${1:-r02k}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/${R}_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -n 2 gpurun_out/${R}_gputests.log
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/${R}_bench_reference_arm.json 2>> gpurun_out/${R}_bench.err; echo "ref arm rc=$?"
python tools/config_times.py > gpurun_out/${R}_config_times.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_c4_xyz_16_2.csv \
    python tools/profile_step.py --workload c4_xyz_16_2 --mode v3 --warmup 1 --steps 1 > gpurun_out/${R}_launches.log 2>&1
for spec in "k_bucket_emit 1 1" "k_tile_desc 1 1"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 -f \
      -o gpurun_out/${R}_$1 python tools/profile_step.py --workload c4_xyz_16_2 --mode v3 --warmup 1 --steps 1 \
      > gpurun_out/${R}_$1.log 2>&1
  echo "$1 rc=$?"
done
# the one-launch circuit kernel on config 5 (whole circuit = one launch of k_small_circuit)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small_circuit -s 2 -c 1 -f \
    -o gpurun_out/${R}_k_small_circuit python tools/profile_step.py --workload c5_32q_clifford_t --mode v3 --warmup 2 --steps 1 \
    > gpurun_out/${R}_k_small_circuit.log 2>&1
echo "k_small_circuit rc=$?"
python tools/program_times.py > gpurun_out/${R}_program_times.txt 2>&1
