#!/bin/bash
# ncu evidence for one round: launch list of the bench step + full captures of its hot kernels
R=${1:-r01h}
W=${2:-c4_xyz_16_2}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_${W}.csv \
    python tools/profile_step.py --workload $W --mode v3 --warmup 1 --steps 1 > gpurun_out/${R}_launches.log 2>&1
# the measured step is the second one: skip the launches of the warm-up step
for spec in "k_onesweep 5 1" "k_group_emit 1 1" "k_group_prep_small 3 1" "k_small_merge 1 1"; do
  set -- $spec
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 -f \
      -o gpurun_out/${R}_$1 python tools/profile_step.py --workload $W --mode v3 --warmup 1 --steps 1 \
      > gpurun_out/${R}_$1.log 2>&1
  echo "$1 rc=$?"
done
# the kernels of the gate-by-gate mode (v1) on a mid-size point of the ladder
for spec in "k_clifford 1 1" "k_split 83 1" "k_reduce 16 1" "k_sort_hist 16 1"; do
  set -- $spec
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 -f \
      -o gpurun_out/${R}_v1_$1 python tools/profile_step.py --workload c4_xyz_14_2 --mode v1 --warmup 0 --steps 1 \
      > gpurun_out/${R}_v1_$1.log 2>&1
  echo "v1 $1 rc=$?"
done
ls -la gpurun_out | tail -20
