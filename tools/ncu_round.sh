#!/bin/bash
# ncu evidence for one round: launch list at full size + full captures of the hot kernels at (14,2)
R=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_c4_16_2.csv \
    python tools/profile_step.py --workload c4_xyz_16_2 --mode v3 --warmup 1 --steps 1 > gpurun_out/${R}_launches.log 2>&1
for k in k_onesweep k_expand_emit k_reduce k_clifford k_sort_hist; do
  case $k in
    k_onesweep) skip=4; cnt=2;;        # 4 passes per step: skip the warm-up step
    k_expand_emit|k_clifford) skip=3; cnt=1;;   # 2 per step, the second one is the big one
    k_reduce) skip=1; cnt=1;;
    k_sort_hist) skip=1; cnt=1;;
    *) skip=2; cnt=1;;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c $cnt -f \
      -o gpurun_out/${R}_${k} python tools/profile_step.py --workload c4_xyz_14_2 --mode v3 --warmup 1 --steps 1 \
      > gpurun_out/${R}_${k}.log 2>&1
  echo "$k rc=$?"
done
# traffic of the dominant kernel at the bench workload itself (first pass of the measured step)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 4 -c 1 -f \
    -o gpurun_out/${R}_k_onesweep_16_2 python tools/profile_step.py --workload c4_xyz_16_2 --mode v3 --warmup 1 --steps 1 \
    > gpurun_out/${R}_k_onesweep_16_2.log 2>&1
echo "onesweep@16_2 rc=$?"
ls -la gpurun_out | tail -20
