#!/bin/bash
# usage: tools/ncu_one.sh <tag> <kernel-regex> <skip> <count> [workload] [mode]
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 -f \
    -o gpurun_out/$1 python tools/profile_step.py --workload ${5:-c4_xyz_14_2} --mode ${6:-v3} --warmup 1 --steps 1 \
    > gpurun_out/$1.log 2>&1
echo "$1 rc=$?"
