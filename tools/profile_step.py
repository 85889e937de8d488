"""One warm-up step + N measured steps of a workload, nothing else: the command ncu wraps.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
        python tools/profile_step.py --workload c4_xyz_16_2 --mode v3
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4_xyz_16_2")
ap.add_argument("--mode", default="v3")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
args = ap.parse_args()
n, gates = workloads.build(args.workload)
for i in range(args.warmup + args.steps):
    rep = qx.run(gates, n, args.mode, download=False)
    rep.device["store"].close()
print(args.workload, args.mode, "final terms", sum(rep.rank_trace[-1]), rep.device)
