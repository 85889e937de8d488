"""Per-generator term-gate update counts (v1 semantics) of the bench workloads,
measured with the GPU's own v1 mode; written to gpurun_out/updates.json and then committed as
tests/golden/updates.json (the CPU arm of bench.py has no GPU to count with).  The totals are
pinned against the reference where it could run: c2 = 4350, c4(8,4) = 12 816 194, c5 = 31 171 459
(tests/golden/configs.npz, digests.json)."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads

out = {}
for name in sys.argv[1:] or ["c2_10q_near_clifford", "c4_xyz_8_4", "c4_xyz_12_2", "c4_xyz_14_2", "c4_xyz_16_2",
                             "c5_32q_clifford_t"]:
    n, gates = workloads.build(name)
    rep = qx.run(gates, n, "v1", download=False)
    rep.device["store"].close()
    out[name] = rep.device["updates_per_generator"]
    print(name, sum(out[name]), rep.rank_trace[-1], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/updates.json", "w") as fh:
    json.dump({"_meta": {"source": "GPU v1 mode, tools/make_updates.py"}, "data": out}, fh)
