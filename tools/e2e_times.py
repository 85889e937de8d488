"""e2e timing of the public API (pinned download) on one workload, with the per-phase walls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads
name = sys.argv[1] if len(sys.argv) > 1 else "c4_xyz_16_2"
n, gates = workloads.build(name)
for i in range(6):
    t0 = time.perf_counter()
    rep = qx.run(gates, n, "v3", pinned=True)
    t1 = time.perf_counter()
    tot = sum(g.rank for g in rep.final.generators)
    print(f"step {i}: {1e3 * (t1 - t0):8.2f} ms  terms {tot}  {rep.device}  timings {{{', '.join(f'{k}: {1e3*v:.2f}' for k, v in rep.timings.items())}}}")
    del rep
