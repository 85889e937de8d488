import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads, _native as nat
n, gates = workloads.build("c4_xyz_16_2")
for gens in ([0], list(range(1, 16)), list(range(16))):
    qx.run(gates, n, "v3", generators=gens, download=False).device["store"].close()
    nat.profile_enable(True); nat.profile_reset()
    rep = qx.run(gates, n, "v3", generators=gens, download=False); rep.device["store"].close()
    p = nat.profile_read(); nat.profile_enable(False)
    print(gens[:3], "... terms", sum(rep.rank_trace[-1]), "emit", round(p["dense_emit"]["ms"], 3), "sort", round(p["sort_pass"]["ms"], 3))
