import time, sys
sys.path.insert(0, '.')
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads
for name in ("c4_xyz_20_2", "c4_xyz_20_4"):
    n, gates = workloads.build(name)
    t = time.time()
    try:
        rep = qx.run(gates, n, "v3", download=False)
        print(name, "ran?!", sum(rep.rank_trace[-1]))
        rep.device["store"].close()
    except Exception as e:
        print(name, type(e).__name__, str(e)[:300], f"{time.time()-t:.2f}s")
n, gates = workloads.build("c4_xyz_12_2")
rep = qx.run(gates, n, "v3")
print("after:", sum(rep.rank_trace[-1]))
