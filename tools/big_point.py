"""A GPU-only point of the config-4 ladder: run resident, check sum(lambda^2) = 1 per generator."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads, _native as nat
name = sys.argv[1] if len(sys.argv) > 1 else "c4_xyz_18_2"
n, gates = workloads.build(name)
for i in range(2):
    t0 = time.perf_counter()
    rep = qx.run(gates, n, "v3", download=False)
    st = rep.device["store"]
    st.synchronize()
    dt = time.perf_counter() - t0
    norms = st.norms()
    cap, hbm = st.capacity()
    print(f"{name} run {i}: {1e3 * dt:.2f} ms, final terms {sum(rep.rank_trace[-1])}, max |sum l^2 - 1| = {np.max(np.abs(norms - 1)):.3e}, HBM {hbm / 1e9:.1f} GB")
    st.close()
