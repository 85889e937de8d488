"""Where the e2e milliseconds go: the packed download (copy + host widening) of the bench result on
its own, against a plain copy of the same bytes, and the whole public-API run."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads, _native as nat

n, gates = workloads.build(sys.argv[1] if len(sys.argv) > 1 else "c4_xyz_16_2")
for i in range(4):
    rep = qx.run(gates, n, "v3", download=False, keep_narrow=2) if "keep_narrow" in qx.run.__code__.co_varnames else qx.run(gates, n, "v3", download=False)
    st = rep.device["store"]
    st.synchronize()
    t0 = time.perf_counter()
    off, keys, lam = st.download_async(pinned=True)
    t1 = time.perf_counter()
    st.synchronize()
    t2 = time.perf_counter()
    print(f"download alone: issue {1e3 * (t1 - t0):.2f} ms, done {1e3 * (t2 - t0):.2f} ms, {st.d2h_bytes / 1e9:.3f} GB "
          f"-> {st.d2h_bytes / (t2 - t0) / 1e9:.1f} GB/s  terms {int(off[-1])}")
    st.close()
    del keys, lam
for i in range(3):
    t0 = time.perf_counter()
    rep = qx.run(gates, n, "v3", pinned=True)
    t1 = time.perf_counter()
    print(f"run(pinned=True): {1e3 * (t1 - t0):.2f} ms  {rep.device.get('streamed_ranges')} ranges")
    del rep
