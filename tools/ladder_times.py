"""Times of the xyz_chain ladder points through the public API (v3, results stay on the device)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads, _native
points = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(8, 4), (10, 3), (12, 2), (14, 2)]
for n, layers in points:
    _, gates = workloads.config4(n, layers)
    best, info = 1e9, None
    for i in range(5):
        t0 = time.perf_counter()
        rep = qx.run(gates, n, "v3", download=False)
        rep.device["store"].synchronize()
        best = min(best, time.perf_counter() - t0)
        info = _native.dense_last()
        terms = sum(rep.device["store"].ranks())
        rep.device["store"].close()
    print(f"xyz_chain({n},{layers}) v3: {1e3 * best:8.3f} ms  final terms {terms}  last grouped step {info}")
