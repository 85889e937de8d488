"""Wall time of resident steps vs the sum of their kernel-class times (what the host, the syncs and
the launch gaps cost)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads, _native as nat
name = sys.argv[1] if len(sys.argv) > 1 else "c4_xyz_16_2"
n, gates = workloads.build(name)
def step():
    t0 = time.perf_counter()
    rep = qx.run(gates, n, "v3", download=False)
    rep.device["store"].synchronize()
    t1 = time.perf_counter()
    rep.device["store"].close()
    return t1 - t0, rep
for _ in range(3): step()
walls = [step()[0] for _ in range(10)]
nat.profile_enable(True); nat.profile_reset()
for _ in range(5): step()
prof = nat.profile_read(); nat.profile_enable(False)
kern = sum(v["ms"] for v in prof.values()) / 5
print(f"{name}: wall {1e3 * min(walls):.3f} ms (median {1e3 * sorted(walls)[5]:.3f}), kernels {kern:.3f} ms, gap {1e3 * min(walls) - kern:.3f} ms")
_, rep = step()
print({k: round(1e3 * v, 3) for k, v in rep.timings.items()})
