"""Host timeline of one resident step: every DeviceStore call with its start and duration (no extra
synchronisation), to see where the host waits for the device and where the device waits for the host."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import store as store_mod, workloads, lut as lut_mod, circuit as circ_mod

name = sys.argv[1] if len(sys.argv) > 1 else "c4_xyz_16_2"
mode = sys.argv[2] if len(sys.argv) > 2 else "v3"
log = []
T0 = [0.0]

def wrap(obj, attr, label=None):
    orig = getattr(obj, attr)
    def timed(*a, **k):
        t0 = time.perf_counter()
        out = orig(*a, **k)
        log.append((label or attr, 1e3 * (t0 - T0[0]), 1e3 * (time.perf_counter() - t0)))
        return out
    setattr(obj, attr, timed)

for m in ("__init__", "init_z", "apply_clifford", "apply_split", "apply_operator", "apply_operator_run",
          "count_operator", "merge", "sort", "ranks", "synchronize", "run_program", "order_for_operator", "close"):
    if hasattr(store_mod.DeviceStore, m):
        wrap(store_mod.DeviceStore, m)
wrap(lut_mod, "build_lut")
n, gates = workloads.build(name)
for i in range(4):
    log.clear()
    T0[0] = time.perf_counter()
    rep = qx.run(gates, n, mode, download=False)
    rep.device["store"].synchronize()
    total = 1e3 * (time.perf_counter() - T0[0])
    rep.device["store"].close()
print(f"{name} {mode}: {total:.3f} ms")
for label, start, dur in log:
    print(f"  {start:8.3f} ms  +{dur:7.3f}  {label}")
