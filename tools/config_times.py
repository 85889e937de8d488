"""Wall time of every BASELINE config through the public API (best of N), with the device log."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads, _native as nat

REF = {  # reference seconds measured in the survey, v1 / v3
    "c1_4q_clifford_t": (0.003, 0.004), "c2_10q_near_clifford": (0.11, 0.15), "c3_16q_clifford": (0.80, 1.12),
    "c4_xyz_8_4": (1.28, 37.3), "c4_xyz_12_2": (2.22, 0.97), "c5_32q_clifford_t": (29.0, 122.6),
}
for name in sys.argv[1:] or list(REF):
    n, gates = workloads.build(name)
    for mi, mode in enumerate(("v1", "v3")):
        best, rep = 1e9, None
        for _ in range(5):
            l0 = nat.launch_count()
            t0 = time.perf_counter()
            rep = qx.run(gates, n, mode)
            best = min(best, time.perf_counter() - t0)
            launches = nat.launch_count() - l0
        print(f"{name:24s} {mode}: {best * 1e3:9.3f} ms  (reference {REF[name][mi]:8.3f} s, x{REF[name][mi] / best:9.0f})  "
              f"launches {launches:5d}  {rep.device['clifford_runs']} runs / {rep.device['branch_ops']} branch / "
              f"{rep.device['merges']} merges / {rep.device['sorts']} sorts  host: "
              + " ".join(f"{k}={v * 1e3:.2f}" for k, v in rep.timings.items()), flush=True)
