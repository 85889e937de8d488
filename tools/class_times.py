"""Per kernel-class CUDA-event times of one workload/mode (instrumented run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads, _native as nat
name, mode = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "v3")
n, gates = workloads.build(name)
qx.run(gates, n, mode, download=False).device["store"].close()
nat.profile_enable(True); nat.profile_reset()
rep = qx.run(gates, n, mode, download=False); rep.device["store"].close()
for k, v in nat.profile_read().items():
    if v["launches"]:
        print(f"{name} {mode} {k:16s} {v['launches']:5d} launches {v['ms']:10.3f} ms  {v['alg_bytes'] / max(v['ms'], 1e-9) / 1e6:9.1f} GB/s")
print(rep.device)
