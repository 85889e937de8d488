"""Where the time of a one-launch run goes (tools/program_times.py [workload ...]): host phases by
perf_counter, the circuit kernel by CUDA events (profile class small_merge)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads, engine, _native as nat
from paper_2505_03307_b200.store import DeviceStore

for name in sys.argv[1:] or ["c1_4q_clifford_t", "c2_10q_near_clifford", "c3_16q_clifford", "c5_32q_clifford_t"]:
    n, gates = workloads.build(name)
    for mode in ("v1", "v3"):
        m = engine.Mode.coerce(mode)
        for _ in range(3):
            qx.run(gates, n, mode)
        plan = engine._plan_for(gates, n, m)
        prog = plan._programs[(m, 0)]
        best = {}
        for _ in range(20):
            t = [time.perf_counter()]
            st = DeviceStore(n, n, 0, 0); t.append(time.perf_counter())
            t.append(time.perf_counter())
            fitted, rows, _, segs = st.run_program(prog, 1e-12, init_qubits=list(range(n)), to_host=True); t.append(time.perf_counter())
            t.append(time.perf_counter())
            st.close(); t.append(time.perf_counter())
            t0 = time.perf_counter(); qx.run(gates, n, mode); t.append(time.perf_counter() - t0)
            for k, v in zip(("create", "init_z", "run_program", "download", "close"), np.diff(t[:6])):
                best[k] = min(best.get(k, 1e9), v)
            best["run()"] = min(best.get("run()", 1e9), t[6])
        nat.profile_enable(True); nat.profile_reset()
        st = DeviceStore(n, n, 0, 0); st.run_program(prog, 1e-12, init_qubits=list(range(n)), to_host=True); st.close()
        prof = nat.profile_read()["small_merge"]; nat.profile_enable(False)
        print(f"{name:22s} {mode}: " + " ".join(f"{k}={v*1e3:.3f}" for k, v in best.items()) +
              f"  kernel={prof['ms']:.3f} ms  steps={prog.steps}", flush=True)
