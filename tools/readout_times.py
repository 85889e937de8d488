"""Read-out (density expansion, prob_z, expectation) wall times on the configs the reference can read out."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads
for name in ("c1_4q_clifford_t", "c2_10q_near_clifford"):
    n, gates = workloads.build(name)
    rep = qx.run(gates, n, "v3")
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        ex = qx.density_expansion(rep.final)
        p = [qx.prob_z(rep.final, k, ex) for k in range(n)]
        best = min(best, time.perf_counter() - t0)
    print(f"{name}: expansion of {len(ex.codes)} words + prob_z of {n} qubits: {1e3 * best:.2f} ms; p0 = {[round(v[0], 4) for v in p][:4]}")
