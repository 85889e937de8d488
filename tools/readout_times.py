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

# Heisenberg read-out (north star kernel 4: <0|U^dag W U|0>, one store segment per observable)
def timed(label, gates, n, words, mode="v1"):
    best, vals = 1e9, None
    for _ in range(3):
        t0 = time.perf_counter()
        vals = qx.expectation_heisenberg(gates, n, words, mode)
        best = min(best, time.perf_counter() - t0)
    print(f"{label}: {len(words)} observables, n={n}, {len(gates)} gates: {1e3 * best:.2f} ms; first = {[round(float(v), 4) for v in vals[:3]]}")

n, gates = workloads.build("c1_4q_clifford_t")
timed("c1 all words", gates, n, list(range(4 ** n)))
n, gates = workloads.build("c2_10q_near_clifford")
timed("c2 Z_k", gates, n, [3 * 4 ** (n - 1 - k) for k in range(n)])
n, gates = workloads.build("c5_32q_clifford_t")
timed("c5 Z_k", gates, n, [3 * 4 ** (n - 1 - k) for k in range(n)])
n = 100                                            # multi-word keys (csrc/wide.cu)
gates = qx.gen_ghz(n)
timed("ghz(100) Z_iZ_j + X..X", gates, n, [3 * 4 ** (n - 1 - i) + 3 * 4 ** (n - 1 - i - 1) for i in range(n - 1)] + [(4 ** n - 1) // 3])
m = 10
gates = workloads.gen_xyz_chain(m, 2, 1, 4)
timed("xyz_chain(10,2) on the first 10 of 70 qubits, Z_k", gates, 70, [3 * 4 ** (70 - 1 - k) for k in range(m)], "v3")
