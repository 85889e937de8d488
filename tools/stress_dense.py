"""Randomised parity stress of the grouped operator step: circuits whose operators mix generic
rotations, single-axis rotations, Clifford gates and identity columns on 9-12 qubits, large enough
for the grouped path (raw fan-out well above the small-merge limit), against the CPU oracle."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import stabsim_port as oracle
import paper_2505_03307_b200 as qx

def circuit(rng, n, heavy):
    gates = []
    for layer in range(3 if n <= 8 else 2):
        for q in range(n):
            kind = rng.integers(0, 6) if rng.uniform() > heavy else 0
            if kind <= 2:                                   # generic rotation: full mixing
                for g in ("RX", "RY", "RZ"):
                    gates.append(qx.Instruction(g, (q,), float(rng.uniform(0, 6.28))))
            elif kind == 3:                                 # one axis: partial mixing
                gates.append(qx.Instruction(str(rng.choice(["RX", "RY", "RZ"])), (q,), float(rng.uniform(0, 6.28))))
            elif kind == 4:                                 # Clifford
                gates.append(qx.Instruction(str(rng.choice(["H", "S", "X", "SX"])), (q,)))
        order = rng.permutation(n)                          # an entangling chain over a random qubit order
        for a, b in zip(order[:-1], order[1:]):
            if rng.uniform() < 0.85:
                gates.append(qx.Instruction("CX", (int(a), int(b))))
        if rng.integers(0, 2):
            gates.append(qx.Instruction("H", (int(rng.integers(n)),)))
    return gates

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
worst, t0, dense = 0.0, time.time(), 0
for case in range(cases):
    rng = np.random.default_rng([77, case])
    n = int(rng.integers(8, 12))
    gates = circuit(rng, n, float(rng.choice([0.0, 0.5, 0.8])))
    want = oracle.run(gates, n, "v3")
    got = qx.run(gates, n, "v3")
    assert got.rank_trace == want["rank_trace"], (case, "rank trace")
    for g, (lam, idx) in zip(got.final.generators, want["final"]):
        assert np.array_equal(g.keys(), idx), (case, "keys")
        if len(lam):
            worst = max(worst, float(np.max(np.abs(g.lambdas - lam))))
    dense += 1
    print(f"case {case}: n={n} gates={len(gates)} max rank {max(map(max, want['rank_trace']))} dev {worst:.1e} ok", flush=True)
print(f"{dense} circuits, worst coefficient deviation {worst:.3e}, {time.time() - t0:.0f} s")
assert worst < 1e-10
