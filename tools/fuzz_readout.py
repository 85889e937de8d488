"""Fuzz the read-out and the kernel-level API against the CPU oracle (not a test):
    python tools/fuzz_readout.py [seconds] [seed]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import stabsim_port as oracle
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads, lut

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t_end = time.time() + budget
case = 0
bad = {}
def note(kind, info):
    bad[kind] = bad.get(kind, 0) + 1
    print("MISMATCH", kind, info, flush=True)

while time.time() < t_end:
    rng = np.random.default_rng([seed, case]); case += 1
    n = int(rng.integers(1, 8))
    gates = workloads.gen_random(n, int(rng.integers(0, 50)), rng)
    # ---- read-out: expansion, prob_z, expectation, Heisenberg route
    final = qx.run(gates, n, "v3").final
    want_final = oracle.run(gates, n, "v3")["final"]
    try:
        wex = oracle.density_expansion(want_final, n)
    except Exception as e:
        wex = type(e).__name__
    try:
        ex = qx.density_expansion(final)
    except Exception as e:
        ex = type(e).__name__
    if isinstance(wex, str) or isinstance(ex, str):
        if wex != ex:
            note("expansion error", (case - 1, n, wex, ex))
        continue
    wd = {int(c): float(v) for c, v in zip(*wex)}
    # v3 coefficients may differ from the oracle's in the last bit, so words whose
    # coefficient cancels to rounding residue may be present on one side only: compare values
    for k in set(wd) | set(ex.coeffs):
        if abs(ex.coeffs.get(k, 0.0) - wd.get(k, 0.0)) > 1e-10:
            note("expansion", (case - 1, n, k))
            break
    # the read-out kernels alone, on the oracle's generators: word sets must be identical
    ex2 = qx.density_expansion(qx.GeneratorSet(n, [qx.SimpleGenerator(n, l, i) for l, i in want_final]))
    if set(ex2.coeffs) != set(wd) or any(abs(ex2.coeffs[k] - v) > 1e-12 for k, v in wd.items()):
        note("expansion kernel", (case - 1, n))
    for k in range(n):
        if abs(qx.prob_z(final, k, ex)[0] - oracle.prob_z(want_final, n, k, wex)[0]) > 1e-10:
            note("prob_z", (case - 1, n, k))
    words = [int(v) for v in rng.integers(0, 4 ** n, size=6)]
    hz = qx.expectation_heisenberg(gates, n, words, mode=str(rng.choice(["v1", "v3"])))
    for wv, h in zip(words, hz):
        if abs(h - oracle.expectation(want_final, n, wv, wex)) > 1e-10 or abs(qx.expectation(final, wv, ex) - h) > 1e-10:
            note("expectation", (case - 1, n, wv))
    # the same observables above 32 qubits (multi-word keys): the circuit on the first n of nw qubits,
    # Z or I on the idle ones (expectation 1 there)
    if case % 4 == 0:
        nw = n + int(rng.integers(33, 90))
        tail = sum(3 * 4 ** (nw - 1 - j) for j in range(n, nw) if rng.random() < 0.2)
        hw = qx.expectation_heisenberg(gates, nw, [wv * 4 ** (nw - n) + tail for wv in words], mode="v1")
        if np.max(np.abs(hw - hz)) > 1e-10:
            note("wide heisenberg", (case - 1, n, nw))
    # ---- kernel-level: random generator with duplicates through apply_1q / apply_cx / canonicalize
    terms = int(rng.integers(1, 40))
    idx = rng.integers(0, 4 ** n, size=terms)
    lam = rng.uniform(-1, 1, size=terms)
    g = qx.SimpleGenerator(n, lam, idx)
    eps = float(rng.choice([1e-12, 1e-3, 0.0]))
    got = qx.canonicalize(g, eps)
    wl, wi = oracle.merge(lam, idx.astype(np.uint64), eps)
    if not (np.array_equal(got.keys(), wi) and np.array_equal(got.lambdas, wl)):
        note("canonicalize", (case - 1, n, eps))
    gate = str(rng.choice(["H", "S", "X", "SX", "RX", "RY", "RZ"]))
    theta = float(rng.choice([0.0, np.pi / 2, np.pi, rng.uniform(0, 6.3)]))
    q = int(rng.integers(0, n))
    got = qx.apply_1q(g, gate, q, theta, eps)
    wl, wi = oracle.conj_1q_v1(lam, idx.astype(np.uint64), n, q, oracle.axis_map(gate, theta), eps)
    if not (np.array_equal(got.keys(), wi) and np.max(np.abs(got.lambdas - wl), initial=0.0) < 1e-12):
        note("apply_1q", (case - 1, n, gate, theta, eps))
    if n >= 2:
        c, t = (int(v) for v in rng.choice(n, size=2, replace=False))
        got = qx.apply_cx(g, c, t)
        wl, wi = oracle.conj_cx(lam, idx.astype(np.uint64), n, c, t)
        if not (np.array_equal(got.keys(), wi) and np.array_equal(got.lambdas, wl)):
            note("apply_cx", (case - 1, n, c, t))
print(f"{case} cases, mismatches: {bad}")
