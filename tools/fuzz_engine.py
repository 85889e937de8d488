"""Fuzz the public API against the CPU oracle: random circuits over every gate, n in [1, 11] plus the
one-word boundary n = 31, 32, all three modes, a few eps values.  Not a test (minutes of oracle time):
    python tools/fuzz_engine.py [seconds] [seed]"""
import math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import stabsim_port as oracle
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t_end = time.time() + budget
case = fails = 0
kinds = {}
while time.time() < t_end:
    rng = np.random.default_rng([seed, case])
    case += 1
    kind = int(rng.integers(0, 10))
    if kind == 0:
        n = int(rng.choice([31, 32]))
        gates = workloads.near_clifford(n, int(rng.integers(20, 200)), int(rng.integers(0, 6)), int(rng.integers(0, 1 << 30)))
    elif kind == 1:
        # mid-size near-Clifford: Clifford base, a few rotations of any axis (quarter turns included)
        n = int(rng.integers(12, 31))
        gates = workloads.gen_random(n, int(rng.integers(50, 300)), rng, gates=("H", "S", "X", "SX", "CX"))
        for _ in range(int(rng.integers(0, 9))):
            theta = float(rng.choice([math.pi / 4, math.pi / 2, math.pi, -math.pi / 2, rng.uniform(0, 6.3)]))
            rot = qx.Instruction(str(rng.choice(["RX", "RY", "RZ"])), (int(rng.integers(0, n)),), theta)
            gates.insert(int(rng.integers(0, len(gates) + 1)), rot)
    else:
        n = int(rng.integers(1, 12))
        m = int(rng.integers(0, 70 if n <= 8 else 40))
        gates = workloads.gen_random(n, m, rng)
    eps = float(rng.choice([1e-12, 1e-12, 1e-12, 1e-9, 1e-6, 0.0]))
    for mode in ("v1", "v2", "v3"):
        try:
            want = oracle.run(gates, n, mode, eps)
            werr = None
        except Exception as e:                      # collapse / resource limits: same class expected
            want, werr = None, type(e).__name__
        try:
            got = qx.run(gates, n, mode, eps)
            gerr = None
        except Exception as e:
            got, gerr = None, type(e).__name__
        ok = werr == gerr
        if ok and want is not None:
            ok = got.rank_trace == want["rank_trace"]
            for g, (lam, idx) in zip(got.final.generators, want["final"]):
                ok = ok and np.array_equal(g.keys(), idx) and np.max(np.abs(g.lambdas - lam), initial=0.0) < 1e-10
        if not ok:
            fails += 1
            kinds[(mode, eps, werr, gerr)] = kinds.get((mode, eps, werr, gerr), 0) + 1
            print(f"MISMATCH case {case - 1} seed {seed} n={n} m={len(gates)} mode={mode} eps={eps} oracle={werr} gpu={gerr}", flush=True)
print(f"{case} circuits x 3 modes, {fails} mismatches", kinds)
