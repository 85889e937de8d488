"""Fuzz the corners of run(): eps large enough to drop input terms (the merge-after-every-step
schedule, NumericalCollapseError with the reference's generator / step), and caller-supplied
initial generators (unsorted, with duplicates and tiny terms), against the CPU oracle.
Not a test:  python tools/fuzz_eager.py [seconds] [seed]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import stabsim_port as oracle
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t_end = time.time() + budget
case = fails = collapses = 0
while time.time() < t_end:
    rng = np.random.default_rng([seed, case]); case += 1
    n = int(rng.integers(1, 8))
    gates = workloads.gen_random(n, int(rng.integers(0, 40)), rng)
    eps = float(rng.choice([0.05, 0.3, 0.6, 0.8, 1.0, 1.0 + 1e-9, 2.0, 1e-12]))
    initial = None
    if rng.integers(0, 2):
        initial = []
        for _ in range(n):
            size = int(rng.integers(1, 12))
            keys = rng.integers(0, 4 ** n, size=size).astype(np.uint64)      # duplicates likely for small n
            lam = rng.uniform(-1, 1, size=size) * rng.choice([1.0, 1e-13, 1e-6], size=size)
            initial.append((lam, keys))
    for mode in ("v1", "v2", "v3"):
        res = []
        for runner in (lambda: oracle.run(gates, n, mode, eps, initial=initial),
                       lambda: qx.run(gates, n, mode, eps, initial=initial)):
            try:
                res.append(("ok", runner()))
            except Exception as e:
                res.append((type(e).__name__, str(e)))
        (wk, want), (gk, got) = res
        ok = wk == gk
        if ok and wk == "NumericalCollapseError":
            collapses += 1
            ok = want == got                                     # same generator, same step in the message
        elif ok and wk == "ok":
            ok = got.rank_trace == want["rank_trace"]
            for g, (lam, idx) in zip(got.final.generators, want["final"]):
                ok = ok and np.array_equal(g.keys(), idx) and float(np.max(np.abs(g.lambdas - lam), initial=0.0)) < 1e-10
        if not ok:
            fails += 1
            print("MISMATCH", case - 1, "n", n, "gates", len(gates), mode, "eps", eps, "initial" if initial else "init_z",
                  wk, gk, (want if wk != "ok" else ""), (got if gk != "ok" else ""), flush=True)
print(f"{case} circuits x 3 modes, {collapses} collapses compared by message, {fails} mismatches")
