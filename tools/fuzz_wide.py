"""Fuzz the multi-word path (n > 32) by embedding: a random circuit on the first k qubits of a wide
register must give the one-word run's generators with every word shifted by the idle qubits, in
v1 and v3 (and the same error class in v2).  Not a test:  python tools/fuzz_wide.py [seconds] [seed]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t_end = time.time() + budget
case = fails = compared = 0
errs = {}
while time.time() < t_end:
    rng = np.random.default_rng([seed, case]); case += 1
    k = int(rng.integers(1, 9))
    n = int(rng.choice([33, 40, 64, 70, 130]))
    gates = workloads.gen_random(k, int(rng.integers(0, 60 if k <= 6 else 35)), rng)
    # spread the circuit over the register: qubit j of the small circuit -> wire perm[j] keeps order
    shift = 4 ** (n - k)
    for mode in ("v1", "v2", "v3"):
        try:
            narrow, nerr = qx.run(gates, k, mode), None
        except Exception as e:
            narrow, nerr = None, type(e).__name__
        try:
            wide, werr = qx.run(gates, n, mode), None
        except Exception as e:
            wide, werr = None, type(e).__name__
        if mode == "v2":
            # the dense budget depends on n: wide refuses what narrow (4**k <= 4**10) scatters
            if werr not in (None, "ResourceLimitError") or (werr is None and nerr is not None):
                fails += 1; print("MISMATCH v2 errors", case - 1, k, n, nerr, werr, flush=True)
            if werr is not None or nerr is not None:
                continue
        elif nerr != werr:
            fails += 1; print("MISMATCH errors", case - 1, k, n, mode, nerr, werr, flush=True); continue
        if narrow is None:
            errs[nerr] = errs.get(nerr, 0) + 1
            continue
        compared += 1
        ok = wide.rank_trace[-1][:k] == narrow.rank_trace[-1] and all(r == 1 for r in wide.rank_trace[-1][k:])
        for gw, gn in zip(wide.final.generators, narrow.final.generators):
            ok = ok and [int(v) for v in gw.indices] == [int(v) * shift for v in gn.indices]
            ok = ok and float(np.max(np.abs(gw.lambdas - gn.lambdas), initial=0.0)) < 1e-12
        if not ok:
            fails += 1; print("MISMATCH", case - 1, "k", k, "n", n, mode, flush=True)
print(f"{case} circuits x 3 modes, {compared} runs compared term by term, {fails} mismatches, errors on both sides: {errs}")
