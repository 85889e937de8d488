"""Fuzz the result download: streamed ranges, 32-bit and packed 16-bit key forms against the plain
download of the resident store, on ansatz circuits of varying size with a random Clifford tail.
Not a test:  python tools/fuzz_download.py [seconds] [seed]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t_end = time.time() + budget
case = fails = 0
while time.time() < t_end:
    rng = np.random.default_rng([seed, case]); case += 1
    n = int(rng.integers(9, 16))
    layers = 2 if n >= 11 else int(rng.integers(2, 4))
    gates = workloads.gen_xyz_chain(n, layers, 1, int(rng.integers(0, 1 << 30)))
    if rng.integers(0, 2):
        gates = gates + workloads.gen_random(n, int(rng.integers(1, 30)), rng, gates=("H", "S", "X", "SX", "CX"))
    if rng.integers(0, 3) == 0:
        gates = gates[: int(rng.integers(len(gates) // 2, len(gates)))]
    rep = qx.run(gates, n, "v3", download=False)
    st = rep.device["store"]
    try:
        plain = [(l.copy(), k.copy()) for l, k in st.segments()]
    finally:
        st.close()
    for pinned in (True, False):
        got = qx.run(gates, n, "v3", pinned=pinned)
        ok = got.rank_trace == rep.rank_trace
        for g, (l, k) in zip(got.final.generators, plain):
            ok = ok and np.array_equal(g.keys(), k) and np.array_equal(g.lambdas, l)
        if not ok:
            fails += 1
            print("MISMATCH", case - 1, n, layers, len(gates), "pinned" if pinned else "pageable", sum(rep.rank_trace[-1]), flush=True)
    print(f"case {case - 1}: n={n} gates={len(gates)} terms={sum(rep.rank_trace[-1])} {got.device.get('streamed_ranges')}", flush=True)
print(f"{case} circuits, {fails} mismatches")
