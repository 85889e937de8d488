"""Micro-benchmark of the v1 gate kernels at scale: N random terms of n qubits in one generator;
qx_apply_clifford (a 15-CX ladder + 1q Cliffords), qx_apply_split (RZ on a middle qubit) and the
merge behind it, timed per kernel class with the library's CUDA-event instrumentation."""
import argparse, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_03307_b200 import _native as nat, lut
from paper_2505_03307_b200.stabilizer import split_tables
from paper_2505_03307_b200.store import DeviceStore

ap = argparse.ArgumentParser()
ap.add_argument("--terms", type=int, default=60_000_000)
ap.add_argument("--qubits", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
n = args.qubits
rng = np.random.default_rng(3)
keys = np.unique(rng.integers(0, 4 ** n, size=args.terms, dtype=np.uint64))
lam = rng.uniform(-1, 1, size=len(keys))
prog = [lut.cx_op(n, q, q + 1) for q in range(n - 1)] + [lut.perm_op(n, q, lut.FIXED_PERMS["H"]) for q in range(0, n, 3)]
prog = np.array(prog, dtype=lut.op_dtype(n))
tabs = split_tables(lut.gate_branch_block("RZ", 0.7))
for rep in range(args.reps + 1):
    with DeviceStore(n, 1, 2 * len(keys) + 16) as st:
        st.upload([(lam, keys)])
        st.synchronize()
        if rep == 1:
            nat.profile_enable(True)
            nat.profile_reset()
        st.apply_clifford(prog)
        st.sort()
        st.apply_split(n // 2, *tabs)
        st.merge(1e-12)
        st.synchronize()
prof = nat.profile_read()
print(f"{len(keys)} terms, n={n}, {len(prog)} Clifford ops per run")
for k, v in prof.items():
    if v["launches"]:
        print(f"  {k:14s} {v['launches']:4d} launches  {v['ms'] / v['launches']:8.3f} ms each  "
              f"{v['alg_bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f} GB/s by algorithmic bytes")
