"""Micro-benchmark of the sort pass: N random terms of n qubits, qx_sort timed per kernel class."""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_03307_b200 import _native as nat
from paper_2505_03307_b200.store import DeviceStore

ap = argparse.ArgumentParser()
ap.add_argument("--terms", type=int, default=100_000_000)
ap.add_argument("--qubits", type=int, default=16)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--pattern", default="random", choices=("random", "const", "sorted", "few"))
args = ap.parse_args()
rng = np.random.default_rng(1)
keys = rng.integers(0, 4 ** args.qubits, size=args.terms, dtype=np.uint64)
if args.pattern == "const":
    keys[:] = 7                      # one bucket: the scatter degenerates to a sequential copy
elif args.pattern == "sorted":
    keys.sort()
elif args.pattern == "few":
    keys = (keys % np.uint64(16)) * np.uint64(0x11111111 & (4 ** args.qubits - 1))   # 16 buckets per pass
lam = rng.uniform(-1, 1, size=args.terms)
with DeviceStore(args.qubits, 1, args.terms + 16) as st:
    st.upload([(lam, keys)])
    st.sort()
    st.synchronize()
    nat.profile_enable(True)
    nat.profile_reset()
    for _ in range(args.reps):
        st.sort()
    st.synchronize()
    prof = nat.profile_read()
    p = prof["sort_pass"]
    print(f"variant={os.environ.get('QX_SORT_VARIANT', '0')} terms={args.terms} n={args.qubits}: "
          f"pass {p['ms'] / p['launches']:.3f} ms x{p['launches'] // args.reps} "
          f"= {p['alg_bytes'] / p['ms'] / 1e6:.0f} GB/s; hist {prof['sort_hist']['ms'] / args.reps:.3f} ms", flush=True)
    print("   pattern", args.pattern)
