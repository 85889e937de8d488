"""Shared helpers of the -m gpu parity tests (they call the product through its public API,
which goes through the C-ABI in lib/libqimax_b200.so; the oracle is only the checker)."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
import stabsim_port as oracle  # noqa: E402,F401

import paper_2505_03307_b200 as qx  # noqa: E402,F401
from paper_2505_03307_b200.store import DeviceStore  # noqa: E402,F401


def report_gens(report):
    return [(g.lambdas, g.keys()) for g in report.final.generators]


def merge_on_device(n, gens, eps=1e-12):
    """Run qx_merge on a list of (lam, keys) segments; returns the merged segments."""
    with DeviceStore(n, len(gens), 0) as st:
        st.upload(gens)
        ranks = st.merge(eps)
        out = [(l.copy(), k.copy()) for l, k in st.segments()]
    assert ranks == [len(l) for l, _ in out]
    return out


def random_terms(rng, n, count, distinct):
    """count terms whose keys are drawn from `distinct` random words of n qubits."""
    pool = rng.integers(0, 2 ** 63, size=distinct, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=distinct, dtype=np.uint64)
    if n < 32:
        pool = pool % np.uint64(4 ** n)
    keys = pool[rng.integers(0, distinct, size=count)]
    lam = rng.uniform(-1, 1, size=count)
    return lam, keys
