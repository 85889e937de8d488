"""Loaders for tests/golden/* (written by oracle/make_golden.py from the reference)."""

from __future__ import annotations

import functools
import hashlib
import json
import os

import numpy as np

from paper_2505_03307_b200.circuit import Instruction

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)["data"]


@functools.lru_cache(maxsize=None)
def load_npz():
    return dict(np.load(os.path.join(GOLDEN, "configs.npz")))


def unhex(values):
    return np.array([float.fromhex(v) for v in values], dtype=np.float64)


def gates(rows):
    return [Instruction(g, tuple(w), float.fromhex(t)) for g, w, t in rows]


def gen(entry):
    """(lambdas float64, indices uint64) of a {"lam": [...hex], "idx": [...int]} record."""
    return unhex(entry["lam"]), np.array(entry["idx"], dtype=np.uint64)


def config(name, mode):
    """Per-generator [(lam, keys)], rank trace and (k, k', updates) of a stored config run."""
    z = load_npz()
    pre = f"{name}__{mode}__"
    off = z[pre + "offsets"]
    keys, lam = z[pre + "keys"], z[pre + "lam"]
    gens = [(lam[off[i]:off[i + 1]], keys[off[i]:off[i + 1]]) for i in range(len(off) - 1)]
    return gens, z[pre + "rank_trace"].tolist(), [int(v) for v in z[pre + "meta"]]


def mix64(keys):
    """Same key -> weight hash as oracle/make_golden.py (splitmix64 finaliser)."""
    z = keys.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


def check_digest(d, lam, keys, tol=1e-10):
    """Compare one generator against its stored digest (made from the reference's own run by
    oracle/make_golden.py): keys bit-exact (sha256); coefficients to `tol` ABSOLUTE on strided
    samples, on the three whole-generator moments and -- where the digest has them -- on the sum
    and the hashed projection of each of 1024 contiguous chunks of the canonical order, so a
    single coefficient off by more than tol anywhere fails its chunk.  The sums here and in the
    digest are numpy's over (nearly) the same numbers in the same order; their own rounding is
    1e-16 * sum|lambda| ~ 1e-13, far below tol."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    assert len(keys) == d["rank"], (len(keys), d["rank"])
    assert hashlib.sha256(keys.tobytes()).hexdigest() == d["sha256"]
    step = max(1, len(keys) // 64)
    assert [int(v) for v in keys[::step]] == d["sample_idx"]
    assert np.max(np.abs(lam[::step] - unhex(d["sample_lam"])), initial=0.0) < tol
    weights = mix64(keys)
    assert abs(lam.sum() - float.fromhex(d["sum"])) < tol
    assert abs(np.dot(lam, lam) - float.fromhex(d["sum_sq"])) < tol
    assert abs(np.dot(lam, weights) - float.fromhex(d["proj"])) < tol
    if "chunks" in d:
        import base64

        c = d["chunks"]
        chunks = int(c["count"])
        want_s = np.frombuffer(base64.b64decode(c["sum"]), dtype="<f8")
        want_p = np.frombuffer(base64.b64decode(c["proj"]), dtype="<f8")
        bounds = (np.arange(chunks + 1, dtype=np.int64) * len(lam)) // chunks
        w = lam * weights
        got_s = np.array([lam[bounds[i]:bounds[i + 1]].sum() for i in range(chunks)])
        got_p = np.array([w[bounds[i]:bounds[i + 1]].sum() for i in range(chunks)])
        bad = np.flatnonzero((np.abs(got_s - want_s) >= tol) | (np.abs(got_p - want_p) >= tol))
        assert len(bad) == 0, f"chunks {bad[:8].tolist()} of {chunks} differ (terms {bounds[bad[0]]}..{bounds[bad[0] + 1]})"


def assert_gens_equal(got, want, tol=1e-10, exact=False):
    """Term sets bit-exact after canonical ordering, coefficients within tol (or bitwise)."""
    assert len(got) == len(want)
    for gi, ((gl, gk), (wl, wk)) in enumerate(zip(got, want)):
        gk = np.asarray(gk, dtype=np.uint64)
        wk = np.asarray(wk, dtype=np.uint64)
        assert gk.shape == wk.shape and np.array_equal(gk, wk), f"generator {gi}: key sets differ"
        if exact:
            assert np.array_equal(np.asarray(gl), np.asarray(wl)), f"generator {gi}: lambdas not bitwise equal"
        elif len(wl):
            dev = float(np.max(np.abs(np.asarray(gl) - np.asarray(wl))))
            assert dev < tol, f"generator {gi}: max |dlambda| = {dev:.3e}"
