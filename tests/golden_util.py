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
    """Compare one generator against its stored digest: keys bit-exact (sha256), lambdas to tol."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    assert len(keys) == d["rank"], (len(keys), d["rank"])
    assert hashlib.sha256(keys.tobytes()).hexdigest() == d["sha256"]
    step = max(1, len(keys) // 64)
    assert [int(v) for v in keys[::step]] == d["sample_idx"]
    assert np.max(np.abs(lam[::step] - unhex(d["sample_lam"])), initial=0.0) < tol
    scale = max(1.0, np.sqrt(len(keys)))
    assert abs(lam.sum() - float.fromhex(d["sum"])) < tol * scale
    assert abs(np.dot(lam, lam) - float.fromhex(d["sum_sq"])) < tol * scale
    assert abs(np.dot(lam, mix64(keys)) - float.fromhex(d["proj"])) < tol * scale


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
