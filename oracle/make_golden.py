"""Generate tests/golden/* by running the UNMODIFIED reference in this container.

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py [--big]

Imports ``stabsim`` read-only from /root/reference/pkg/src (it cannot travel to
the GPU box, so its outputs are committed as fixtures instead).  Floats are
stored as ``float.hex()`` strings or raw float64 arrays, so fixtures are
bit-exact images of what the reference computed here (Python 3.12, numpy 2.3).

Fixtures written:
  circuits.json    gate lists of the BASELINE workloads + campaign circuits
  units.json       kernel-level vectors: apply_cx, _apply_1q_terms, canonicalize,
                   sub+flatten, create_lut_1q, density_expansion, prob_z, expectation
  campaign.json    small random circuits, all three modes, full outputs + readout
  configs.npz      full final generators of C1, C2, C3, C5 and small C4 ladder points
  digests.json     rank/hash/moment digests of the large C4 ladder points (--big)
"""

from __future__ import annotations

import argparse
import base64
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True

import stabsim                                   # noqa: E402  (the reference)
from stabsim import circuit as rc                # noqa: E402
from stabsim import engine as reng               # noqa: E402
from stabsim import lut as rlut                  # noqa: E402
from stabsim import measure as rmeasure          # noqa: E402
from stabsim import stabilizer as rstab          # noqa: E402

from paper_2505_03307_b200 import workloads      # noqa: E402  (only to name the same circuits)


def hx(v):
    return float(v).hex()


def gates_json(insts):
    return [[g.gate, list(g.wires), hx(g.theta)] for g in insts]


def to_ref(insts):
    return [rc.Instruction(g.gate, tuple(g.wires), g.theta) for g in insts]


def gen_json(g):
    return {"lam": [hx(v) for v in g.lambdas], "idx": [int(v) for v in g.indices]}


def mix64(keys):
    """splitmix64 finaliser -> weights in [-1, 1); shared with tests/golden_util.py."""
    z = keys.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


CHUNKS = 1024          # per-generator chunk moments: a coefficient error is localised to rank/1024 terms


def chunk_moments(lam, keys, chunks=CHUNKS):
    """Sum of lambda and of lambda * mix64(key) over `chunks` contiguous ranges of the canonical
    order (range c = [c*r//chunks, (c+1)*r//chunks)), as base64 of little-endian float64; shared
    with tests/golden_util.py.  Any single coefficient off by more than the test's tolerance shows
    up in its chunk (both moments would have to cancel to hide it)."""
    r = len(lam)
    bounds = (np.arange(chunks + 1, dtype=np.int64) * r) // chunks
    w = lam * mix64(keys)
    cs = np.concatenate([[0.0], np.cumsum(lam)])
    cw = np.concatenate([[0.0], np.cumsum(w)])
    # chunk sums by direct summation (not differences of running sums: those would carry the
    # rounding of the whole prefix)
    s = np.array([lam[bounds[c]:bounds[c + 1]].sum() for c in range(chunks)])
    p = np.array([w[bounds[c]:bounds[c + 1]].sum() for c in range(chunks)])
    del cs, cw
    return {"count": chunks, "sum": base64.b64encode(s.astype("<f8").tobytes()).decode(),
            "proj": base64.b64encode(p.astype("<f8").tobytes()).decode()}


def digest(g):
    idx = np.asarray(g.indices)
    keys = idx.astype(np.uint64) if idx.dtype != object else np.array([int(v) for v in idx], dtype=np.uint64)
    lam = np.asarray(g.lambdas, dtype=np.float64)
    step = max(1, len(keys) // 64)
    extra = {"chunks": chunk_moments(lam, keys)} if len(keys) >= 4 * CHUNKS else {}
    return {
        **extra,
        "rank": int(len(keys)),
        "sha256": hashlib.sha256(keys.tobytes()).hexdigest(),
        "sum": hx(lam.sum()), "sum_sq": hx(np.dot(lam, lam)), "sum_abs": hx(np.abs(lam).sum()),
        "proj": hx(np.dot(lam, mix64(keys))),
        "sample_idx": [int(v) for v in keys[::step]],
        "sample_lam": [hx(v) for v in lam[::step]],
    }


def count_updates(insts, n):
    """Term-gate updates in reference v1: ranks before each gate, summed."""
    total = 0
    orig_1q, orig_cx = reng._apply_1q_terms, reng.apply_cx

    def w1(g, inst, eps):
        nonlocal total
        total += g.rank
        return orig_1q(g, inst, eps)

    def wcx(g, c, t):
        nonlocal total
        total += g.rank
        return orig_cx(g, c, t)

    reng._apply_1q_terms, reng.apply_cx = w1, wcx
    try:
        reng.run(insts, n, "v1")
    finally:
        reng._apply_1q_terms, reng.apply_cx = orig_1q, orig_cx
    return total


def make_circuits():
    out = {}
    for name in ("c1_4q_clifford_t", "c2_10q_near_clifford", "c3_16q_clifford",
                 "c4_xyz_8_4", "c4_xyz_12_2", "c4_xyz_16_2", "c5_32q_clifford_t"):
        n, mine = workloads.build(name)
        out[name] = {"n": n, "gates": gates_json(mine)}
    # the same families straight from the reference's generators, to pin workloads.py
    ref = {
        "ghz_5": (5, rc.gen_ghz(5)),
        "graph_ring_6": (6, rc.gen_graph(6, rc.ring_edges(6))),
        "xyz_4_4_2_seed1": (4, rc.gen_xyz_chain(4, 4, 2, 1)),
        "xyz_16_2_1_seed4": (16, rc.gen_xyz_chain(16, 2, 1, 4)),
        "random_5_40_seed9": (5, rc.gen_random(5, 40, 9)),
        "random_clifford_16_984_seed3": (16, rc.gen_random(16, 984, np.random.default_rng(3),
                                                            gates=("H", "S", "X", "SX", "CX"))),
    }
    out["_reference_generators"] = {k: {"n": n, "gates": gates_json(v)} for k, (n, v) in ref.items()}
    return out


def make_units():
    rng = np.random.default_rng(20250503)
    units = {"apply_cx": [], "apply_1q": [], "canonicalize": [], "operator": [], "lut": [], "readout": []}
    # --- apply_cx on random term lists, incl. n = 31/32 (int64 / object paths)
    for n in (2, 3, 5, 16, 31, 32):
        for _ in range(4):
            k = int(rng.integers(1, 40))
            idx = [((int(rng.integers(0, 2 ** 32)) << 32) | int(rng.integers(0, 2 ** 32))) % 4 ** n for _ in range(k)]
            idx = sorted(set(idx))
            lam = rng.uniform(-1, 1, size=len(idx))
            c, t = (int(v) for v in rng.choice(n, size=2, replace=False))
            g = rstab.SimpleGenerator(n, lam, idx)
            o = rstab.apply_cx(g, c, t)
            units["apply_cx"].append({"n": n, "c": c, "t": t, "in": gen_json(g), "out": gen_json(o)})
    # --- v1 single-gate conjugation incl. merge (engine._apply_1q_terms)
    for gate in ("H", "S", "X", "SX", "RX", "RY", "RZ"):
        for n in (1, 3, 6, 32):
            for theta in ((0.0,) if gate in ("H", "S", "X", "SX") else (0.3, math.pi / 4, math.pi / 2, math.pi, 5.1)):
                k = int(rng.integers(1, 60))
                cap = 4 ** min(n, 4)
                idx = sorted({int(v) for v in rng.integers(0, cap, size=k)})
                if n > 4:
                    sh = 4 ** int(rng.integers(0, n - 3))
                    idx = [v * sh for v in idx]
                lam = rng.uniform(-1, 1, size=len(idx))
                q = int(rng.integers(0, n))
                g = rstab.SimpleGenerator(n, lam, idx)
                inst = rc.Instruction(gate, (q,), theta)
                o = reng._apply_1q_terms(g, inst, 1e-12)
                units["apply_1q"].append({"n": n, "gate": gate, "q": q, "theta": hx(theta),
                                          "in": gen_json(g), "out": gen_json(o)})
    # --- canonicalize
    for n, k in ((1, 5), (2, 40), (3, 200), (8, 500), (32, 300)):
        idx = [int(v) for v in rng.integers(0, min(4 ** n, 97), size=k)]
        lam = rng.uniform(-1, 1, size=k)
        lam[rng.integers(0, k, size=k // 5)] *= 1e-13           # some sums fall under eps
        g = rstab.SimpleGenerator(n, lam, idx)
        o = rstab.canonicalize(g, 1e-12)
        units["canonicalize"].append({"n": n, "in": gen_json(g), "out": gen_json(o)})
    # exact cancellation and the reference's KATs (tests/test_stabilizer.py:271-292)
    for n, lam, idx in ((1, [1.0, 1.0], [3, 3]), (1, [1e-15], [2]), (2, [1.0, 2.0, 3.0], [9, 2, 5]),
                        (2, [0.5, -0.5, 1.0], [7, 7, 1])):
        g = rstab.SimpleGenerator(n, lam, idx)
        units["canonicalize"].append({"n": n, "in": gen_json(g), "out": gen_json(rstab.canonicalize(g, 1e-12))})
    # --- operator (sub + flatten), raw and merged, ragged layout
    for n in (1, 2, 3, 4, 6):
        for case in range(4):
            insts = rc.gen_random(n, int(rng.integers(1, 12)), rng, gates=("H", "S", "X", "SX", "RX", "RY", "RZ"))
            part = rc.divide_instruction(insts, n)
            block = rlut.create_lut_1q(part)[0]
            k = int(rng.integers(1, 12))
            idx = sorted({int(v) for v in rng.integers(0, 4 ** n, size=k)})
            lam = rng.uniform(-1, 1, size=len(idx))
            g = rstab.SimpleGenerator(n, lam, idx)
            cg = rstab.sub(g, block, "ragged")
            raw = rstab.flatten(cg, canonical=False)
            merged = rstab.flatten(cg, 1e-12)
            units["operator"].append({"n": n, "gates": gates_json(insts),
                                      "block": [hx(v) for v in block.ravel()],
                                      "in": gen_json(g), "raw": gen_json(raw), "out": gen_json(merged)})
    # --- LUT tensor of a mixed circuit (bit-exact pin for lut.create_lut_1q)
    for n, m, seed in ((3, 25, 12), (5, 80, 13)):
        insts = rc.gen_random(n, m, seed)
        part = rc.divide_instruction(insts, n)
        lut = rlut.create_lut_1q(part)
        units["lut"].append({"n": n, "gates": gates_json(insts), "shape": list(lut.shape),
                             "lut": [hx(v) for v in lut.ravel()], "order": list(part.order)})
    # --- readout: full expansion, prob_z, expectation
    for n, m, seed in ((2, 10, 1), (3, 20, 2), (4, 30, 3), (5, 40, 4), (6, 40, 5)):
        insts = rc.gen_random(n, m, seed)
        rep = reng.run(insts, n, "v3")
        ex = rmeasure.density_expansion(rep.final)
        codes = sorted(ex.coeffs)
        words = [int(v) for v in np.random.default_rng(seed).integers(0, 4 ** n, size=12)]
        units["readout"].append({
            "n": n, "gates": gates_json(insts),
            "final": [gen_json(g) for g in rep.final.generators],
            "codes": codes, "coeffs": [hx(ex.coeffs[c]) for c in codes],
            "prob_z": [[hx(p) for p in rmeasure.prob_z(rep.final, k, ex)] for k in range(n)],
            "words": words, "expect": [hx(rmeasure.expectation(rep.final, w, ex)) for w in words],
        })
    return units


def make_campaign(cases=40):
    out = []
    for case in range(cases):
        rng = np.random.default_rng([2024, case])        # tests/test_acceptance.py:25-48
        n = int(rng.integers(2, 6))
        m = int(rng.integers(1, 61))
        insts = rc.gen_random(n, m, rng)
        entry = {"case": case, "n": n, "gates": gates_json(insts), "modes": {}}
        for mode in ("v1", "v2", "v3"):
            rep = reng.run(insts, n, mode)
            entry["modes"][mode] = {
                "final": [gen_json(g) for g in rep.final.generators],
                "rank_trace": rep.rank_trace, "order": rep.order, "k": rep.k, "k_prime": rep.k_prime,
                "counters": rep.counters,
            }
        ex = rmeasure.density_expansion(reng.run(insts, n, "v3").final)
        gs = reng.run(insts, n, "v3").final
        entry["prob_z"] = [[hx(p) for p in rmeasure.prob_z(gs, k, ex)] for k in range(n)]
        entry["updates"] = count_updates(insts, n)
        out.append(entry)
    return out


def pack_report(store, name, mode, rep, updates=None):
    gens = rep.final.generators
    off = np.zeros(len(gens) + 1, dtype=np.int64)
    off[1:] = np.cumsum([g.rank for g in gens])
    store[f"{name}/{mode}/offsets"] = off
    store[f"{name}/{mode}/keys"] = np.array([int(v) for g in gens for v in g.indices], dtype=np.uint64)
    store[f"{name}/{mode}/lam"] = np.concatenate([g.lambdas for g in gens])
    trace = np.array(rep.rank_trace, dtype=np.int64)
    store[f"{name}/{mode}/rank_trace"] = trace
    store[f"{name}/{mode}/meta"] = np.array([rep.k, rep.k_prime, -1 if updates is None else updates], dtype=np.int64)


def make_configs(big):
    store, digests = {}, {}
    plan = [
        ("c1_4q_clifford_t", ("v1", "v2", "v3")),
        ("c2_10q_near_clifford", ("v1", "v2", "v3")),
        ("c3_16q_clifford", ("v1", "v2", "v3")),
        ("c4_xyz_8_4", ("v1",)),
        ("c5_32q_clifford_t", ("v1", "v3") if big else ("v1",)),
    ]
    for name, modes in plan:
        n, mine = workloads.build(name)
        insts = to_ref(mine)
        t0 = time.perf_counter()
        upd = count_updates(insts, n)
        for mode in modes:
            rep = reng.run(insts, n, mode)
            if name == "c4_xyz_8_4":
                digests[f"{name}/{mode}"] = {"n": n, "updates": upd, "trace_last": rep.rank_trace[-1],
                                             "max_rank": rep.max_rank,
                                             "gens": [digest(g) for g in rep.final.generators]}
            else:
                pack_report(store, name, mode, rep, upd)
        print(f"{name}: {time.perf_counter() - t0:.1f}s updates={upd}", flush=True)
    # readout of C1 (all 256 words) and C2 (prob_z) through the reference expansion
    n, mine = workloads.build("c1_4q_clifford_t")
    rep = reng.run(to_ref(mine), n, "v3")
    ex = rmeasure.density_expansion(rep.final)
    store["c1_4q_clifford_t/expect_all"] = np.array([rmeasure.expectation(rep.final, w, ex) for w in range(4 ** n)])
    store["c1_4q_clifford_t/prob_z"] = np.array([rmeasure.prob_z(rep.final, k, ex) for k in range(n)])
    n, mine = workloads.build("c2_10q_near_clifford")
    rep = reng.run(to_ref(mine), n, "v3")
    ex = rmeasure.density_expansion(rep.final)
    store["c2_10q_near_clifford/prob_z"] = np.array([rmeasure.prob_z(rep.final, k, ex) for k in range(n)])
    codes = np.array(sorted(ex.coeffs), dtype=np.uint64)
    store["c2_10q_near_clifford/exp_codes"] = codes
    store["c2_10q_near_clifford/exp_coeffs"] = np.array([ex.coeffs[int(c)] for c in codes])
    # ladder digests (v3; v1 where it is cheap)
    ladder = [("c4_xyz_8_4", ("v3",)), ("c4_xyz_12_2", ("v1", "v3"))]
    if big:
        ladder += [("c4_xyz_10_3", ("v3",)), ("c4_xyz_14_2", ("v3",))]
    for name, modes in ladder:
        n, mine = workloads.build(name)
        insts = to_ref(mine)
        for mode in modes:
            t0 = time.perf_counter()
            rep = reng.run(insts, n, mode)
            digests[f"{name}/{mode}"] = {"n": n, "trace_last": rep.rank_trace[-1], "max_rank": rep.max_rank,
                                         "gens": [digest(g) for g in rep.final.generators]}
            print(f"{name}/{mode}: {time.perf_counter() - t0:.1f}s ranks={rep.rank_trace[-1]}", flush=True)
    return store, digests


def make_ladder_point(name, mode="v3"):
    """One more ladder digest, merged into digests.json (used for the bench workload itself,
    c4_xyz_16_2: 1.25e8 terms, ~3 minutes and ~20 GB for the reference)."""
    n, mine = workloads.build(name)
    t0 = time.perf_counter()
    rep = reng.run(to_ref(mine), n, mode)
    print(f"{name}/{mode}: reference took {time.perf_counter() - t0:.1f}s ranks={rep.rank_trace[-1]}", flush=True)
    return {f"{name}/{mode}": {"n": n, "trace_last": rep.rank_trace[-1], "max_rank": rep.max_rank,
                               "gens": [digest(g) for g in rep.final.generators]}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also run the minutes-long reference cases")
    ap.add_argument("--ladder", default="", help="only add the digest of this ladder point (e.g. c4_xyz_16_2)")
    ap.add_argument("--only", default="", help="comma list of: circuits,units,campaign,configs")
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))
    os.makedirs(OUT, exist_ok=True)
    meta = {"reference": "stabsim " + stabsim.__version__, "numpy": np.__version__,
            "python": sys.version.split()[0]}

    def dump(name, obj):
        with open(os.path.join(OUT, name), "w") as fh:
            json.dump({"_meta": meta, "data": obj}, fh, separators=(",", ":"))
        print("wrote", name, os.path.getsize(os.path.join(OUT, name)), "bytes", flush=True)

    if args.ladder:
        path = os.path.join(OUT, "digests.json")
        with open(path) as fh:
            old = json.load(fh)["data"]
        old.update(make_ladder_point(args.ladder))
        dump("digests.json", old)
        return
    if not only or "circuits" in only:
        dump("circuits.json", make_circuits())
    if not only or "units" in only:
        dump("units.json", make_units())
    if not only or "campaign" in only:
        dump("campaign.json", make_campaign())
    if not only or "configs" in only:
        store, digests = make_configs(args.big)
        np.savez_compressed(os.path.join(OUT, "configs.npz"), **{k.replace("/", "__"): v for k, v in store.items()})
        print("wrote configs.npz", os.path.getsize(os.path.join(OUT, "configs.npz")), "bytes")
        path = os.path.join(OUT, "digests.json")
        old = {}
        if os.path.exists(path):
            with open(path) as fh:
                old = json.load(fh)["data"]
        old.update(digests)
        dump("digests.json", old)


if __name__ == "__main__":
    main()
