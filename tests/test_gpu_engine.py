"""Circuit-level parity on the GPU: engine.run in every mode against fixtures produced by the
reference (tests/golden) and against the CPU oracle; read-out; error behaviour; determinism."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import oracle, qx, report_gens  # noqa: E402

from paper_2505_03307_b200 import circuit as ir  # noqa: E402
from paper_2505_03307_b200 import lut, workloads  # noqa: E402
from paper_2505_03307_b200.store import DeviceStore  # noqa: E402

TOL = 1e-10
MODES = ("v1", "v2", "v3")


# ------------------------------------------------------------------ reference KATs
def test_empty_circuit_and_coercion():
    for mode in MODES:                                        # tests/test_engine.py:19-26
        rep = qx.run([], 3, mode)
        assert rep.rank_trace == [[1, 1, 1]]
        assert [int(g.indices[0]) for g in rep.final.generators] == [48, 12, 3]
        assert all(list(g.lambdas) == [1.0] for g in rep.final.generators)
    assert qx.Mode.coerce("V2") is qx.Mode.V2
    with pytest.raises(ValueError):
        qx.run([], 2, "v9")


@pytest.mark.parametrize("mode", MODES)
def test_worked_circuit(mode):                                # tests/test_engine.py:38-68
    rep = qx.run([ir.sx(0), ir.rz(0, math.pi / 3), ir.cx(0, 1)], 3, mode)
    g0, g1, g2 = rep.final.generators
    assert list(g0.indices) == [20, 36] and np.allclose(g0.lambdas, [math.sqrt(3) / 2, -0.5], atol=1e-15)
    assert list(g1.indices) == [60] and list(g1.lambdas) == [1.0]
    assert list(g2.indices) == [3] and list(g2.lambdas) == [1.0]
    assert rep.order == [0, 1] and rep.rank_trace == [[1, 1, 1], [2, 1, 1], [2, 1, 1]]


def test_rank_claims_and_counters():                          # tests/test_engine.py:71-104
    for n in (2, 5, 12, 20):
        for mode in MODES:
            rep = qx.run(workloads.gen_ghz(n), n, mode)
            assert all(r == 1 for step in rep.rank_trace for r in step)
            assert len(rep.rank_trace) == rep.k + rep.k_prime + 1
    rep = qx.run(workloads.gen_xyz_chain(4, 4, 2, 1), 4, "v3")
    assert 64 < rep.max_rank <= 256
    layers, repeats, n = 3, 5, 4
    rep = qx.run(workloads.gen_xyz_chain(n, layers, repeats, 0), n, "v3")
    assert rep.counters["gates"] == layers * (3 * n * repeats + n - 1)
    assert rep.counters["sub_flatten_ops"] == rep.k == layers
    assert rep.counters["cx_applications"] == layers * (n - 1)
    rep = qx.run([ir.h(0), ir.s(0)], 1, "v2")
    assert rep.counters["cx_applications"] == 0 and rep.counters["sub_flatten_ops"] == 1


def test_errors():
    with pytest.raises(qx.NumericalCollapseError, match="generator 0 dropped at operator step 0"):
        qx.run([ir.h(0)], 1, "v1", eps=2.0)
    with pytest.raises(qx.NumericalCollapseError, match="generator 0"):
        qx.run([ir.h(0)], 2, "v3", eps=2.0)
    with pytest.raises(qx.ResourceLimitError):                # tests/test_cli.py:92-96
        qx.run(workloads.gen_xyz_chain(11, 1, 1, 0), 11, "v2")
    qx.run(workloads.gen_ghz(20), 20, "v2")                   # one-hot rows: fine at any n
    with pytest.raises(ValueError):
        qx.run([ir.h(5)], 3, "v1")
    rep = qx.run([], 33, "v1")                                 # multi-word keys above 32 qubits
    assert int(rep.final.generators[0].indices[0]) == 3 * 4 ** 32
    with pytest.raises(qx.NativeError):
        qx.run([], 513, "v1")                                  # at most sixteen words per key


def test_oversized_ansatz_is_refused_cleanly():
    """BASELINE config 4 as written (n = 20, four layers) and its two-layer point need > 300 GB of
    terms: ResourceLimitError before anything is allocated, device usable after."""
    for name in ("c4_xyz_20_2", "c4_xyz_20_4"):
        n, gates = workloads.build(name)
        with pytest.raises(qx.ResourceLimitError, match="GB of HBM"):
            qx.run(gates, n, "v3", download=False)
    rep = qx.run(workloads.gen_xyz_chain(8, 2, 1, 4), 8, "v3")
    assert sum(rep.rank_trace[-1]) == 19734


# ------------------------------------------------------------------ fixtures from the reference
def test_campaign_all_modes(golden):
    for entry in golden.load_json("campaign.json"):
        n, gates = entry["n"], golden.gates(entry["gates"])
        for mode, want in entry["modes"].items():
            rep = qx.run(gates, n, mode)
            golden.assert_gens_equal(report_gens(rep), [golden.gen(g) for g in want["final"]], tol=TOL)
            assert rep.rank_trace == want["rank_trace"], (entry["case"], mode)
            assert rep.order == want["order"] and (rep.k, rep.k_prime) == (want["k"], want["k_prime"])
            assert rep.counters == want["counters"]
        final = qx.run(gates, n, "v3").final
        ex = qx.density_expansion(final)
        for k in range(n):
            p = qx.prob_z(final, k, ex)
            assert np.max(np.abs(np.array(p) - golden.unhex(entry["prob_z"][k]))) < TOL


@pytest.mark.parametrize("name,modes", [
    ("c1_4q_clifford_t", MODES), ("c2_10q_near_clifford", MODES), ("c3_16q_clifford", MODES),
    ("c5_32q_clifford_t", ("v1", "v3")),
])
def test_baseline_configs(golden, name, modes):
    n, gates = workloads.build(name)
    for mode in modes:
        want, trace, (k, kp, updates) = golden.config(name, mode)
        rep = qx.run(gates, n, mode)
        golden.assert_gens_equal(report_gens(rep), want, tol=TOL, exact=(name == "c3_16q_clifford"))
        assert rep.rank_trace == trace and (rep.k, rep.k_prime) == (k, kp)


@pytest.mark.parametrize("key", [
    "c4_xyz_8_4/v1", "c4_xyz_8_4/v3", "c4_xyz_12_2/v1", "c4_xyz_12_2/v3", "c4_xyz_10_3/v3", "c4_xyz_14_2/v3",
])
def test_config4_ladder_digests(golden, key):
    d = golden.load_json("digests.json")[key]
    name, mode = key.split("/")
    n, gates = workloads.build(name)
    rep = qx.run(gates, n, mode)
    assert rep.rank_trace[-1] == d["trace_last"] and rep.max_rank == d["max_rank"]
    for g, dg in zip(rep.final.generators, d["gens"]):
        golden.check_digest(dg, g.lambdas, g.keys(), tol=TOL)


def test_oracle_cross_check_midsize():
    # GPU vs the CPU oracle on seeded circuits the fixtures do not cover, full coefficient compare
    for seed, n, m in ((1, 7, 80), (2, 9, 60), (3, 12, 40)):
        gates = workloads.gen_random(n, m, seed)
        for mode in ("v1", "v3"):
            rep = qx.run(gates, n, mode)
            want = oracle.run(gates, n, mode)
            for g, (lam, idx) in zip(rep.final.generators, want["final"]):
                assert np.array_equal(g.keys(), idx) and np.max(np.abs(g.lambdas - lam), initial=0) < TOL
            assert rep.rank_trace == want["rank_trace"]


# ------------------------------------------------------------------ read-out
def test_readout_units(golden):
    for u in golden.load_json("units.json")["readout"]:
        n = u["n"]
        gens = [qx.SimpleGenerator(n, lam, idx.astype(np.int64)) for lam, idx in map(golden.gen, u["final"])]
        gs = qx.GeneratorSet(n, gens)
        ex = qx.density_expansion(gs)
        assert [int(c) for c in ex.codes] == u["codes"]
        assert np.max(np.abs(ex.values - golden.unhex(u["coeffs"]))) < TOL
        for k in range(n):
            assert np.max(np.abs(np.array(qx.prob_z(gs, k, ex)) - golden.unhex(u["prob_z"][k]))) < TOL
        got = [qx.expectation(gs, w, ex) for w in u["words"]]
        assert np.max(np.abs(np.array(got) - golden.unhex(u["expect"]))) < TOL
        back = qx.expectation_heisenberg(golden.gates(u["gates"]), n, u["words"])
        assert np.max(np.abs(back - golden.unhex(u["expect"]))) < TOL


def test_readout_config1_full_and_config2(golden):
    z = golden.load_npz()
    n, gates = workloads.build("c1_4q_clifford_t")
    final = qx.run(gates, n, "v3").final
    ex = qx.density_expansion(final)
    got = np.array([qx.expectation(final, w, ex) for w in range(4 ** n)])
    assert np.max(np.abs(got - z["c1_4q_clifford_t__expect_all"])) < TOL
    got = np.array([qx.prob_z(final, k, ex) for k in range(n)])
    assert np.max(np.abs(got - z["c1_4q_clifford_t__prob_z"])) < TOL
    for mode in ("v1", "v3"):
        back = qx.expectation_heisenberg(gates, n, range(4 ** n), mode)
        assert np.max(np.abs(back - z["c1_4q_clifford_t__expect_all"])) < TOL
    n, gates = workloads.build("c2_10q_near_clifford")
    final = qx.run(gates, n, "v3").final
    ex = qx.density_expansion(final)
    assert np.array_equal(ex.codes, z["c2_10q_near_clifford__exp_codes"])
    assert np.max(np.abs(ex.values - z["c2_10q_near_clifford__exp_coeffs"])) < TOL
    got = np.array([qx.prob_z(final, k, ex) for k in range(n)])
    assert np.max(np.abs(got - z["c2_10q_near_clifford__prob_z"])) < TOL


def test_readout_kats_and_caps():
    ex = qx.density_expansion(qx.init_z(1))                   # tests/test_measure.py:20-37
    assert ex.coeffs == {0: 0.5, 3: 0.5}
    ghz = qx.run(workloads.gen_ghz(2), 2, "v3").final
    assert qx.density_expansion(ghz).coeffs == {0: 0.25, 5: 0.25, 15: 0.25, 10: -0.25}
    flipped = qx.run([ir.x(1)], 2, "v1").final
    assert qx.prob_z(flipped, 1) == (0.0, 1.0)
    for theta in (0.3, 1.1, 2.9):
        g = qx.run([ir.ry(0, theta)], 1, "v3").final
        assert abs(qx.expectation(g, 3) - math.cos(theta)) < 1e-12
    with pytest.raises(qx.ResourceLimitError, match="capped at 12 qubits"):
        qx.density_expansion(qx.init_z(13))
    with pytest.raises(qx.ResourceLimitError, match="term budget"):
        qx.density_expansion(qx.run(workloads.gen_xyz_chain(6, 2, 1, 3), 6, "v3").final, term_budget=500)
    with pytest.raises(ValueError):
        qx.prob_z(qx.init_z(2), 2)
    with pytest.raises(ValueError):
        qx.expectation(qx.init_z(2), 16)
    # n = 16 GHZ through the raised cap (2**16 terms) and Heisenberg at n = 32
    n = 16
    ghz = qx.run(workloads.gen_ghz(n), n, "v1").final
    ex = qx.density_expansion(ghz, max_qubits=16)
    assert len(ex) == 2 ** n and abs(qx.prob_z(ghz, 5, ex)[0] - 0.5) < 1e-12
    n, gates = workloads.build("c5_32q_clifford_t")
    zz = qx.expectation_heisenberg(gates[:400], n, [3 << (2 * k) for k in range(n)])
    want = oracle.expectation_heisenberg(gates[:400], n, [3 << (2 * k) for k in range(n)])
    assert np.max(np.abs(zz - np.array(want))) < TOL


# ------------------------------------------------------------------ determinism, mutation, shards
def test_bitwise_determinism():                               # tests/test_engine.py:135-143
    gates = workloads.gen_xyz_chain(10, 2, 1, 7)
    for mode in MODES[::2]:
        a, b = qx.run(gates, 10, mode), qx.run(gates, 10, mode)
        for ga, gb in zip(a.final.generators, b.final.generators):
            assert np.array_equal(ga.indices, gb.indices) and np.array_equal(ga.lambdas, gb.lambdas)


def test_cx_sign_mutation_is_detected(golden, monkeypatch):   # tests/test_cli.py:198-203
    bad = lut.LUT_SIGN.copy()
    bad[1, 0] = -1
    monkeypatch.setattr(lut, "LUT_SIGN", bad)
    n, gates = workloads.build("c2_10q_near_clifford")
    want, _, _ = golden.config("c2_10q_near_clifford", "v1")
    rep = qx.run(gates, n, "v1")
    with pytest.raises(AssertionError):
        golden.assert_gens_equal(report_gens(rep), want, tol=TOL)


def test_generator_shards_equal_full_run():
    n, gates = workloads.build("c2_10q_near_clifford")
    full = qx.run(gates, n, "v3")
    for ids in ([0, 3, 7], [9], list(range(5, 10))):
        part = qx.run(gates, n, "v3", generators=ids)
        for local, gi in enumerate(ids):
            a, b = part.final.generators[local], full.final.generators[gi]
            assert np.array_equal(a.indices, b.indices) and np.array_equal(a.lambdas, b.lambdas)
        assert [[step[g] for g in ids] for step in full.rank_trace] == part.rank_trace


def test_streamed_finish_equals_plain_download(monkeypatch):
    """run() evolves the last operator per generator range and overlaps each range's download with
    the next range's kernels when the result is large (engine._finish_streamed); the generators it
    returns must be the ones a plain run leaves in HBM."""
    from paper_2505_03307_b200 import engine

    n, gates = workloads.build("c4_xyz_12_2")
    monkeypatch.setattr(engine, "STREAM_MIN_RAW", 1 << 16)       # force the streamed path at this size
    streamed = qx.run(gates, n, "v3", pinned=True)
    assert streamed.device.get("streamed_ranges", 0) >= 2
    plain = qx.run(gates, n, "v3", download=False)
    try:
        segs = plain.device["store"].segments()
    finally:
        plain.device["store"].close()
    assert streamed.rank_trace == plain.rank_trace
    for g, (lam, keys) in zip(streamed.final.generators, segs):
        assert np.array_equal(g.keys(), keys) and np.array_equal(g.lambdas, lam)


@pytest.mark.parametrize("form", [1, 2])
def test_narrow_and_packed_downloads_equal_plain_download(monkeypatch, form):
    """Streamed results of n <= 16 cross PCIe as 32-bit keys (form 1) or, when large, as 16-bit
    low halves + per-generator bucket tables written by the last sort pass (form 2); host threads
    rebuild the 64-bit keys.  Either way run() must return exactly what a plain download gives."""
    from paper_2505_03307_b200 import engine

    n, gates = workloads.build("c4_xyz_14_2")
    monkeypatch.setattr(engine, "_NARROW_FORM", form)
    streamed = qx.run(gates, n, "v3", pinned=True)
    assert streamed.device.get("streamed_ranges", 0) >= 2
    total = sum(g.rank for g in streamed.final.generators)
    if form == 2:
        assert streamed.device["d2h_bytes"] < 12 * total        # at least one range went packed
    else:
        assert streamed.device["d2h_bytes"] == 12 * total
    plain = qx.run(gates, n, "v3", download=False)
    try:
        segs = plain.device["store"].segments()
    finally:
        plain.device["store"].close()
    for g, (lam, keys) in zip(streamed.final.generators, segs):
        assert np.array_equal(g.keys(), keys) and np.array_equal(g.lambdas, lam)


def test_collapse_in_the_grouped_operator_step():
    """An eps above every coefficient empties a generator inside the grouped dense path; the engine
    must report it like the reference (engine.py:148-152)."""
    n, gates = workloads.build("c4_xyz_12_2")
    with pytest.raises(qx.NumericalCollapseError, match="all terms of generator"):
        qx.run(gates, n, "v3", eps=0.9)


def test_eps_zero_takes_the_raw_path_and_matches_the_oracle():
    """eps == 0 keeps exact-zero sums, which the grouped path cannot tell from unreached slots: the
    call must fall back to expand + sort + reduce and still agree with the oracle."""
    n = 9
    gates = qx.gen_xyz_chain(n, 2, 1, rng=11)
    got = qx.run(gates, n, "v3", eps=0.0)
    want = oracle.run(gates, n, "v3", eps=0.0)
    assert got.rank_trace == want["rank_trace"]
    for g, (lam, idx) in zip(got.final.generators, want["final"]):
        assert np.array_equal(g.keys(), idx) and np.max(np.abs(g.lambdas - lam)) < TOL


def _mixed_layers(rng, n, heavy):
    """Layers of per-qubit operators (generic rotation / one-axis rotation / Clifford / nothing)
    followed by a CX chain over a random qubit order: supports spread like on the ansatz circuits,
    so operators have large fan-outs, partial mixing and, at three layers, groups with many sources."""
    gates = []
    for _ in range(3 if n <= 8 else 2):
        for q in range(n):
            kind = rng.integers(0, 6) if rng.uniform() > heavy else 0
            if kind <= 2:
                gates += [qx.Instruction(g, (q,), float(rng.uniform(0, 6.28))) for g in ("RX", "RY", "RZ")]
            elif kind == 3:
                gates.append(qx.Instruction(str(rng.choice(["RX", "RY", "RZ"])), (q,), float(rng.uniform(0, 6.28))))
            elif kind == 4:
                gates.append(qx.Instruction(str(rng.choice(["H", "S", "X", "SX"])), (q,)))
        order = rng.permutation(n)
        gates += [qx.Instruction("CX", (int(a), int(b))) for a, b in zip(order[:-1], order[1:]) if rng.uniform() < 0.85]
        if rng.integers(0, 2):
            gates.append(qx.Instruction("H", (int(rng.integers(n)),)))
    return gates


@pytest.mark.parametrize("case", range(14))
def test_random_entangling_circuits_against_oracle(case):
    """The grouped operator step on operators of every shape (tools/stress_dense.py runs more)."""
    rng = np.random.default_rng([77, case])
    n = int(rng.integers(8, 12))
    gates = _mixed_layers(rng, n, float(rng.choice([0.0, 0.5, 0.8])))
    want = oracle.run(gates, n, "v3")
    got = qx.run(gates, n, "v3")
    assert got.rank_trace == want["rank_trace"]
    for g, (lam, idx) in zip(got.final.generators, want["final"]):
        assert np.array_equal(g.keys(), idx)
        assert len(lam) == 0 or np.max(np.abs(g.lambdas - lam)) < TOL


def test_dense_layout_with_eps_zero_keeps_every_word():
    """v2 with eps = 0: a generator that branches goes through the reference's 4**n scatter buffer and
    comes back with EVERY word, exact zeros included (stabilizer.py:277-286); found by
    tools/fuzz_engine.py.  Checked against the oracle port (which equals the reference here)."""
    for seed, n, m in ((1, 1, 27), (2, 2, 39), (3, 3, 15), (4, 5, 30)):
        gates = workloads.gen_random(n, m, seed)
        got = qx.run(gates, n, "v2", eps=0.0)
        want = oracle.run(gates, n, "v2", 0.0)
        assert got.rank_trace == want["rank_trace"]
        for g, (lam, idx) in zip(got.final.generators, want["final"]):
            assert np.array_equal(g.keys(), idx) and np.max(np.abs(g.lambdas - lam), initial=0.0) < TOL
    g = qx.SimpleGenerator(2, [1.0], [5])                        # XX through RY on both qubits
    block = np.broadcast_to(lut.axis_map("RY", 0.7).T, (2, 3, 3)).copy()
    dense = qx.flatten(qx.sub(g, block, "dense"), eps=0.0)
    assert dense.rank == 16 and int((dense.lambdas == 0.0).sum()) == 12
    assert qx.flatten(qx.sub(g, block, "ragged"), eps=0.0).rank == 4


def test_v1_and_v3_coefficients_are_bitwise_the_oracles():
    """Sums of three or more contributions to one word are added in the reference's order -- sources
    grouped by branch-count pattern (stabilizer.py:294-296), canonical inside a group -- so small
    circuits reproduce the oracle (= the reference) bit for bit in v3 as they do in v1.  Without
    qx_store_order_for_operator 9 of these 250 circuits differ in the last bit."""
    for case in range(250):
        rng = np.random.default_rng([1, 19800 + case])
        n = int(rng.integers(1, 8))
        gates = workloads.gen_random(n, int(rng.integers(0, 50)), rng)
        for mode in ("v1", "v3"):
            got = qx.run(gates, n, mode).final
            want = oracle.run(gates, n, mode)["final"]
            for g, (lam, idx) in zip(got.generators, want):
                assert np.array_equal(g.keys(), idx) and np.array_equal(g.lambdas, lam), (case, mode)


def test_raw_flatten_order_is_the_references():
    """flatten(canonical=False): strings grouped by branch-count pattern, stable inside a group,
    branches in C order (stabilizer.py:289-322) -- the oracle's expand_operator, element for element."""
    rng = np.random.default_rng(77)
    for _ in range(20):
        n = int(rng.integers(2, 6))
        idx = rng.choice(4 ** n, size=min(4 ** n, int(rng.integers(3, 30))), replace=False)
        g = qx.SimpleGenerator(n, rng.uniform(-1, 1, size=len(idx)), idx)
        names = [str(v) for v in rng.choice(["H", "RX", "RY", "RZ", "S"], size=n)]
        block = np.stack([lut.compose_block([ir.Instruction(name, (q,), float(rng.uniform(0, 6.3)) if name[0] == "R" else 0.0)])
                          for q, name in enumerate(names)])
        raw = qx.flatten(qx.sub(g, block), canonical=False)
        wl, wi = oracle.expand_operator(g.lambdas, g.keys(), n, block)
        assert np.array_equal(raw.keys(), wi) and np.array_equal(raw.lambdas, wl)
