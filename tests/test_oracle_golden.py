"""Pin the CPU oracle (oracle/stabsim_port.py) against the reference.

Two sources: the known-answer vectors the reference's own tests
hold for this path, restated here with their file:line, and fixtures produced
by running the reference itself (oracle/make_golden.py).  Keys must be
bit-exact; v1/v3 coefficients bitwise equal (same numpy primitives, same
order); v2 within 1e-12.
"""

import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
import stabsim_port as port  # noqa: E402

from paper_2505_03307_b200 import circuit as ir  # noqa: E402
from paper_2505_03307_b200 import workloads as wl  # noqa: E402
from paper_2505_03307_b200.errors import NumericalCollapseError, ResourceLimitError  # noqa: E402

U64 = np.uint64


def gens_of(res):
    return res["final"]


# ---------------------------------------------------------------- reference KATs
def test_init_z_kat():
    # tests/test_stabilizer.py:95-98
    assert [int(i[0]) for _, i in port.init_z(3)] == [48, 12, 3]


@pytest.mark.parametrize("mode", ["v1", "v2", "v3"])
def test_worked_circuit_kat(mode):
    # tests/test_engine.py:38-68
    res = port.run([ir.sx(0), ir.rz(0, math.pi / 3), ir.cx(0, 1)], 3, mode)
    (l0, i0), (l1, i1), (l2, i2) = res["final"]
    assert list(i0) == [20, 36] and np.allclose(l0, [math.sqrt(3) / 2, -0.5], atol=1e-15)
    assert list(i1) == [60] and list(l1) == [1.0]
    assert list(i2) == [3] and list(l2) == [1.0]
    assert res["order"] == [0, 1]
    assert res["rank_trace"] == [[1, 1, 1], [2, 1, 1], [2, 1, 1]]


def test_cx_kats():
    # tests/test_stabilizer.py:219-229, 262-267; tests/test_lut.py:126-150
    lam, idx = port.conj_cx(np.ones(1), np.array([16], dtype=U64), 3, 0, 1)
    assert list(idx) == [20] and list(lam) == [1.0]
    lam, idx = port.conj_cx(np.array([0.5, -math.sqrt(3) / 2]), np.array([16, 32], dtype=U64), 3, 0, 1)
    assert list(idx) == [20, 36]
    for (c, t), want in {(1, 0): (1, 1, 1), (0, 3): (3, 3, 1), (1, 3): (2, 2, -1), (2, 2): (1, 3, -1),
                         (3, 0): (3, 0, 1), (0, 1): (0, 1, 1), (2, 0): (2, 1, 1)}.items():
        assert (port.CX_C[c, t], port.CX_T[c, t], port.CX_S[c, t]) == want
    with pytest.raises(ValueError):
        port.conj_cx(np.ones(1), np.array([5], dtype=U64), 2, 1, 1)


def test_flatten_golden_kat():
    # tests/test_stabilizer.py:140-155: 2(3Y+4Z)(Z) + (I)(X+Z) -> idx [1,3,11,15], lam [1,1,6,8]
    # rebuilt through a block whose rows give exactly those cells
    block = np.zeros((2, 3, 3))
    block[0] = np.eye(3)
    block[0, 1] = [0.0, 3.0, 4.0]          # Y -> 3Y + 4Z on qubit 0
    block[1] = np.eye(3)
    block[1, 0] = [1.0, 0.0, 1.0]          # X -> X + Z on qubit 1
    lam, idx = port.operator_v3(np.array([2.0, 1.0]), np.array([2 * 4 + 3, 1], dtype=U64), 2, block)
    assert list(idx) == [1, 3, 11, 15] and list(lam) == [1.0, 1.0, 6.0, 8.0]


def test_merge_kats():
    # tests/test_stabilizer.py:271-292
    lam, idx = port.merge(np.array([1.0, 1.0]), np.array([3, 3], dtype=U64))
    assert list(lam) == [2.0] and list(idx) == [3]
    lam, idx = port.merge(np.array([1e-15]), np.array([2], dtype=U64), 1e-12)
    assert len(lam) == 0
    lam, idx = port.merge(np.array([1.0, 2.0, 3.0]), np.array([9, 2, 5], dtype=U64))
    assert list(idx) == [2, 5, 9]


def test_readout_kats():
    # tests/test_measure.py:20-37, 91-94, 147-150
    codes, vals = port.density_expansion(port.init_z(1), 1)
    assert dict(zip(map(int, codes), vals)) == {0: 0.5, 3: 0.5}
    ghz = port.run(wl.gen_ghz(2), 2, "v3")["final"]
    ex = port.density_expansion(ghz, 2)
    got = dict(zip(map(int, ex[0]), ex[1]))
    assert got == {0: 0.25, 5: 0.25, 15: 0.25, 10: -0.25}
    flipped = port.run([ir.x(1)], 2, "v1")["final"]
    assert port.prob_z(flipped, 2, 1) == (0.0, 1.0)
    for theta in (0.3, 1.1, 2.9):
        g = port.run([ir.ry(0, theta)], 1, "v3")["final"]
        assert abs(port.expectation(g, 1, 3) - math.cos(theta)) < 1e-12
    with pytest.raises(ResourceLimitError):
        port.density_expansion(port.init_z(13), 13)


def test_rank_claims_and_guards():
    # tests/test_acceptance.py:119-127; tests/test_engine.py:71-88; tests/test_cli.py:92-96
    for n in (2, 5, 12, 20):
        res = port.run(wl.gen_ghz(n), n, "v1")
        assert all(r == 1 for step in res["rank_trace"] for r in step)
        assert len(res["rank_trace"]) == res["k"] + res["k_prime"] + 1
    res = port.run(wl.gen_xyz_chain(4, 4, 2, 1), 4, "v3")
    assert 64 < max(max(s) for s in res["rank_trace"]) <= 256
    with pytest.raises(ResourceLimitError):
        port.run(wl.gen_xyz_chain(11, 1, 1, 0), 11, "v2")
    with pytest.raises(ValueError):
        port.run([], 2, "v9")
    with pytest.raises(NumericalCollapseError, match="generator 0"):
        port.run([ir.h(0)], 1, "v1", eps=2.0)


# ---------------------------------------------------------------- fixtures from the reference
def test_units_apply_cx(golden):
    for u in golden.load_json("units.json")["apply_cx"]:
        lam, idx = golden.gen(u["in"])
        got = port.conj_cx(lam, idx, u["n"], u["c"], u["t"])
        golden.assert_gens_equal([got], [golden.gen(u["out"])], exact=True)


def test_units_apply_1q(golden):
    for u in golden.load_json("units.json")["apply_1q"]:
        lam, idx = golden.gen(u["in"])
        m = port.axis_map(u["gate"], float.fromhex(u["theta"]))
        got = port.conj_1q_v1(lam, idx, u["n"], u["q"], m)
        golden.assert_gens_equal([got], [golden.gen(u["out"])], exact=True)


def test_units_canonicalize(golden):
    for u in golden.load_json("units.json")["canonicalize"]:
        got = port.merge(*golden.gen(u["in"]), 1e-12)
        golden.assert_gens_equal([got], [golden.gen(u["out"])], exact=True)


def test_units_operator(golden):
    for u in golden.load_json("units.json")["operator"]:
        n = u["n"]
        block = golden.unhex(u["block"]).reshape(n, 3, 3)
        mine = port.lut_blocks(port.partition(golden.gates(u["gates"]), n), n)[0]
        assert np.array_equal(mine, block)
        lam, idx = golden.gen(u["in"])
        raw = port.expand_operator(lam, idx, n, block)
        golden.assert_gens_equal([raw], [golden.gen(u["raw"])], exact=True)      # raw order too
        golden.assert_gens_equal([port.operator_v3(lam, idx, n, block)], [golden.gen(u["out"])], exact=True)
        golden.assert_gens_equal([port.operator_v2(lam, idx, n, block)], [golden.gen(u["out"])], tol=1e-12)


def test_units_readout(golden):
    for u in golden.load_json("units.json")["readout"]:
        n = u["n"]
        gens = [golden.gen(g) for g in u["final"]]
        codes, vals = port.density_expansion(gens, n)
        assert [int(c) for c in codes] == u["codes"]
        assert np.array_equal(vals, golden.unhex(u["coeffs"]))
        for k in range(n):
            assert list(port.prob_z(gens, n, k, (codes, vals))) == list(golden.unhex(u["prob_z"][k]))
        for w, e in zip(u["words"], golden.unhex(u["expect"])):
            assert port.expectation(gens, n, w, (codes, vals)) == e


def test_campaign(golden):
    for entry in golden.load_json("campaign.json"):
        n, gates = entry["n"], golden.gates(entry["gates"])
        for mode, want in entry["modes"].items():
            res = port.run(gates, n, mode)
            ref = [golden.gen(g) for g in want["final"]]
            if mode == "v2":
                golden.assert_gens_equal(res["final"], ref, tol=1e-12)
            else:
                golden.assert_gens_equal(res["final"], ref, exact=True)
            assert res["rank_trace"] == want["rank_trace"]
            assert res["order"] == want["order"] and (res["k"], res["k_prime"]) == (want["k"], want["k_prime"])
            assert res["counters"] == want["counters"]
        assert port.count_updates(gates, n) == entry["updates"]
        final = port.run(gates, n, "v3")["final"]
        ex = port.density_expansion(final, n)
        for k in range(n):
            assert list(port.prob_z(final, n, k, ex)) == list(golden.unhex(entry["prob_z"][k]))


def test_heisenberg_matches_expansion(golden):
    # the oracle's back-propagation read-out agrees with the reference's expansion read-out
    for u in golden.load_json("units.json")["readout"]:
        n, gates = u["n"], golden.gates(u["gates"])
        got = port.expectation_heisenberg(gates, n, u["words"], "v1")
        assert np.max(np.abs(np.array(got) - golden.unhex(u["expect"]))) < 1e-10
