"""Kernel-level parity on the GPU: each C-ABI entry point against the reference's unit vectors
(tests/golden/units.json, produced by the reference itself) and against the CPU oracle on seeded
random inputs.  Keys must match bit-exactly; coefficients within 1e-10 (float64)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import DeviceStore, merge_on_device, oracle, qx, random_terms  # noqa: E402

from paper_2505_03307_b200 import _native, lut  # noqa: E402
from paper_2505_03307_b200.stabilizer import SimpleGenerator, keys_to_indices  # noqa: E402

TOL = 1e-10


def _sg(n, lam, keys):
    return SimpleGenerator(n, lam, keys_to_indices(np.asarray(keys, dtype=np.uint64), n))


def test_units_apply_cx(golden):
    for u in golden.load_json("units.json")["apply_cx"]:
        lam, idx = golden.gen(u["in"])
        out = qx.apply_cx(_sg(u["n"], lam, idx), u["c"], u["t"])
        golden.assert_gens_equal([(out.lambdas, out.keys())], [golden.gen(u["out"])], exact=True)


def test_units_apply_1q(golden):
    for u in golden.load_json("units.json")["apply_1q"]:
        lam, idx = golden.gen(u["in"])
        out = qx.apply_1q(_sg(u["n"], lam, idx), u["gate"], u["q"], float.fromhex(u["theta"]))
        golden.assert_gens_equal([(out.lambdas, out.keys())], [golden.gen(u["out"])], tol=TOL)


def test_units_canonicalize(golden):
    for u in golden.load_json("units.json")["canonicalize"]:
        lam, idx = golden.gen(u["in"])
        out = qx.canonicalize(_sg(u["n"], lam, idx), 1e-12)
        golden.assert_gens_equal([(out.lambdas, out.keys())], [golden.gen(u["out"])], tol=TOL)


def test_units_operator(golden):
    for u in golden.load_json("units.json")["operator"]:
        n = u["n"]
        block = golden.unhex(u["block"]).reshape(n, 3, 3)
        lam, idx = golden.gen(u["in"])
        g = _sg(n, lam, idx)
        raw = qx.flatten(qx.sub(g, block), canonical=False)
        # raw lists: same multiset of (key, coefficient); order is term-major on the device
        wl, wk = golden.gen(u["raw"])
        assert sorted(zip(raw.keys().tolist(), raw.lambdas.tolist())) == sorted(zip(wk.tolist(), wl.tolist()))
        for layout in ("ragged", "dense"):
            out = qx.flatten(qx.sub(g, block, layout), 1e-12)
            golden.assert_gens_equal([(out.lambdas, out.keys())], [golden.gen(u["out"])], tol=TOL)


def test_kats_from_reference_tests():
    # tests/test_stabilizer.py:219-229 (CX), :271-292 (merge), :140-155 (golden flatten)
    out = qx.apply_cx(SimpleGenerator(3, [1.0], [16]), 0, 1)
    assert list(out.indices) == [20] and list(out.lambdas) == [1.0]
    out = qx.canonicalize(SimpleGenerator(1, [1.0, 1.0], [3, 3]))
    assert list(out.lambdas) == [2.0] and list(out.indices) == [3]
    out = qx.canonicalize(SimpleGenerator(1, [1e-15], [2]), eps=1e-12)
    assert out.is_degenerate
    out = qx.canonicalize(SimpleGenerator(2, [1.0, 2.0, 3.0], [9, 2, 5]))
    assert list(out.indices) == [2, 5, 9]
    block = np.zeros((2, 3, 3))
    block[:] = np.eye(3)
    block[0, 1] = [0.0, 3.0, 4.0]
    block[1, 0] = [1.0, 0.0, 1.0]
    out = qx.flatten(qx.sub(SimpleGenerator(2, [2.0, 1.0], [11, 1]), block))
    assert list(out.indices) == [1, 3, 11, 15] and list(out.lambdas) == [1.0, 1.0, 6.0, 8.0]
    with pytest.raises(ValueError):
        qx.apply_cx(SimpleGenerator(2, [1.0], [5]), 1, 1)
    with pytest.raises(ValueError):
        qx.sub(SimpleGenerator(2, [1.0], [5]), np.zeros((3, 3, 3)))
    big = qx.apply_cx(qx.init_z(32).generators[0], 1, 0)
    assert int(big.indices[0]) == 3 * 4 ** 31 + 3 * 4 ** 30        # n > 31: Python-int indices


@pytest.mark.parametrize("n,count,distinct", [
    (1, 5, 3), (2, 33, 9), (4, 1000, 200), (8, 4096, 4096), (16, 8192, 3000), (32, 8192, 8000),   # small path
    (5, 8193, 700), (16, 100_000, 40_000), (32, 300_000, 299_000), (10, 1_000_000, 600_000),          # large path
    (16, 3_000_000, 1_000_000),
])
def test_merge_matches_oracle(n, count, distinct):
    rng = np.random.default_rng(count * 31 + n)
    lam, keys = random_terms(rng, n, count, distinct)
    lam[rng.integers(0, count, size=max(1, count // 7))] *= 1e-13
    (gl, gk), = merge_on_device(n, [(lam, keys)])
    wl, wk = oracle.merge(lam, keys)
    assert np.array_equal(gk, wk)
    assert np.array_equal(gl, wl)          # same summation order as np.add.at -> bitwise


def test_merge_many_segments_with_empties():
    rng = np.random.default_rng(5)
    n = 12
    sizes = [0, 7, 0, 20_000, 1, 0, 9000, 4608, 4609, 0]
    gens = [random_terms(rng, n, s, max(1, s // 2)) if s else (np.zeros(0), np.zeros(0, dtype=np.uint64)) for s in sizes]
    got = merge_on_device(n, gens)
    for (gl, gk), (lam, keys) in zip(got, gens):
        wl, wk = oracle.merge(lam, keys)
        assert np.array_equal(gk, wk) and np.array_equal(gl, wl)
    small = [g if len(g[0]) <= 8192 else (g[0][:100], g[1][:100]) for g in gens]
    got = merge_on_device(n, small)
    for (gl, gk), (lam, keys) in zip(got, small):
        wl, wk = oracle.merge(lam, keys)
        assert np.array_equal(gk, wk) and np.array_equal(gl, wl)


def test_merge_adversarial_keys():
    n = 16
    # all equal, already sorted, reverse sorted, two values alternating; sums that cancel exactly
    same = (np.full(20_000, 0.25), np.full(20_000, 12345, dtype=np.uint64))
    asc = (np.ones(30_000), np.arange(30_000, dtype=np.uint64) * np.uint64(65537) % np.uint64(4 ** n))
    desc = (np.ones(30_000), asc[1][::-1].copy())
    alt = (np.tile([1.0, -1.0], 10_000), np.tile(np.array([7, 7], dtype=np.uint64), 10_000))
    got = merge_on_device(n, [same, asc, desc, alt])
    for (gl, gk), (lam, keys) in zip(got, [same, asc, desc, alt]):
        wl, wk = oracle.merge(lam, keys)
        assert np.array_equal(gk, wk) and np.array_equal(gl, wl)
    assert len(got[3][0]) == 0             # exact cancellation -> dropped -> empty generator


def test_clifford_run_matches_oracle():
    rng = np.random.default_rng(11)
    for n in (2, 7, 16, 31, 32):
        gates = qx.gen_random(n, 300, rng, gates=("H", "S", "X", "SX", "CX"))
        lam, keys = random_terms(rng, n, 5001, 5001)
        prog = []
        wl, wk = lam.copy(), keys.copy()
        for g in gates:
            if g.gate == "CX":
                prog.append(lut.cx_op(n, *g.wires))
                wl, wk = oracle.conj_cx(wl, wk, n, *g.wires)
            else:
                prog.append(lut.perm_op(n, g.wires[0], lut.FIXED_PERMS[g.gate]))
                m = oracle.axis_map(g.gate)
                # oracle single-gate conjugation without merge: permutation => first branch only
                a1 = {d: int(np.nonzero(m[:, d - 1])[0][0]) + 1 for d in (1, 2, 3)}
                sg = {d: m[a1[d] - 1, d - 1] for d in (1, 2, 3)}
                sh = np.uint64(2 * (n - 1 - g.wires[0]))
                d = ((wk >> sh) & np.uint64(3)).astype(np.int64)
                newd = np.array([0, a1[1], a1[2], a1[3]], dtype=np.uint64)[d]
                wk = (wk & ~(np.uint64(3) << sh)) | (newd << sh)
                wl = wl * np.array([1.0, sg[1], sg[2], sg[3]])[d]
        with DeviceStore(n, 1, 0) as st:
            st.upload([(lam, keys)])
            st.apply_clifford(prog)
            (gl, gk), = st.segments()
            assert np.array_equal(gk, wk) and np.array_equal(gl, wl)


def test_split_and_operator_raw_match_oracle():
    rng = np.random.default_rng(21)
    for n in (3, 9, 16, 32):
        lam, keys = random_terms(rng, n, 6000, 6000)
        # v1 split on a random qubit for each rotation family
        for gate in ("RX", "RY", "RZ"):
            q, theta = int(rng.integers(n)), float(rng.uniform(0, 6.28))
            out = qx.apply_1q(SimpleGenerator(n, lam, keys_to_indices(keys, n)), gate, q, theta)
            wl0, wk0 = oracle.conj_1q_v1(lam, keys, n, q, oracle.axis_map(gate, theta))
            assert np.array_equal(out.keys(), wk0) and np.max(np.abs(out.lambdas - wl0)) < TOL
        # v3 operator with rotations on every qubit, few input terms (big fan-out)
        gates = [qx.Instruction(str(rng.choice(["RX", "RY", "RZ"])), (j,), float(rng.uniform(0, 6.28))) for j in range(min(n, 10))]
        block = oracle.lut_blocks(oracle.partition(gates, n), n)[0]
        few = SimpleGenerator(n, lam[:5], keys_to_indices(keys[:5], n))
        out = qx.flatten(qx.sub(few, block))
        wl, wk = oracle.operator_v3(lam[:5], keys[:5], n, block)
        assert np.array_equal(out.keys(), wk) and np.max(np.abs(out.lambdas - wl)) < TOL
        counts = qx.stabilizer.branch_counts(qx.sub(few, block))
        assert int(counts.sum()) == len(oracle.expand_operator(lam[:5], keys[:5], n, block)[0])


def test_partition_by_owner_roundtrip(golden):
    rng = np.random.default_rng(3)
    n, world = 14, 4
    gens = [random_terms(rng, n, s, s) for s in (5000, 1, 70_000)] + [(np.zeros(0), np.zeros(0, dtype=np.uint64))]
    with DeviceStore(n, len(gens), 0) as st:
        st.upload(gens)
        counts = st.partition_by_owner(world)
        # owner = splitmix64(key) % world, computed independently on the host
        for s, (lam, keys) in enumerate(gens):
            z = keys + np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
            owner = (z % np.uint64(world)).astype(np.int64)
            assert [int((owner == r).sum()) for r in range(world)] == counts[:, s].tolist()
        d_keys, d_lam, _ = st.device_view()
        st.assemble(d_keys, d_lam, counts)          # loop-back: receive what was sent
        back = st.segments()
        for (bl, bk), (lam, keys) in zip(back, gens):
            assert sorted(zip(bk.tolist(), bl.tolist())) == sorted(zip(keys.tolist(), lam.tolist()))


def test_zi_sums_and_norms():
    rng = np.random.default_rng(8)
    n = 9
    gens = [random_terms(rng, n, s, s) for s in (1, 300, 70_000)]
    with DeviceStore(n, 3, 0) as st:
        st.upload(gens)
        zi, nr = st.zi_sums(), st.norms()
    for (lam, keys), a, b in zip(gens, zi, nr):
        mask = (((keys >> np.uint64(1)) ^ keys) & np.uint64(0x5555555555555555)) == 0
        assert abs(a - lam[mask].sum()) < 1e-9 and abs(b - np.dot(lam, lam)) < 1e-9


@pytest.mark.parametrize("n,terms,rot_qubits,n_ops,mix", [
    (3, 40, 3, 0, 1), (6, 300, 6, 25, 1),         # small merge path, 32-bit working keys
    (12, 60, 9, 40, 1), (16, 8, 12, 15, 1),       # large fan-out: grouped dense path, narrow keys
    (16, 2000, 5, 200, 1),                        # small fan-out: raw expansion, many sources per tile
    (20, 50, 9, 60, 1), (32, 20, 10, 300, 1),     # 64-bit working keys
    (14, 30, 10, 0, 1),                           # narrow keys without a Clifford run
    (8, 3000, 8, 30, 3), (10, 2000, 10, 0, 3),    # dense path: hundreds of sources per group, many tiles
    (9, 500, 9, 12, 2), (18, 40, 11, 50, 3),      # dense path: partial mixing; 64-bit working keys
    (7, 400, 7, 9, 3),                            # dense path: every tile spans several groups
])
def test_operator_run_equals_three_steps(n, terms, rot_qubits, n_ops, mix):
    """qx_apply_operator_run (grouped dense accumulation or raw expansion, Clifford run folded in,
    narrow keys) must give bit-for-bit what qx_apply_operator + qx_apply_clifford + qx_merge give,
    which in turn are checked against the oracle above.  mix = rotations stacked per qubit."""
    rng = np.random.default_rng(n * 1000 + terms + n_ops)
    gens = []
    for s in (terms, 1, max(1, terms // 3)):
        lam, keys = random_terms(rng, n, s, s)
        keys = np.unique(keys)
        gens.append((lam[: len(keys)], keys))
    qs = rng.choice(n, size=rot_qubits, replace=False)
    gates = [qx.Instruction(str(rng.choice(["RX", "RY", "RZ"])), (int(j),), float(rng.uniform(0, 6.28)))
             for _ in range(mix) for j in qs]
    block = oracle.lut_blocks(oracle.partition(gates, n), n)[0]
    counts, axes, weights = lut.operator_tables(block)
    prog = []
    for g in qx.gen_random(n, n_ops, rng, gates=("H", "S", "X", "SX", "CX")) if n_ops else []:
        prog.append(lut.cx_op(n, *g.wires) if g.gate == "CX" else lut.perm_op(n, g.wires[0], lut.FIXED_PERMS[g.gate]))
    with DeviceStore(n, len(gens), 0) as st:
        st.upload(gens)
        st.apply_operator(counts, axes, weights)
        st.apply_clifford(prog)
        want_ranks = st.merge(1e-12)
        want = [(l.copy(), k.copy()) for l, k in st.segments()]
    with DeviceStore(n, len(gens), 0) as st:
        st.upload(gens)
        raw, ranks = st.apply_operator_run(counts, axes, weights, prog, 1e-12)
        got = [(l.copy(), k.copy()) for l, k in st.segments()]
    assert ranks == want_ranks and raw >= sum(ranks)
    for (gl, gk), (wl, wk) in zip(got, want):
        assert np.array_equal(gk, wk)
        if terms >= 400 and mix > 1:
            # groups with >= 64 sources take the factored sum (dense.cu): same terms, products
            # associated differently, so coefficients agree to rounding
            assert np.max(np.abs(gl - wl)) < 1e-12
        else:
            assert np.array_equal(gl, wl)      # sign flips are exact, summation order unchanged


@pytest.mark.parametrize("n,qubits,count,bucket", [
    (8, list(range(8)), 4000, True), (8, list(range(8)), 4000, False),     # 32-bit keys, all digits
    (9, [0, 2, 3, 5, 6, 7, 8], 2000, True),                              # seven digits, the rest identity or idle
    (22, [1, 4, 5, 9, 13, 14, 20, 21], 5000, True),                      # 64-bit keys, digits spread over the word
    (22, [1, 4, 5, 9, 13, 14, 20, 21], 5000, False),
    (10, list(range(10)), 1200, False),                                  # ten digits: the tensor in global memory
    (24, [0, 1, 4, 5, 9, 13, 14, 20, 21, 22, 23], 1300, False),          # eleven digits, 64-bit keys
    (12, list(range(12)), 1400, False),                                  # twelve digits next to smaller groups
])
def test_groups_summed_mode_by_mode(n, qubits, count, bucket):
    """Groups with many sources on at most 8 digits have their sums formed one qubit at a time
    ahead of the slot kernel (dense.cu k_group_kron; k_kron_mode above 8 digits): the same products as stabilizer.py:300-337,
    associated per qubit instead of per source, so keys are the reference's and coefficients agree
    to rounding (|sum| <= sum of |lambda| ~ 1e3 here, 1e-16 relative per operation)."""
    rng = np.random.default_rng(n * 77 + count)
    shift = np.uint64(2) * (np.uint64(n - 1) - np.array(qubits, dtype=np.uint64))
    gens = []
    for c, lowest in ((count, 1), (count // 3, 0), (3, 1)):       # lowest = 0: identities mixed in -> several groups
        digits = rng.integers(lowest, 4, size=(c * 2, len(qubits))).astype(np.uint64)
        keys = np.unique((digits << shift).sum(axis=1, dtype=np.uint64))[:c]
        gens.append((rng.uniform(0.2, 1.0, size=len(keys)) * rng.choice([-1.0, 1.0], size=len(keys)), keys))
    gates = [qx.Instruction(g, (int(j),), float(rng.uniform(0.3, 5.9))) for j in qubits for g in ("RX", "RY", "RZ")]
    counts, axes, weights = lut.operator_tables(oracle.lut_blocks(oracle.partition(gates, n), n)[0])
    prog = [lut.perm_op(n, int(qubits[0]), lut.FIXED_PERMS["H"]), lut.cx_op(n, int(qubits[0]), int(qubits[1]))]
    with DeviceStore(n, len(gens), 0) as st:
        st.upload(gens)
        st.apply_operator(counts, axes, weights)
        st.apply_clifford(prog)
        want_ranks = st.merge(1e-12)
        want = [(l.copy(), k.copy()) for l, k in st.segments()]
    before = _native.bucket_enable(bucket)
    try:
        with DeviceStore(n, len(gens), 0) as st:
            st.upload(gens)
            _, ranks = st.apply_operator_run(counts, axes, weights, prog, 1e-12)
            info, cap = _native.dense_last(), _native.bucket_last()["cap"]
            got = [(l.copy(), k.copy()) for l, k in st.segments()]
    finally:
        _native.bucket_enable(before)
    if bucket and cap > 0:
        assert info["kron_groups"] == 0           # the bucketed step took it: its sums stay in source order
    else:
        assert info["kron_groups"] >= 1 and info["kron_sources"] >= count // 2, info
    assert ranks == want_ranks
    for (gl, gk), (wl, wk) in zip(got, want):
        assert np.array_equal(gk, wk)
        assert np.max(np.abs(gl - wl)) < 1e-11


def test_operator_run_with_corrupted_cx_table_is_table_driven():
    """A CX table that is not the conjugation (mutation test, reference tests/test_cli.py:198-203)
    must not be 'repaired' by the homomorphism shortcut: the call falls back to the table-driven
    three-step sequence and reproduces the corrupted result."""
    rng = np.random.default_rng(77)
    n = 8
    lam, keys = random_terms(rng, n, 200, 200)
    keys = np.unique(keys)
    lam = lam[: len(keys)]
    gates = [qx.Instruction("RY", (j,), 0.3 + j) for j in range(5)]
    block = oracle.lut_blocks(oracle.partition(gates, n), n)[0]
    counts, axes, weights = lut.operator_tables(block)
    prog = [lut.cx_op(n, 0, 1), lut.cx_op(n, 1, 2), lut.perm_op(n, 2, lut.FIXED_PERMS["H"]), lut.cx_op(n, 2, 3)]
    bad = np.array(lut.LUT_SIGN).copy()
    bad[1, 0] = -1
    outs = []
    for fused in (False, True):
        with DeviceStore(n, 1, 0) as st:
            st.set_cx_tables(bad)
            st.upload([(lam, keys)])
            if fused:
                st.apply_operator_run(counts, axes, weights, prog, 1e-12)
            else:
                st.apply_operator(counts, axes, weights)
                st.apply_clifford(prog)
                st.merge(1e-12)
            outs.append([(l.copy(), k.copy()) for l, k in st.segments()][0])
    assert np.array_equal(outs[0][1], outs[1][1]) and np.array_equal(outs[0][0], outs[1][0])
    with DeviceStore(n, 1, 0) as st:
        st.upload([(lam, keys)])
        st.apply_operator_run(counts, axes, weights, prog, 1e-12)
        good = [(l.copy(), k.copy()) for l, k in st.segments()][0]
    assert not np.array_equal(good[0], outs[0][0])
