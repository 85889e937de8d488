"""The bucketed operator step (csrc/bucket.cuh: slots leave the kernel in canonical order, no sort)
against the three-step sequence qx_apply_operator + qx_apply_clifford + qx_merge (raw expansion,
table-driven Clifford kernel, radix sort + in-order reduce -- itself checked against the oracle in
test_gpu_kernels.py) and against the grouped step + sort it replaces: bit for bit, keys and
coefficients (reference semantics: stabilizer.py:289-337 products qubit 0 first, sources in input
order, drop rule |sum| >= eps, ascending unique keys).

Cases are built so that every branch of the kernel runs: one and two sources per group (the fast
table path), three and more (further sources straight from the operator table), classes of radix
1 / 2 / 3, buckets of more than three tiles (parked), 64-bit working keys (n > 16), no Clifford
run behind the operator, a CX ladder behind it, narrow (32-bit) output, parts of a partitioned
run, and operators the planner must refuse (a ladder running the other way)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import DeviceStore, oracle, qx  # noqa: E402

from paper_2505_03307_b200 import _native, lut  # noqa: E402


def _block(n, rng, gates_per_qubit):
    """(n,3,3) block of an operator: gates_per_qubit[j] = list of rotation names on qubit j."""
    gates = [qx.Instruction(g, (j,), float(rng.uniform(0.3, 5.9))) for j, gs in enumerate(gates_per_qubit) for g in gs]
    return oracle.lut_blocks(oracle.partition(gates, n), n)[0] if gates else np.tile(np.eye(3), (n, 1, 1))


def _ladder(n, lo, hi, reverse=False):
    pairs = [(q, q + 1) for q in range(lo, hi)]
    if reverse:
        pairs = [(t, c) for c, t in reversed(pairs)]
    return [lut.cx_op(n, c, t) for c, t in pairs]


def _word(n, axes):
    """key of the word with axis code axes[j] on qubit j"""
    k = 0
    for j, a in enumerate(axes):
        k |= int(a) << (2 * (n - 1 - j))
    return np.uint64(k)


def _three_steps(n, gens, tables, prog, eps):
    with DeviceStore(n, len(gens), 0) as st:
        st.upload(gens)
        st.apply_operator(*tables)
        st.apply_clifford(prog)
        ranks = st.merge(eps)
        return ranks, [(l.copy(), k.copy()) for l, k in st.segments()]


def _run(n, gens, tables, prog, eps, bucket, part=None):
    before = _native.bucket_enable(bucket)
    try:
        with DeviceStore(n, len(gens), 0) as st:
            st.upload(gens)
            if part is None:
                _, ranks = st.apply_operator_run(*tables, prog, eps)
            else:
                ranks, _ = st.apply_operator_run_part(*tables, prog, eps, *part)
            out = [(l.copy(), k.copy()) for l, k in st.segments()]
        return ranks, out, _native.bucket_last()
    finally:
        _native.bucket_enable(before)


def _assert_same(got, want, exact=True):
    assert len(got) == len(want)
    for (gl, gk), (wl, wk) in zip(got, want):
        assert np.array_equal(gk, wk)
        if exact:
            assert np.array_equal(gl, wl)
        else:
            assert np.max(np.abs(gl - wl), initial=0.0) < 1e-12


CASES = {
    # name: (n, supports of the sources of each generator as axis strings, rotations per qubit, program)
    "one_source_full_mixing": dict(n=12, gens=[["ZZZZZZZZZZZZ"], ["IXYZXYZXYZXY"], ["IIIIIIZZZZZZ"]],
                                   rot=["RX", "RY", "RZ"], prog="ladder"),
    "two_sources_one_group": dict(n=12, gens=[["XXXXXXXXXXXX", "YXXXXXXXXXXX"], ["ZZZZZZZZZZZI", "ZZZZZZZZZZZX", "IIIIZZZZZZZZ"]],
                                  rot=["RX", "RZ"], prog="ladder"),
    "five_sources_one_group": dict(n=11, gens=[["XXXXXXXXXXX", "YXXXXXXXXXX", "ZXXXXXXXXXX", "XYXXXXXXXXX", "XZXXXXXXXXX"]],
                                   rot=["RY", "RZ", "RX"], prog="ladder"),
    "no_program": dict(n=11, gens=[["XYZXYZXYZXY"], ["ZZZZZZZZZZZ", "YYYYYYYYYYY"]], rot=["RZ", "RY"], prog=None),
    "radix_two_classes": dict(n=16, gens=[["XYXYXYXYXYXYXYXY"], ["YYYYYYYYYYYYYYYY", "XXXXXXXXXXXXXXXX"]], rot=["RZ"], prog=None),
    "mixed_radix": dict(n=16, gens=[["XYZXYZXYZXYZXYZX"], ["ZZZZZZZZZZZZZZZZ", "XXXXXXXXXXXXXXXX"]], rot="mixed", prog=None),
    "partial_ladder": dict(n=12, gens=[["ZZZZZZZZZZZZ"], ["XXXXXXXXXXXX"]], rot=["RX", "RY"], prog="ladder_low"),
    "clifford_1q_and_ladder": dict(n=12, gens=[["ZYXZYXZYXZYX"], ["XXXXXXIIIIII", "IIIIIIXXXXXX"]], rot=["RY", "RZ"], prog="ladder_hs"),
    "many_tiles_per_bucket": dict(n=12, gens=[["ZZZZZZZZZZZZ", "ZZZZZZZZZIII", "ZZZZZZZZIIZI", "ZZZZZZZZIIZZ"]], rot=["RX", "RY"], prog=None),
    "sixty_four_bit_keys": dict(n=18, gens=[["IIIIIIXYZXYZXYZXYZ"], ["ZZIIIIIZZZZZZZZZZZ", "ZZIIIIIYYYYYYYYYYY"]], rot=["RX", "RZ"], prog="ladder"),
    "reverse_ladder_refused": dict(n=12, gens=[["ZZZZZZZZZZZZ"], ["XYZXYZXYZXYZ"]], rot=["RX", "RY"], prog="reverse"),
}


def _build(case, seed):
    rng = np.random.default_rng(seed)
    n = case["n"]
    code = {"I": 0, "X": 1, "Y": 2, "Z": 3}
    gens = []
    for words in case["gens"]:
        keys = np.array(sorted({int(_word(n, [code[c] for c in w])) for w in words}), dtype=np.uint64)
        gens.append((rng.uniform(0.2, 1.0, size=len(keys)) * rng.choice([-1.0, 1.0], size=len(keys)), keys))
    if case["rot"] == "mixed":
        pool = [["RX", "RY"], ["RZ"], ["RY", "RX"], ["RY"], ["RX", "RZ", "RY"], ["RX"]]
        per_qubit = [pool[j % len(pool)] for j in range(n)]
    else:
        per_qubit = [list(case["rot"]) for _ in range(n)]
    tables = lut.operator_tables(_block(n, rng, per_qubit))
    prog = {None: [], "ladder": _ladder(n, 0, n - 1), "ladder_low": _ladder(n, n // 2, n - 1),
            "reverse": _ladder(n, 0, n - 1, reverse=True),
            "ladder_hs": [lut.perm_op(n, q, lut.FIXED_PERMS[g]) for q, g in ((n - 1, "H"), (n - 2, "S"), (n - 3, "SX"))]
                         + _ladder(n, 0, n - 1)}[case["prog"]]
    return n, gens, tables, prog


@pytest.mark.parametrize("name", sorted(CASES))
def test_bucketed_step_is_bitwise_the_three_step_sequence(name):
    n, gens, tables, prog = _build(CASES[name], seed=len(name))
    eps = 1e-12
    want_ranks, want = _three_steps(n, gens, tables, prog, eps)
    ranks_g, grouped, _ = _run(n, gens, tables, prog, eps, bucket=False)
    ranks_b, bucketed, info = _run(n, gens, tables, prog, eps, bucket=True)
    assert ranks_g == want_ranks and ranks_b == want_ranks
    _assert_same(grouped, want)
    _assert_same(bucketed, want)
    if name == "reverse_ladder_refused":
        assert info["cap"] == 0, "a ladder whose images reach the top bits must take the grouped step + sort"
    else:
        assert info["cap"] > 0, f"{name}: the bucketed step did not run ({info})"
    for lam, keys in bucketed:
        assert np.all(np.diff(keys.astype(np.uint64)) > 0)


def test_large_eps_drops_whole_buckets_and_generators():
    """Drop rule inside the kernel: an eps that removes most slots (and one generator entirely)
    gives the same term sets, ranks and collapse as the three-step sequence."""
    n, gens, tables, prog = _build(CASES["one_source_full_mixing"], seed=5)
    gens[2] = (gens[2][0] * 1e-9, gens[2][1])
    eps = 1e-4
    want_ranks, want = _three_steps(n, gens, tables, prog, eps)
    ranks, got, info = _run(n, gens, tables, prog, eps, bucket=True)
    assert info["cap"] > 0 and ranks == want_ranks and want_ranks[2] == 0
    assert 0 < sum(want_ranks) < 0.8 * info["slots"]
    _assert_same(got, want)


@pytest.mark.parametrize("parts", [2, 3, 5])
def test_parts_of_a_partitioned_run_are_disjoint_key_ranges(parts):
    """qx_apply_operator_run_part on the bucketed step: part p works off a contiguous range of
    buckets, i.e. of (generator, key) order; the shares are disjoint and their union is the result."""
    n, gens, tables, prog = _build(CASES["two_sources_one_group"], seed=9)
    eps = 1e-12
    want_ranks, want = _three_steps(n, gens, tables, prog, eps)
    shares = [_run(n, gens, tables, prog, eps, bucket=True, part=(p, parts)) for p in range(parts)]
    assert all(info["cap"] > 0 for _, _, info in shares)
    for g in range(len(gens)):
        lam = np.concatenate([out[g][0] for _, out, _ in shares])
        keys = np.concatenate([out[g][1] for _, out, _ in shares])
        assert np.array_equal(keys, want[g][1]) and np.array_equal(lam, want[g][0])
    assert [sum(r[g] for r, _, _ in shares) for g in range(len(gens))] == want_ranks


def test_narrow_output_for_download():
    """A store that is only downloaded next keeps 32-bit keys (qx_store_set_keep_narrow): the
    bucketed step writes them directly; the download widens them on the host."""
    n, gens, tables, prog = _build(CASES["one_source_full_mixing"], seed=3)
    want_ranks, want = _three_steps(n, gens, tables, prog, 1e-12)
    with DeviceStore(n, len(gens), 0) as st:
        st.upload(gens)
        st.set_keep_narrow(1)
        _, ranks = st.apply_operator_run(*tables, prog, 1e-12)
        info = _native.bucket_last()
        off, keys, lam = st.download_async(True)
        st.synchronize()
        got = [(lam[off[i]:off[i + 1]].copy(), keys[off[i]:off[i + 1]].copy()) for i in range(len(gens))]
    assert info["cap"] > 0 and ranks == want_ranks
    _assert_same(got, want)


def test_engine_results_do_not_depend_on_the_bucketed_step():
    """Public API: xyz_chain(12, 2) in v3 with the bucketed step on and off, bit for bit; and the
    oracle on the same circuit within 1e-10 (keys exact)."""
    n = 12
    circ = qx.gen_xyz_chain(n, 2, 1, rng=4)
    before = _native.bucket_enable(True)
    try:
        on = qx.run(circ, n, "v3", device=0)
        took = _native.bucket_last()["cap"] > 0
        _native.bucket_enable(False)
        off = qx.run(circ, n, "v3", device=0)
    finally:
        _native.bucket_enable(before)
    assert took and on.rank_trace == off.rank_trace
    for a, b in zip(on.final.generators, off.final.generators):
        assert np.array_equal(a.keys(), b.keys()) and np.array_equal(a.lambdas, b.lambdas)
    want = oracle.run(circ, n, "v3")
    for g, (lam, idx) in zip(on.final.generators, want["final"]):
        assert np.array_equal(g.keys(), idx) and np.max(np.abs(g.lambdas - lam)) < 1e-10
