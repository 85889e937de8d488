"""More than 32 qubits on the GPU (multi-word keys, csrc/wide.cu) against fixtures computed by the
UNMODIFIED reference with Python big-int indices (tests/golden/wide.json, oracle/make_golden_wide.py):
Clifford circuits up to 130 qubits in v1 and v3, near-Clifford circuits in v1 and v3, the apply_cx unit
case; plus the multi-word merge/split against a big-int model on random terms, and the limits
above 32 qubits."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import DeviceStore, qx  # noqa: E402

from paper_2505_03307_b200 import lut  # noqa: E402
from paper_2505_03307_b200.stabilizer import SimpleGenerator, split_tables  # noqa: E402

TOL = 1e-10


def _cases(golden):
    return golden.load_json("wide.json")


def test_reference_circuits_above_32_qubits(golden):
    data = _cases(golden)
    assert len(data["cases"]) >= 18
    for case in data["cases"]:
        n = case["n"]
        gates = [qx.Instruction(g, tuple(w), float.fromhex(t)) for g, w, t in case["gates"]]
        rep = qx.run(gates, n, case["mode"])
        assert rep.rank_trace[-1] == case["rank_trace_last"], case["name"]
        for g, want in zip(rep.final.generators, case["final"]):
            assert g.indices.dtype == object
            assert [int(v) for v in g.indices] == [int(v) for v in want["idx"]], case["name"]
            lam = np.array([float.fromhex(v) for v in want["lam"]])
            if case["max_rank"] == 1:
                assert np.array_equal(g.lambdas, lam), case["name"]          # Clifford: exactly +-1
            else:
                assert np.max(np.abs(g.lambdas - lam)) < TOL, case["name"]


def test_apply_cx_big_int_unit(golden):
    u = _cases(golden)["apply_cx"]
    g = SimpleGenerator(u["n"], u["in"]["lam"], [int(v) for v in u["in"]["idx"]])
    out = qx.apply_cx(g, u["c"], u["t"])
    assert [int(v) for v in out.indices] == [int(v) for v in u["out"]["idx"]]
    assert out.lambdas.tolist() == u["out"]["lam"]


@pytest.mark.parametrize("n,terms", [(40, 3000), (70, 1500), (130, 900), (40, 60000), (100, 20000), (130, 9000)])
def test_split_and_merge_against_big_int_model(n, terms):
    """qx_apply_split_wide + the multi-word merge on random terms (the store grows past its first
    allocation on the way) against the reference's v1 rule done with Python ints."""
    rng = np.random.default_rng(n)
    keys = sorted({int.from_bytes(rng.bytes((2 * n + 7) // 8), "little") % 4 ** n for _ in range(terms)})
    lam = rng.uniform(-1, 1, size=len(keys))
    q, theta = n // 3, 0.77
    block = lut.gate_branch_block("RY", theta)
    a1, w1, a2, w2 = split_tables(block)
    sh = 2 * (n - 1 - q)
    model = {}
    for k, l in zip(keys, lam):                                   # firsts then seconds, engine.py:211-217
        d = (k >> sh) & 3
        base = k & ~(3 << sh)
        model[base | (int(a1[d]) << sh)] = model.get(base | (int(a1[d]) << sh), 0.0) + l * w1[d]
    for k, l in zip(keys, lam):
        d = (k >> sh) & 3
        if w2[d] != 0.0:
            base = k & ~(3 << sh)
            model[base | (int(a2[d]) << sh)] = model.get(base | (int(a2[d]) << sh), 0.0) + l * w2[d]
    want = sorted((k, v) for k, v in model.items() if abs(v) >= 1e-12)
    with DeviceStore(n, 2, 0) as st:
        obj = np.empty(len(keys), dtype=object)
        obj[:] = keys
        st.upload([(lam, obj), (lam[:1], obj[:1])])
        st.apply_split(q, a1, w1, a2, w2)
        ranks = st.merge(1e-12)
        (gl, gk), _ = st.segments()
        norms = st.norms()
    assert ranks[0] == len(want) and [int(v) for v in gk] == [k for k, _ in want]
    assert np.max(np.abs(gl - np.array([v for _, v in want]))) < 1e-12
    assert abs(norms[0] - sum(v * v for _, v in want)) < 1e-9


@pytest.mark.parametrize("n,sizes,pool", [(40, (50000, 0, 7, 20000), 9000), (70, (3, 30000, 30000), 50000),
                                          (200, (12000, 1), 4000)])
def test_large_multiword_merge_sums_runs_in_input_order(n, sizes, pool):
    """Generators beyond one CTA's shared memory: permutation sorted word by word (stable LSD over
    the words), then one reduce pass.  Raw terms drawn from a small pool of words (runs of many
    duplicates), some in exactly cancelling pairs; sums must be BITWISE what sequential addition
    in input order gives (np.add.at, reference stabilizer.py:333-335), empty generators included."""
    rng = np.random.default_rng([n, pool])
    words = [int.from_bytes(rng.bytes((2 * n + 7) // 8), "little") % 4 ** n for _ in range(pool)]
    words[0], words[1] = 0, 4 ** n - 1                            # extremes of the key range
    segs, want = [], []
    for size in sizes:
        pick = rng.integers(0, pool, size=size)
        lam = rng.uniform(-1, 1, size=size)
        for j in range(0, size - 1, 7):                           # cancelling pairs -> dropped or partial
            pick[j + 1], lam[j + 1] = pick[j], -lam[j]
        obj = np.empty(size, dtype=object)
        obj[:] = [words[p] for p in pick]
        segs.append((lam, obj))
        model = {}
        for k, l in zip(obj, lam):
            model[k] = model.get(k, 0.0) + float(l)
        want.append(sorted((k, v) for k, v in model.items() if abs(v) >= 1e-12))
    with DeviceStore(n, len(sizes), 0) as st:
        st.upload(segs)
        ranks = st.merge(1e-12)
        got = st.segments()
    assert list(ranks) == [len(w) for w in want]
    for (gl, gk), w in zip(got, want):
        assert [int(v) for v in gk] == [k for k, _ in w]
        assert gl.tolist() == [v for _, v in w]                   # bitwise


@pytest.mark.parametrize("n,mode", [(36, "v1"), (36, "v3"), (70, "v3")])
def test_high_rank_circuit_embedded_above_32_qubits(n, mode):
    """The whole multi-word pipeline at a rank where every merge is the large one (generators of
    up to 7.9e4 terms): xyz_chain(10,2) on the first ten of n qubits must give the one-word run's
    generators with every word shifted by the idle qubits (word * 4**(n-10)); the one-word path is
    itself pinned on the reference (tests/test_gpu_configs.py)."""
    from paper_2505_03307_b200 import workloads
    gates = workloads.gen_xyz_chain(10, 2, 1, 4)
    narrow = qx.run(gates, 10, mode)
    wide = qx.run(gates, n, mode)
    assert wide.rank_trace[-1][:10] == narrow.rank_trace[-1] and set(wide.rank_trace[-1][10:]) == {1}
    shift = 4 ** (n - 10)
    for gw, gn in zip(wide.final.generators, narrow.final.generators):
        assert [int(v) for v in gw.indices] == [int(v) * shift for v in gn.indices]
        assert np.max(np.abs(gw.lambdas - gn.lambdas)) < 1e-12
    if mode == "v3":
        # the operators ran as grouped one-word steps on the generators' support (qx_store_compact /
        # qx_store_expand): same kernels, same order of every sum as the one-word run -- bit for bit
        assert wide.device.get("compacted_operators", 0) == 2
        for gw, gn in zip(wide.final.generators, narrow.final.generators):
            assert np.array_equal(gw.lambdas, gn.lambdas)
    for j in range(10, n):
        g = wide.final.generators[j]
        assert [int(v) for v in g.indices] == [3 * 4 ** (n - 1 - j)] and g.lambdas.tolist() == [1.0]


def test_long_single_wire_operator_above_32_qubits():
    """Forty rotations on ONE wire inside one operator: the multi-word walk doubles the raw list per
    split and must sum duplicates in between (found by tools/fuzz_wide.py: it ran out of memory)."""
    n = 70
    rng = np.random.default_rng(3)
    gates = [qx.Instruction(str(rng.choice(["RX", "RY", "RZ"])), (0,), float(rng.uniform(0, 6.3))) for _ in range(40)]
    narrow = qx.run(gates, 1, "v3")
    wide = qx.run(gates, n, "v3")
    assert wide.rank_trace[-1] == narrow.rank_trace[-1] + [1] * (n - 1)
    g, want = wide.final.generators[0], narrow.final.generators[0]
    assert [int(v) for v in g.indices] == [int(v) * 4 ** (n - 1) for v in want.indices]
    assert np.max(np.abs(g.lambdas - want.lambdas)) < 1e-12


def test_limits_above_32_qubits():
    n = 36
    gates = [qx.Instruction("H", (0,)), qx.Instruction("RY", (0,), 0.3), qx.Instruction("CX", (0, 35))]
    with pytest.raises(qx.ResourceLimitError, match="dense flatten"):
        qx.run(gates, n, "v2")                                    # reference stabilizer.py:264-276
    # ... but only for rows that are not one-hot: RZ leaves every Z_j alone (dense fast path)
    calm = [qx.Instruction("RZ", (3,), 0.4), qx.Instruction("CX", (3, 4)), qx.Instruction("RZ", (4,), 1.1)]
    assert qx.run(calm, n, "v2").rank_trace[-1] == [1] * n
    for mode in ("v1", "v3"):
        rep = qx.run(gates, n, mode)
        assert rep.rank_trace[-1][0] == 2 and rep.final.generators[35].rank == 1
    with pytest.raises(qx.NativeError, match="at most"):
        qx.run([qx.Instruction("H", (0,))], 600, "v1")
    ghz = qx.run(qx.gen_ghz(400), 400, "v1")                      # "hundreds of qubits for Clifford"
    assert ghz.max_rank == 1 and int(ghz.final.generators[0].indices[0]) == (4 ** 400 - 1) // 3
    with DeviceStore(n, 1, 0) as st:
        st.init_z([0])
        assert st.zi_sums().tolist() == [1.0]                     # Z_0: no X/Y digit in any key word
        with pytest.raises(qx.NativeError, match="one-word keys"):
            st.partition_by_owner(2)


@pytest.mark.parametrize("n,mode", [(40, "v1"), (70, "v1"), (70, "v3")])
def test_heisenberg_read_out_above_32_qubits(n, mode):
    """<0|U^dag W U|0> with multi-word keys (north star kernel 4 at any width): a near-Clifford
    circuit on the first m of n qubits and observables supported there must give the one-word
    read-out's values; words reaching into the idle qubits are 1 on Z/I digits there and 0 on X/Y."""
    m = 8
    gates = qx.gen_random(m, 80, 11)
    rng = np.random.default_rng(5)
    small = [int(v) for v in rng.integers(0, 4 ** m, size=24)] + [0, 4 ** m - 1]
    want = qx.expectation_heisenberg(gates, m, small, mode)
    shift = 4 ** (n - m)
    got = qx.expectation_heisenberg(gates, n, [w * shift for w in small], mode)
    assert np.max(np.abs(got - want)) < 1e-12
    assert np.max(np.abs(want)) > 1e-3                            # the comparison is not 0 == 0
    z_tail = sum(3 * 4 ** (n - 1 - j) for j in (m, n // 2, n - 1))          # Z on three idle qubits
    x_tail = 1 * 4 ** (n - 1 - (n - 2))                                     # X on one idle qubit
    got = qx.expectation_heisenberg(gates, n, [w * shift + z_tail for w in small] + [small[0] * shift + x_tail], mode)
    assert np.max(np.abs(got[:-1] - want)) < 1e-12 and got[-1] == 0.0


def test_heisenberg_read_out_of_a_wide_clifford_state():
    """GHZ on 100 qubits: stabilizers Z_i Z_j and X...X have expectation exactly 1, single Z exactly 0."""
    n = 100
    gates = qx.gen_ghz(n)
    digit = lambda a, j: a * 4 ** (n - 1 - j)
    words = [digit(3, 0) + digit(3, 99), digit(3, 17) + digit(3, 64), (4 ** n - 1) // 3, digit(3, 5),
             digit(1, 0), 0]
    got = qx.expectation_heisenberg(gates, n, words, "v1")
    assert got.tolist() == [1.0, 1.0, 1.0, 0.0, 0.0, 1.0]



def test_compact_and_expand_round_trip_on_a_segment_subset():
    """qx_store_support / qx_store_compact / qx_store_expand against a big-int model: supports per
    segment, taken segments packed over the selected qubits in order, the others left alone."""
    n, rng = 90, np.random.default_rng(11)
    sel = sorted(rng.choice(n, size=20, replace=False).tolist())
    segs, take = [], []
    for g in range(7):
        inside = g % 3 != 1
        pool = sel if inside else list(range(n))
        size = int(rng.integers(0 if g == 4 else 1, 400))
        words = set()
        while len(words) < size:
            w = 0
            for q in rng.choice(pool, size=int(rng.integers(1, 9)), replace=False):
                w |= int(rng.integers(1, 4)) << (2 * (n - 1 - int(q)))
            words.add(w)
        obj = np.empty(size, dtype=object)
        obj[:] = sorted(words)
        segs.append((rng.uniform(-1, 1, size=size), obj))
        take.append(inside)
    with DeviceStore(n, len(segs), 0) as st:
        st.upload(segs)
        masks = st.support()
        for (lam, keys), m in zip(segs, masks):
            want = 0
            for k in keys:
                for q in range(n):
                    if (int(k) >> (2 * (n - 1 - q))) & 3:
                        want |= 1 << q
            assert m == want
        narrow = st.compact(sel, take)
        try:
            got = narrow.segments()
            for (lam, keys), (nl, nk), t in zip(segs, got, take):
                if not t:
                    assert len(nl) == 0
                    continue
                packed = [sum(((int(k) >> (2 * (n - 1 - q))) & 3) << (2 * (len(sel) - 1 - j)) for j, q in enumerate(sel))
                          for k in keys]
                assert [int(v) for v in nk] == packed and packed == sorted(packed)
                assert np.array_equal(nl, lam)
            narrow.merge(0.0)                                   # a step on the one-word side (order kept: keys unique)
            st.expand_from(narrow, sel, take)
        finally:
            narrow.close()
        back = st.segments()
    for (lam, keys), (bl, bk) in zip(segs, back):
        assert [int(v) for v in bk] == [int(v) for v in keys] and np.array_equal(bl, lam)
    with DeviceStore(n, len(segs), 0) as st:
        st.upload(segs)
        with pytest.raises(ValueError, match="outside the selected"):
            st.compact(sel, [True] * len(segs)).close()


def test_operator_on_support_with_idle_and_clifford_only_generators():
    """v3 above 32 qubits on a circuit whose operators mix rotations with Clifford gates on far
    qubits: generators the operator does not touch are left alone, the others go through the
    one-word grouped step; against the same circuit on relabelled (adjacent) qubits."""
    n = 80
    place = [3, 17, 40, 41, 66, 79]
    rng = np.random.default_rng(21)
    small = qx.gen_random(len(place), 60, rng)
    big = [qx.Instruction(g.gate, tuple(place[w] for w in g.wires), g.theta) for g in small]
    a = qx.run(small, len(place), "v3")
    b = qx.run(big, n, "v3")
    assert b.device.get("compacted_operators", 0) >= 1
    for j, q in enumerate(place):
        ga, gb = a.final.generators[j], b.final.generators[q]
        spread = []
        for v in ga.indices:
            w = 0
            for jj, qq in enumerate(place):
                w |= ((int(v) >> (2 * (len(place) - 1 - jj))) & 3) << (2 * (n - 1 - qq))
            spread.append(w)
        assert [int(v) for v in gb.indices] == spread
        assert np.array_equal(gb.lambdas, ga.lambdas)
    for q in range(n):
        if q not in place:
            g = b.final.generators[q]
            assert [int(v) for v in g.indices] == [3 * 4 ** (n - 1 - q)] and g.lambdas.tolist() == [1.0]


def test_generators_an_operator_leaves_alone_are_still_sorted_at_the_end():
    """Found by tools/fuzz_wide.py: a generator that a compacted operator step does not touch keeps
    the order the last Clifford run left it in -- the deferred re-sort must still happen."""
    from paper_2505_03307_b200 import workloads
    for case in (16865, 17061):
        rng = np.random.default_rng([7, case])
        k = int(rng.integers(1, 9))
        n = int(rng.choice([33, 40, 64, 70, 130]))
        gates = workloads.gen_random(k, int(rng.integers(0, 60 if k <= 6 else 35)), rng)
        narrow, wide = qx.run(gates, k, "v3"), qx.run(gates, n, "v3")
        shift = 4 ** (n - k)
        for gw, gn in zip(wide.final.generators, narrow.final.generators):
            assert [int(v) for v in gw.indices] == [int(v) * shift for v in gn.indices]
            assert np.array_equal(gw.lambdas, gn.lambdas)
