"""The drop rule at its boundary (reference stabilizer.py:336: keep iff |sum| >= eps).

eps is a parameter, so a term can be put EXACTLY on the boundary: take the coefficient v of some
output term from a first run and run again with eps = |v|.  The reference keeps that term
(>=) and drops every term one unit in the last place below it.

* Paths whose sums are associated like the reference's -- raw expansion + sort + in-order reduce,
  the grouped step for groups below 64 sources, the bucketed step -- are bitwise the reference's,
  so they must keep/drop EXACTLY the same terms for every such eps (checked on terms sitting on
  the boundary and on their nearest neighbours in value).
* The factored sum of the grouped step (groups of >= 64 sources, dense.cu: sources that share
  their high digits share the high product; or, where that is cheaper, the whole group contracted
  one qubit at a time, k_group_kron / k_kron_mode) associates the products differently: its
  coefficients are within rounding of the reference's, not bitwise, and a term whose reference
  value IS eps can come out one ulp below and be dropped.  The test below documents exactly
  that: every difference between the two term sets is a term whose two values straddle eps and
  differ by rounding (< 1e-13 here); away from the boundary the sets agree.  (With the default eps = 1e-12 the
  chance that one of ~1e8 sums lies within 1e-16 relative of eps is ~1e-8 per run: never seen in
  any campaign, but not excluded -- DESIGN.md section 4.)"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import DeviceStore, oracle, qx  # noqa: E402

from paper_2505_03307_b200 import _native, lut  # noqa: E402


def _tables(n, rng):
    gates = [qx.Instruction(g, (j,), float(rng.uniform(0.3, 5.9))) for j in range(n) for g in ("RX", "RY", "RZ")]
    return lut.operator_tables(oracle.lut_blocks(oracle.partition(gates, n), n)[0])


def _full_support_sources(n, count, rng):
    digits = rng.integers(1, 4, size=(count * 2, n))
    keys = np.unique((digits.astype(np.uint64) << (np.uint64(2) * np.arange(n, dtype=np.uint64)[::-1])).sum(axis=1))[:count]
    return rng.uniform(0.2, 1.0, size=len(keys)) * rng.choice([-1.0, 1.0], size=len(keys)), keys


def _three_steps(n, gens, tables, eps):
    with DeviceStore(n, len(gens), 0) as st:
        st.upload(gens)
        st.apply_operator(*tables)
        st.merge(eps)
        return [(l.copy(), k.copy()) for l, k in st.segments()]


def _fused(n, gens, tables, eps, bucket):
    before = _native.bucket_enable(bucket)
    try:
        with DeviceStore(n, len(gens), 0) as st:
            st.upload(gens)
            st.apply_operator_run(*tables, [], eps)
            return [(l.copy(), k.copy()) for l, k in st.segments()], _native.bucket_last()
    finally:
        _native.bucket_enable(before)


def test_bitwise_paths_keep_and_drop_exactly_the_reference_terms():
    rng = np.random.default_rng(41)
    n = 10
    gens = [_full_support_sources(n, 3, rng), _full_support_sources(n, 1, rng)]
    tables = _tables(n, rng)
    (lam0, keys0), _ = _three_steps(n, gens, tables, 1e-300)
    mags = np.sort(np.abs(lam0))
    for pick in (len(mags) // 7, len(mags) // 2, len(mags) - 5):
        for eps in (mags[pick], np.nextafter(mags[pick], 1.0), np.nextafter(mags[pick], 0.0)):
            want = _three_steps(n, gens, tables, float(eps))
            assert len(want[0][0]) == int(np.sum(np.abs(lam0) >= eps))            # the boundary term itself is kept
            grouped, _ = _fused(n, gens, tables, float(eps), bucket=False)
            bucketed, info = _fused(n, gens, tables, float(eps), bucket=True)
            assert info["cap"] > 0
            for got in (grouped, bucketed):
                for (gl, gk), (wl, wk) in zip(got, want):
                    assert np.array_equal(gk, wk) and np.array_equal(gl, wl)


def test_factored_sums_differ_from_the_reference_only_on_the_boundary():
    rng = np.random.default_rng(43)
    n = 9
    gens = [_full_support_sources(n, 200, rng)]          # one group of 200 sources: the factored sum
    tables = _tables(n, rng)
    (lam_e, keys_e), = _three_steps(n, gens, tables, 1e-300)
    ((lam_f, keys_f),), _ = _fused(n, gens, tables, 1e-300, bucket=False)
    assert np.array_equal(keys_e, keys_f)
    # 200 contributions of magnitude <= 1 per slot: rounding of the sum ~ 200 * 1.1e-16
    assert np.max(np.abs(lam_e - lam_f)) < 1e-13, "factored sums agree with the reference's to rounding"
    below = np.flatnonzero(np.abs(lam_f) < np.abs(lam_e))
    assert len(below), "some factored sum is smaller in magnitude than the reference's by a last-place unit"
    flips = 0
    for k in below[:: max(1, len(below) // 6)][:6]:
        eps = float(abs(lam_e[k]))                                   # reference: |v| >= eps, kept
        (wl, wk), = _three_steps(n, gens, tables, eps)
        ((fl, fk),), _ = _fused(n, gens, tables, eps, bucket=False)
        assert keys_e[k] in wk
        only_ref = np.setdiff1d(wk, fk)
        only_fac = np.setdiff1d(fk, wk)
        flips += len(only_ref) + len(only_fac)
        for key in np.concatenate([only_ref, only_fac]):
            i = int(np.searchsorted(keys_e, key))
            lo, hi = sorted((abs(lam_e[i]), abs(lam_f[i])))
            assert lo < eps <= hi and (hi - lo) < 1e-13                   # straddles eps, rounding apart
        common = np.intersect1d(wk, fk)
        assert len(common) >= len(wk) - len(only_ref)
    assert flips >= 1, "the term put on the boundary flips in the factored path (documented limit)"
