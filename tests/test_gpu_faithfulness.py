"""The reference's own acceptance strategy (its tests/test_acceptance.py
criteria 1, 2, 10, tests/test_stabilizer.py TestApplyCx / TestCanonicalize / TestFlatten /
TestOperatorFaithfulness, tests/test_measure.py) run against the GPU path, with an independent
dense checker (tests/dense_check.py: 2^n x 2^n matrices, no code shared with the package or the
oracle port) in the role of the reference's tests/dense_ref.py.  Everything goes through the public
API and so through the C ABI."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import dense_check as dc  # noqa: E402
from gpu_util import qx  # noqa: E402

from paper_2505_03307_b200 import lut, workloads  # noqa: E402
from paper_2505_03307_b200.stabilizer import SimpleGenerator, branch_counts  # noqa: E402

SEED = 2024          # the reference's campaign seed (tests/test_acceptance.py:25-48)


def _campaign(size, lo=2, hi=6, max_gates=61, seed=SEED):
    for case in range(size):
        rng = np.random.default_rng([seed, case])
        n = int(rng.integers(lo, hi))
        yield n, workloads.gen_random(n, int(rng.integers(1, max_gates)), rng)


def _random_generator(rng, n, terms):
    idx = rng.choice(4 ** n, size=min(terms, 4 ** n), replace=False)
    return SimpleGenerator(n, rng.uniform(-1, 1, size=len(idx)), idx)


# ---------------------------------------------------------------- criterion 1 and 2
def test_generators_equal_conjugated_z_in_every_mode():
    """P_j = U Z_j U^dagger as matrices (tests/test_acceptance.py:51-64), 1e-9 like the reference."""
    worst = 0.0
    for n, gates in _campaign(60):
        for mode in ("v1", "v2", "v3"):
            rep = qx.run(gates, n, mode)
            for j, g in enumerate(rep.final.generators):
                want = dc.conjugate(dc.word(3 * 4 ** (n - 1 - j), n), gates, n)
                worst = max(worst, float(np.abs(dc.generator_matrix(g) - want).max()))
    assert worst < 1e-9, worst


def test_modes_agree_on_the_campaign():
    """Index sets equal, coefficients within 1e-10 (tests/test_acceptance.py:67-74)."""
    for n, gates in _campaign(60):
        _, agreement = qx.run_all_modes(gates, n)
        assert agreement.index_sets_equal and agreement.max_lambda_deviation < 1e-10


# ---------------------------------------------------------------- kernel-level API
@pytest.mark.parametrize("seed", range(6))
def test_apply_cx_is_an_involution_and_a_conjugation(seed):
    """tests/test_stabilizer.py:233-260: twice = identity after canonical ordering, and the matrix
    of the output is CX G CX."""
    rng = np.random.default_rng([7, seed])
    n = int(rng.integers(2, 6))
    g = _random_generator(rng, n, int(rng.integers(1, 12)))
    c, t = (int(v) for v in rng.choice(n, size=2, replace=False))
    once = qx.apply_cx(g, c, t)
    assert once.rank == g.rank
    twice = qx.canonicalize(qx.apply_cx(once, c, t))
    base = qx.canonicalize(g)
    assert list(twice.indices) == list(base.indices) and np.array_equal(twice.lambdas, base.lambdas)
    cx = [qx.Instruction("CX", (c, t))]
    assert np.abs(dc.generator_matrix(once) - dc.conjugate(dc.generator_matrix(g), cx, n)).max() < 1e-12
    with pytest.raises(ValueError):
        qx.apply_cx(g, c, c)


@pytest.mark.parametrize("seed", range(4))
def test_canonicalize_properties(seed):
    """tests/test_stabilizer.py:271-303: merges duplicates, ascending, idempotent, rank <= 4**n."""
    rng = np.random.default_rng([11, seed])
    n = int(rng.integers(1, 4))
    idx = rng.integers(0, 4 ** n, size=300)
    g = SimpleGenerator(n, rng.uniform(-1, 1, size=300), idx)
    out = qx.canonicalize(g)
    assert out.rank <= 4 ** n
    assert list(out.indices) == sorted(set(int(v) for v in out.indices))
    again = qx.canonicalize(out)
    assert list(again.indices) == list(out.indices) and np.array_equal(again.lambdas, out.lambdas)
    assert np.abs(dc.generator_matrix(out) - dc.generator_matrix(g)).max() < 1e-12
    gone = qx.canonicalize(SimpleGenerator(1, [0.5, -0.5], [3, 3]))
    assert gone.rank == 0 and gone.is_degenerate


@pytest.mark.parametrize("seed", range(6))
def test_sub_flatten_equals_dense_conjugation(seed):
    """tests/test_stabilizer.py:306-321: one operator U_k (a block of composed gates per qubit)
    substituted and flattened = conjugation by the tensor product of the gate sequences; both
    layouts agree (:182-188); raw branches = branch_counts <= 3**(non-identity digits) (:190-198)."""
    rng = np.random.default_rng([13, seed])
    n = int(rng.integers(1, 5))
    g = _random_generator(rng, n, int(rng.integers(1, 6)))
    per_wire, gates = [], []
    for q in range(n):
        seq = [qx.Instruction(name, (q,), float(rng.uniform(0, 2 * math.pi)) if name.startswith("R") else 0.0)
               for name in rng.choice(["H", "S", "X", "SX", "RX", "RY", "RZ"], size=int(rng.integers(0, 4)))]
        per_wire.append(seq)
        gates.extend(seq)
    block = np.stack([lut.compose_block(seq) for seq in per_wire])
    ragged = qx.flatten(qx.sub(g, block, "ragged"))
    dense = qx.flatten(qx.sub(g, block, "dense"))
    assert list(ragged.indices) == list(dense.indices)
    assert np.max(np.abs(ragged.lambdas - dense.lambdas), initial=0.0) < 1e-12
    want = dc.conjugate(dc.generator_matrix(g), gates, n)
    assert np.abs(dc.generator_matrix(ragged) - want).max() < 1e-10
    raw = qx.flatten(qx.sub(g, block), canonical=False)
    counts = branch_counts(qx.sub(g, block))
    assert raw.rank == int(counts.sum())
    weight = [sum(1 for j in range(n) if (int(i) >> (2 * j)) & 3) for i in g.indices]   # non-identity digits
    assert int(counts.sum()) <= sum(3 ** w for w in weight)
    assert np.abs(dc.generator_matrix(raw) - want).max() < 1e-10          # unmerged list: same operator


def test_dense_layout_guards():
    """tests/test_stabilizer.py:200-215: the dense layout refuses a branching expansion above its
    4**10 budget and keeps one-hot rows cheap at any n."""
    n = 12
    block = np.broadcast_to(lut.axis_map("RY", 0.9).T, (n, 3, 3)).copy()
    g = SimpleGenerator(n, [1.0], [(4 ** n - 1) // 3])                       # XX...X
    with pytest.raises(qx.ResourceLimitError):
        qx.flatten(qx.sub(g, block, "dense"))
    n = 20
    eye = np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
    out = qx.flatten(qx.sub(qx.init_z(n).generators[0], eye, "dense"))
    assert list(out.indices) == [3 * 4 ** (n - 1)] and out.lambdas.tolist() == [1.0]


# ---------------------------------------------------------------- read-out
def test_expansion_equals_the_projector_and_is_a_pure_state():
    """tests/test_measure.py:39-58: the expansion is |psi><psi| in the Pauli basis; trace 1, purity 1."""
    for n, gates in _campaign(12, lo=1, hi=5, max_gates=41, seed=SEED + 2):
        final = qx.run(gates, n, "v3").final
        ex = qx.density_expansion(final)
        psi = dc.state(gates, n)
        rho = np.outer(psi, psi.conj())
        got = np.zeros_like(rho)
        for idx, c in ex.coeffs.items():
            got += c * dc.word(idx, n)
        assert np.abs(got - rho).max() < 1e-10
        assert abs(2 ** n * ex.coeff(0) - 1.0) < 1e-12                        # only I...I has a trace
        assert abs(2 ** n * sum(c * c for c in ex.coeffs.values()) - 1.0) < 1e-10


def test_prob_z_and_expectation_against_the_state_vector():
    """tests/test_acceptance.py:169-183 (criterion 10): 100 circuits, both read-out routes, 1e-9."""
    worst = 0.0
    for n, gates in _campaign(100, lo=1, hi=5, max_gates=41, seed=SEED + 1):
        final = qx.run(gates, n, "v3").final
        ex = qx.density_expansion(final)
        psi = dc.state(gates, n)
        for k in range(n):
            p0, p1 = qx.prob_z(final, k, ex)
            assert p0 + p1 == 1.0                                            # tests/test_measure.py:113-121
            via = 0.5 * (1.0 + qx.expectation(final, 3 * 4 ** (n - 1 - k), ex))
            want = dc.prob_zero(psi, k, n)
            worst = max(worst, abs(p0 - want), abs(via - want))
    assert worst < 1e-9, worst


@pytest.mark.parametrize("theta", [0.0, 0.3, math.pi / 2, 2.0, math.pi, 5.1])
def test_bloch_rotation_closed_form(theta):
    """tests/test_measure.py:147-150: <Z> = cos(theta) after RX or RY, <Y> = -sin, <X> = sin."""
    for gate, axis, sign in (("RX", 2, -1.0), ("RY", 1, 1.0)):
        final = qx.run([qx.Instruction(gate, (0,), theta)], 1, "v3").final
        assert abs(qx.expectation(final, 3) - math.cos(theta)) < 1e-12
        assert abs(qx.expectation(final, axis) - sign * math.sin(theta)) < 1e-12


@pytest.mark.parametrize("n", [2, 3, 6, 10])
def test_ghz_is_unbiased_and_correlated(n):
    """tests/test_measure.py:97-106,143-145: every qubit 50/50, <Z_0 Z_k> = 1."""
    final = qx.run(qx.gen_ghz(n), n, "v3").final
    ex = qx.density_expansion(final)
    for k in range(n):
        assert qx.prob_z(final, k, ex) == (0.5, 0.5)
    for k in range(1, n):
        assert qx.expectation(final, 3 * 4 ** (n - 1) + 3 * 4 ** (n - 1 - k), ex) == 1.0
    assert qx.expectation(final, 0, ex) == 1.0
    with pytest.raises(ValueError):
        qx.prob_z(final, n, ex)
    with pytest.raises(ValueError):
        qx.expectation(final, 4 ** n, ex)
