"""CPU tests (no GPU): the host tables of the product and the oracle port against the independent
dense checker (tests/dense_check.py) -- the reference's acceptance criteria 3, 4 and 7
(tests/test_acceptance.py:77-101,130-142) and its differential criterion 1 for the ORACLE, so that
the checker the GPU tests lean on is itself pinned by something that shares no code with it."""

import math
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, ".."))

import dense_check as dc  # noqa: E402
import stabsim_port as oracle  # noqa: E402

from paper_2505_03307_b200 import circuit, lut, workloads  # noqa: E402
from paper_2505_03307_b200.circuit import Instruction  # noqa: E402


def _pauli_components(m):
    """(X, Y, Z) components of a 2x2 Hermitian matrix by trace projection."""
    return np.array([np.trace(m @ dc.PAULI[a]).real / 2 for a in (1, 2, 3)])


@pytest.mark.parametrize("gate", ["H", "S", "X", "SX", "RX", "RY", "RZ"])
def test_single_qubit_maps_equal_dense_conjugation(gate):
    """axis_map(gate, theta)[:, p-1] = components of U P_p U^dagger: 7 gates x 3 axes x 32 angles,
    1e-12 (tests/test_acceptance.py:77-88); product and oracle tables both."""
    for theta in np.linspace(0.0, 2 * math.pi, 32, endpoint=False):
        u = dc.unitary_1q(gate, float(theta))
        for table in (lut.axis_map(gate, float(theta)), oracle.axis_map(gate, float(theta))):
            for p in (1, 2, 3):
                want = _pauli_components(u @ dc.PAULI[p] @ u.conj().T)
                assert np.max(np.abs(np.asarray(table)[:, p - 1] - want)) < 1e-12, (gate, theta, p)


def test_cx_tables_equal_dense_conjugation():
    """All 16 (control, target) axis pairs: CX (P_c x P_t) CX = sign * (P_c' x P_t') exactly
    (tests/test_acceptance.py:91-101, tests/test_lut.py:126-150), and the table is an involution."""
    cx = [Instruction("CX", (0, 1))]
    for c in range(4):
        for t in range(4):
            c2, t2, sign = lut.cx_lookup(c, t)
            got = dc.conjugate(dc.word(4 * c + t, 2), cx, 2)
            assert np.array_equal(got, sign * dc.word(4 * c2 + t2, 2)), (c, t)
            c3, t3, sign3 = lut.cx_lookup(c2, t2)
            assert (c3, t3, sign * sign3) == (c, t, 1)
    assert lut.cx_lookup(1, 3) == (2, 2, -1) and lut.cx_lookup(2, 2) == (1, 3, -1)   # the two minus signs


def test_composed_blocks_equal_the_product_of_the_gates():
    """compose_block of a gate sequence on one wire = conjugation by the product of the unitaries
    (the U_{k,j} of reference lut.py:67-74), row p = image of axis p."""
    rng = np.random.default_rng(5)
    for _ in range(40):
        seq = [Instruction(str(g), (0,), float(rng.uniform(0, 2 * math.pi)) if str(g).startswith("R") else 0.0)
               for g in rng.choice(["H", "S", "X", "SX", "RX", "RY", "RZ"], size=int(rng.integers(1, 6)))]
        block = lut.compose_block(seq)
        for p in (1, 2, 3):
            want = _pauli_components(dc.conjugate(dc.PAULI[p], seq, 1))
            assert np.max(np.abs(block[p - 1] - want)) < 1e-12


def test_operator_grouping_properties():
    """divide_instruction (tests/test_acceptance.py:130-142): strictly alternating chain, |K - K'| <= 1,
    every gate kept once, per-wire order kept, and the replayed circuit is the same unitary action."""
    for case in range(30):
        rng = np.random.default_rng([77, case])
        n = int(rng.integers(1, 6))
        gates = workloads.gen_random(n, int(rng.integers(0, 50)), rng)
        part = circuit.divide_instruction(gates, n)
        assert all(a != b for a, b in zip(part.order, part.order[1:]))
        assert abs(part.k - part.k_prime) <= 1 and part.k + part.k_prime == len(part.order)
        assert sum(part.operator_sizes()) == len(gates)
        assert all(len(i.wires) == 2 for v in part.v_groups for i in v)
        assert all(len(i.wires) == 1 and i.wires[0] == w for u in part.u_groups for w, cell in u.items() for i in cell)
        replay = part.replay()
        for q in range(n):                                       # per-wire order is untouched
            assert [g for g in replay if q in g.wires] == [g for g in gates if q in g.wires]
        if n <= 3 and gates:
            z = dc.word(3, n)
            assert np.abs(dc.conjugate(z, replay, n) - dc.conjugate(z, gates, n)).max() < 1e-12
        assert circuit.create_chain(part.k, part.k_prime, not part.order or part.order[0] == 0) == part.order


class _G:
    def __init__(self, n, lam, idx):
        self.n, self.lambdas, self.indices = n, lam, idx


@pytest.mark.parametrize("mode", ["v1", "v2", "v3"])
def test_oracle_generators_equal_conjugated_z(mode):
    """The oracle port itself against dense matrices on the reference's campaign seeds
    (tests/test_acceptance.py:25-64): P_j = U Z_j U^dagger within 1e-9."""
    worst = 0.0
    for case in range(40):
        rng = np.random.default_rng([2024, case])
        n = int(rng.integers(2, 6))
        gates = workloads.gen_random(n, int(rng.integers(1, 61)), rng)
        res = oracle.run(gates, n, mode)
        for j, (lam, idx) in enumerate(res["final"]):
            want = dc.conjugate(dc.word(3 * 4 ** (n - 1 - j), n), gates, n)
            worst = max(worst, float(np.abs(dc.generator_matrix(_G(n, lam, idx)) - want).max()))
    assert worst < 1e-9, worst


def test_oracle_readout_equals_the_state_vector():
    """Oracle prob_z / expectation against |psi|^2 marginals (criterion 10, tests/test_acceptance.py:169-183)."""
    worst = 0.0
    for case in range(40):
        rng = np.random.default_rng([2025, case])
        n = int(rng.integers(1, 5))
        gates = workloads.gen_random(n, int(rng.integers(1, 41)), rng)
        final = oracle.run(gates, n, "v3")["final"]
        ex = oracle.density_expansion(final, n)
        psi = dc.state(gates, n)
        for k in range(n):
            want = dc.prob_zero(psi, k, n)
            worst = max(worst, abs(oracle.prob_z(final, n, k, ex)[0] - want),
                        abs(0.5 * (1 + oracle.expectation(final, n, 3 * 4 ** (n - 1 - k), ex)) - want))
    assert worst < 1e-9, worst
