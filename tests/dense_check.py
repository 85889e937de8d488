"""Independent dense checker for the -m gpu tests: operators as 2^n x 2^n matrices.

Shares nothing with the package or with ``oracle/`` -- gates are applied to a (2,)*2n operator
tensor with ``np.tensordot`` on the qubit's axes, Pauli words are built digit by digit the same way --
so agreement between a generator set and ``U Z_j U^dagger`` computed here is meaningful on its own
(the role ``tests/dense_ref.py`` plays in the reference's suite: SURVEY.md 8c "second, independent
oracle").  Conventions of the reference: R_a(theta) = exp(-i theta a / 2), qubit 0 most significant,
axis codes I=0 X=1 Y=2 Z=3.
"""

import numpy as np

_S2 = 1.0 / np.sqrt(2.0)
PAULI = np.zeros((4, 2, 2), dtype=complex)
PAULI[0] = [[1, 0], [0, 1]]
PAULI[1] = [[0, 1], [1, 0]]
PAULI[2] = [[0, -1j], [1j, 0]]
PAULI[3] = [[1, 0], [0, -1]]


def unitary_1q(gate, theta=0.0):
    if gate == "H":
        return _S2 * (PAULI[1] + PAULI[3])
    if gate == "S":
        return np.array([[1, 0], [0, 1j]])
    if gate == "X":
        return PAULI[1].copy()
    if gate == "SX":
        return 0.5 * ((1 + 1j) * PAULI[0] + (1 - 1j) * PAULI[1])
    axis = {"RX": 1, "RY": 2, "RZ": 3}[gate]
    return np.cos(0.5 * theta) * PAULI[0] - 1j * np.sin(0.5 * theta) * PAULI[axis]


def _left_1q(op, u, q):
    """u on qubit q from the left: contracts row axis q of the (2,)*2n tensor."""
    return np.moveaxis(np.tensordot(u, op, axes=([1], [q])), 0, q)


def _right_1q(op, u, q, n):
    """u^dagger on qubit q from the right: contracts column axis n + q."""
    return np.moveaxis(np.tensordot(op, u.conj().T, axes=([n + q], [0])), -1, n + q)


_CX4 = np.zeros((2, 2, 2, 2), dtype=complex)            # [c', t', c, t]
for _c in range(2):
    for _t in range(2):
        _CX4[_c, _t ^ _c, _c, _t] = 1.0


def _left_cx(op, c, t):
    out = np.tensordot(_CX4, op, axes=([2, 3], [c, t]))
    return np.moveaxis(out, [0, 1], [c, t])


def _right_cx(op, c, t, n):
    out = np.tensordot(op, _CX4, axes=([n + c, n + t], [0, 1]))   # CX is real and symmetric as a matrix
    return np.moveaxis(out, [-2, -1], [n + c, n + t])


def conjugate(op_matrix, instructions, n):
    """U op U^dagger for the circuit, gate by gate."""
    op = np.asarray(op_matrix, dtype=complex).reshape((2,) * (2 * n))
    for inst in instructions:
        if len(inst.wires) == 2:
            c, t = inst.wires
            op = _right_cx(_left_cx(op, c, t), c, t, n)
        else:
            u = unitary_1q(inst.gate, inst.theta)
            q = inst.wires[0]
            op = _right_1q(_left_1q(op, u, q), u, q, n)
    return op.reshape(2 ** n, 2 ** n)


def word(index, n):
    """Matrix of the Pauli word with base-4 index `index`."""
    m = np.ones((1, 1), dtype=complex)
    for j in range(n):
        m = np.kron(m, PAULI[(int(index) >> (2 * (n - 1 - j))) & 3])
    return m


def generator_matrix(g):
    m = np.zeros((2 ** g.n, 2 ** g.n), dtype=complex)
    for lam, idx in zip(g.lambdas, g.indices):
        m += float(lam) * word(int(idx), g.n)
    return m


def state(instructions, n):
    """U |0...0> as a vector."""
    psi = np.zeros((2,) * n, dtype=complex)
    psi[(0,) * n] = 1.0
    for inst in instructions:
        if len(inst.wires) == 2:
            c, t = inst.wires
            psi = np.moveaxis(np.tensordot(_CX4, psi, axes=([2, 3], [c, t])), [0, 1], [c, t])
        else:
            q = inst.wires[0]
            psi = np.moveaxis(np.tensordot(unitary_1q(inst.gate, inst.theta), psi, axes=([1], [q])), 0, q)
    return psi.reshape(-1)


def prob_zero(psi, k, n):
    p = np.abs(psi.reshape((2,) * n)) ** 2
    return float(np.take(p, 0, axis=k).sum())
