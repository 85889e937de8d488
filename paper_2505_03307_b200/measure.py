"""Read-out: density expansion, Z probabilities, Pauli expectations -- on the GPU.

Mirror of the reference's ``measure.py`` (``density_expansion`` :40-73,
``prob_z`` :94-111, ``expectation`` :114-123, ``PauliExpansion`` :28-37) with the
same caps, the same exceptions and the same formulas; the pairwise word products
and the complex merge run in ``libqimax_b200.so`` (``csrc/readout.cu``).

``expectation_heisenberg`` is the addition SURVEY.md section 5.7' calls option B
and BASELINE.json's north star calls kernel (4): <psi|W|psi> = <0|U^dagger W U|0>
is obtained by pushing the single word W back through the inverse circuit with the
same gate-apply / merge kernels and summing the coefficients of the Z/I-only
words with a warp-shuffle reduction.  Its cost is polynomial in the stabilizer
rank, so it is the only read-out that works beyond 12 qubits.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .circuit import Instruction
from .errors import ConsistencyError, ResourceLimitError
from .stabilizer import GeneratorSet, indices_to_keys

DENSITY_MAX_QUBITS = 12          # reference measure.py:23
DEFAULT_TERM_BUDGET = 2_000_000  # reference measure.py:24
_IMAG_TOL = 1e-10


class PauliExpansion:
    """Sparse Pauli-basis expansion of a density operator (reference measure.py:28-37).

    Held as ascending word codes + coefficients; ``coeffs`` builds the reference's
    dict view on demand.
    """

    def __init__(self, n: int, codes, values=None):
        # reference signature: PauliExpansion(n, coeffs: dict) (measure.py:31-33); the device
        # read-out hands over the sorted arrays directly
        self.n = n
        if values is None:
            items = sorted((int(c), float(v)) for c, v in dict(codes).items())
            codes = np.array([c for c, _ in items], dtype=np.uint64)
            values = np.array([v for _, v in items], dtype=np.float64)
        self.codes = codes
        self.values = values
        self._dict = None

    @property
    def coeffs(self) -> dict:
        if self._dict is None:
            self._dict = {int(c): float(v) for c, v in zip(self.codes, self.values)}
        return self._dict

    def coeff(self, index: int) -> float:
        index = int(index)
        if index < 0 or index >= 4 ** self.n:
            return 0.0
        pos = int(np.searchsorted(self.codes, np.uint64(index)))
        if pos < len(self.codes) and int(self.codes[pos]) == index:
            return float(self.values[pos])
        return 0.0

    def __len__(self):
        return len(self.codes)


def density_expansion(gs: GeneratorSet, max_qubits: int = DENSITY_MAX_QUBITS,
                      term_budget: int = DEFAULT_TERM_BUDGET, device=None) -> PauliExpansion:
    """Expand 2^-n prod_j (I + P_j) into Pauli-word coefficients (reference measure.py:40-73)."""
    n = gs.n
    if n > max_qubits:
        raise ResourceLimitError(f"density expansion capped at {max_qubits} qubits, got {n}")
    lib = nat.lib()
    handle = C.c_void_p()
    dev = nat.default_device() if device is None else int(device)
    nat.check(lib.qx_expansion_create(dev, n, 4096, C.byref(handle)))
    try:
        for g in gs.generators:
            keys = np.ascontiguousarray(indices_to_keys(g.indices, n))
            lam = np.ascontiguousarray(g.lambdas, dtype=np.float64)
            # reference measure.py:59: raise as soon as the raw list is longer than the budget,
            # whatever the budget (0 or negative budgets fail on the first generator)
            nat.check(lib.qx_expansion_multiply(handle, nat.ptr(keys), nat.ptr(lam), len(lam),
                                                max(int(term_budget), 0)))
        worst = C.c_double()
        nat.check(lib.qx_expansion_max_abs_imag(handle, C.byref(worst)))
        if worst.value > _IMAG_TOL:
            raise ConsistencyError(
                f"density expansion produced a non-real coefficient (imag {worst.value:.3e})"
            )
        count = C.c_int64()
        nat.check(lib.qx_expansion_size(handle, C.byref(count)))
        codes = np.empty(count.value, dtype=np.uint64)
        re = np.empty(count.value, dtype=np.float64)
        nat.check(lib.qx_expansion_download(handle, nat.ptr(codes), nat.ptr(re), None, count.value))
    finally:
        lib.qx_expansion_destroy(handle)
    return PauliExpansion(n, codes, re * 0.5 ** n)


def prob_z(gs: GeneratorSet, k: int, expansion: PauliExpansion = None) -> tuple:
    """(p0, p1) of measuring qubit k (reference measure.py:94-111)."""
    n = gs.n
    if not 0 <= k < n:
        raise ValueError(f"qubit {k} out of range for n={n}")
    if expansion is None:
        expansion = density_expansion(gs)
    p0 = 0.5 + 2.0 ** (n - 1) * expansion.coeff(3 * 4 ** (n - 1 - k))
    if not -1e-10 <= p0 <= 1.0 + 1e-10:
        raise ConsistencyError(f"probability {p0} for qubit {k} outside [0, 1]")
    p0 = min(1.0, max(0.0, p0))
    return p0, 1.0 - p0


def expectation(gs: GeneratorSet, word: int, expansion: PauliExpansion = None) -> float:
    """Expectation of a Pauli word given as base-4 index (reference measure.py:114-123)."""
    n = gs.n
    if not 0 <= word < 4 ** n:
        raise ValueError(f"word index {word} out of range [0, 4**{n})")
    if expansion is None:
        expansion = density_expansion(gs)
    return 2.0 ** n * expansion.coeff(word)


# ------------------------------------------------------------------------------
# Heisenberg read-out: polynomial in rank, any n the store holds (multi-word keys above 32 qubits)
# ------------------------------------------------------------------------------
def inverse_circuit(instructions) -> list:
    """Gates reversed and inverted: S^-1 = S^3, SX^-1 = SX^3, R(t)^-1 = R(-t); H, X, CX self-inverse."""
    out = []
    for g in reversed(list(instructions)):
        if g.gate in ("S", "SX"):
            out += [g, g, g]
        elif g.gate in ("RX", "RY", "RZ"):
            out.append(Instruction(g.gate, g.wires, -g.theta))
        else:
            out.append(g)
    return out


def expectation_heisenberg(instructions, n: int, words, mode="v1", eps: float = 1e-12,
                           device=None) -> np.ndarray:
    """<psi|W|psi> for every word in ``words`` (psi = circuit applied to |0...0>).

    One store segment per word; the inverse circuit is run on all of them at once, then
    ``qx_store_zi_sums`` adds up the coefficients of the words without X/Y digits
    (<0|Q|0> = 1 exactly for those, 0 otherwise).
    """
    from .engine import run

    words = [int(w) for w in words]
    for w in words:
        if not 0 <= w < 4 ** n:
            raise ValueError(f"word index {w} out of range [0, 4**{n})")
    if not words:
        return np.zeros(0)
    if n > 32:      # multi-word keys: Python ints, as the reference's big-int indices (stabilizer.py:40-59)
        initial = [(np.ones(1), np.array([w], dtype=object)) for w in words]
    else:
        initial = [(np.ones(1), np.array([w], dtype=np.uint64)) for w in words]
    report = run(inverse_circuit(instructions), n, mode, eps, device=device, initial=initial,
                 download=False)
    store = report.device["store"]
    try:
        return store.zi_sums()
    finally:
        store.close()
