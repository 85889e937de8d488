"""Generator containers and the kernel-level operations, GPU-backed.

Host-side mirror of the reference's ``stabilizer.py`` interface for the hot
path: the same names, argument meaning and error behaviour
(``SimpleGenerator`` :83-109, ``GeneratorSet`` :157-166, ``init_z`` :169-174,
``sub`` :189-206, ``flatten`` :240-256, ``canonicalize`` :325-337,
``apply_cx`` :340-363, ``rank_stats`` :366-369), so the reference's unit
tests can be pointed at this module.  All arithmetic happens in
``libqimax_b200.so`` on the GPU; these functions upload one generator, run the
kernel(s), and download the result.  They are pure (inputs never mutated).

For whole circuits use ``engine.run`` -- it keeps the terms in HBM between
gates instead of round-tripping per call.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import lut as _lut
from .errors import ResourceLimitError
from .store import DeviceStore

DEFAULT_EPS = 1e-12                 # reference stabilizer.py:38
DENSE_FLATTEN_BUDGET = 4 ** 10      # reference stabilizer.py:45
_INT64_MAX_QUBITS = 31              # 4**31 - 1 < 2**63
MAX_QUBITS = 32                     # one uint64 key per term on the device; more words above (n <= 512)


def index_dtype(n: int):
    """int64 up to 31 qubits, Python ints (object) beyond (reference stabilizer.py:48-49)."""
    return np.int64 if n <= _INT64_MAX_QUBITS else object


def make_index_array(values, n: int) -> np.ndarray:
    if index_dtype(n) is object:
        out = np.empty(len(values), dtype=object)
        out[:] = [int(v) for v in values]
        return out
    return np.asarray(values, dtype=np.int64)


def keys_to_indices(keys: np.ndarray, n: int) -> np.ndarray:
    """Device keys (uint64) -> the reference's index array dtype."""
    if index_dtype(n) is object:
        if isinstance(keys, np.ndarray) and keys.dtype == np.uint64:
            return keys.astype(object)             # Python ints, converted in C (n = 32: 34 k terms of C5)
        return make_index_array(keys.tolist(), n)
    return keys.view(np.int64) if keys.dtype == np.uint64 else keys.astype(np.int64)


def indices_to_keys(indices, n: int) -> np.ndarray:
    """Reference index array (int64 or object) -> uint64 keys, range-checked; above 32 qubits an
    object array of Python ints (the device splits them into 64-bit words, store.py)."""
    if n > MAX_QUBITS:
        vals = [int(v) for v in indices]
        if any(v < 0 or v >= 4 ** n for v in vals):
            raise ValueError(f"word index out of range [0, 4**{n})")
        out = np.empty(len(vals), dtype=object)
        out[:] = vals
        return out
    if isinstance(indices, np.ndarray) and indices.dtype == np.int64:
        if len(indices) and int(indices.min()) < 0:
            raise ValueError("negative word index")
        return indices.astype(np.uint64)
    vals = [int(v) for v in indices]
    if any(v < 0 or v >= 4 ** n for v in vals):
        raise ValueError(f"word index out of range [0, 4**{n})")
    return np.array(vals, dtype=np.uint64)


@dataclass(eq=False)
class SimpleGenerator:
    """A generator as a weighted sum of Pauli words (reference stabilizer.py:83-109)."""

    n: int
    lambdas: np.ndarray
    indices: np.ndarray

    def __post_init__(self):
        self.lambdas = np.asarray(self.lambdas, dtype=np.float64)
        want = index_dtype(self.n)
        if not isinstance(self.indices, np.ndarray) or self.indices.dtype != want:
            self.indices = make_index_array(self.indices, self.n)
        if len(self.lambdas) != len(self.indices):
            raise ValueError("lambdas and indices must have equal length")

    @property
    def rank(self) -> int:
        return len(self.lambdas)

    @property
    def is_degenerate(self) -> bool:
        return self.rank == 0

    def copy(self) -> "SimpleGenerator":
        return SimpleGenerator(self.n, self.lambdas.copy(), self.indices.copy())

    def keys(self) -> np.ndarray:
        return indices_to_keys(self.indices, self.n)


@dataclass
class GeneratorSet:
    """The n generators of an n-qubit state (reference stabilizer.py:157-166)."""

    n: int
    generators: list

    def __post_init__(self):
        if len(self.generators) != self.n:
            raise ValueError(f"expected exactly {self.n} generators, got {len(self.generators)}")


def init_z(n: int) -> GeneratorSet:
    """Generators of |0...0>: Z_j with coefficient 1 (reference stabilizer.py:169-174)."""
    if n < 1:
        raise ValueError(f"qubit count must be positive, got {n}")
    return GeneratorSet(n, [SimpleGenerator(n, [1.0], [3 * 4 ** (n - 1 - j)]) for j in range(n)])


def rank_stats(gs: GeneratorSet) -> tuple:
    counts = [g.rank for g in gs.generators]
    return counts, sum(counts) / len(counts)


def generator_set_to_dict(gs: GeneratorSet) -> dict:
    """JSON-ready dump (reference stabilizer.py:372-383)."""
    return {
        "n": gs.n,
        "generators": [
            {"lambda": [float(v) for v in g.lambdas], "index": [int(v) for v in g.indices]}
            for g in gs.generators
        ],
    }


# ------------------------------------------------------------------------------
# kernel-level operations on one generator
# ------------------------------------------------------------------------------
def _one_segment(g: SimpleGenerator, capacity: int = 0) -> DeviceStore:
    st = DeviceStore(g.n, 1, max(capacity, 2 * g.rank + 2))
    st.upload([(g.lambdas, g.keys())])
    return st


def _fetch(st: DeviceStore, n: int) -> SimpleGenerator:
    (lam, keys), = st.segments()
    return SimpleGenerator(n, lam.copy(), keys_to_indices(keys.copy(), n))


def apply_cx(g: SimpleGenerator, c: int, t: int) -> SimpleGenerator:
    """Conjugate every word by CX(c, t); term count unchanged, output unsorted
    (reference stabilizer.py:340-363)."""
    n = g.n
    if c == t:
        raise ValueError(f"control and target must differ, got {c}")
    if not (0 <= c < n and 0 <= t < n):
        raise ValueError(f"wires ({c}, {t}) out of range for n={n}")
    with _one_segment(g) as st:
        st.apply_clifford([_lut.cx_op(n, c, t)])
        return _fetch(st, n)


def canonicalize(g: SimpleGenerator, eps: float = DEFAULT_EPS) -> SimpleGenerator:
    """Merge duplicate words, drop |coefficient| < eps, sort ascending
    (reference stabilizer.py:325-337)."""
    if g.rank == 0:
        return g.copy()
    with _one_segment(g) as st:
        st.merge(eps)
        return _fetch(st, g.n)


def apply_1q(g: SimpleGenerator, gate: str, q: int, theta: float = 0.0,
             eps: float = DEFAULT_EPS) -> SimpleGenerator:
    """One single-qubit gate on one generator, merged: the reference's
    ``engine._apply_1q_terms`` (engine.py:183-218)."""
    n = g.n
    if not 0 <= q < n:
        raise ValueError(f"wire {q} out of range for n={n}")
    block = _lut.gate_branch_block(gate, theta)
    with _one_segment(g) as st:
        table = _lut.perm_word(block)
        if table is not None:
            st.apply_clifford([_lut.perm_op(n, q, table)])
        else:
            st.apply_split(q, *split_tables(block))
        st.merge(eps)
        return _fetch(st, n)


def split_tables(block: np.ndarray) -> tuple:
    """Per-digit (a1, w1, a2, w2) of a lone gate (reference engine.py:190-202)."""
    counts, axes, weights = _lut.branch_table(block)
    if int(counts.max()) > 2:
        raise ValueError("a single gate maps an axis to at most two axes")
    a1 = np.zeros(4, dtype=np.int32)
    a2 = np.zeros(4, dtype=np.int32)
    w1 = np.zeros(4)
    w2 = np.zeros(4)
    w1[0] = 1.0
    a1[1:], w1[1:] = axes[:, 0], weights[:, 0]
    a2[1:], w2[1:] = axes[:, 1], weights[:, 1]
    return a1, w1, a2, w2


def indices_to_digits(indices: np.ndarray, n: int) -> np.ndarray:
    """Packed word indices -> (S, n) axis codes, qubit 0 first (reference stabilizer.py:62-69)."""
    idx = np.asarray(indices)
    out = np.empty((len(idx), n), dtype=np.int64)
    if idx.dtype == object or n > _INT64_MAX_QUBITS:
        for s, v in enumerate(idx):
            v = int(v)
            for j in range(n):
                out[s, j] = (v >> (2 * (n - 1 - j))) & 3
        return out
    vals = idx.astype(np.int64)
    for j in range(n):
        out[:, j] = (vals >> np.int64(2 * (n - 1 - j))) & np.int64(3)
    return out


def digits_to_indices(digits: np.ndarray, n: int) -> np.ndarray:
    """(S, n) axis codes -> packed word indices (reference stabilizer.py:72-80)."""
    digits = np.asarray(digits)
    if index_dtype(n) is object:
        out = np.empty(len(digits), dtype=object)
        for s in range(len(digits)):
            v = 0
            for j in range(n):
                v = (v << 2) | int(digits[s, j])
            out[s] = v
        return out
    acc = np.zeros(len(digits), dtype=np.int64)
    for j in range(n):
        acc = (acc << np.int64(2)) | digits[:, j].astype(np.int64)
    return acc


@dataclass(eq=False)
class DenseComplexGenerator:
    """Complex form, dense layout: (S, n, 4) zero-padded weights (reference stabilizer.py:112-120).

    A host-side view for callers and tests: ``sub`` fills it in, ``flatten`` takes it back.  The
    engine never builds it -- on the device the (S, n, 4) tensor is never materialised (a4)."""

    n: int
    lambdas: np.ndarray
    weights: np.ndarray
    _source: tuple = field(default=None, repr=False)

    layout = "dense"


@dataclass(eq=False)
class RaggedComplexGenerator:
    """Complex form, ragged layout (reference stabilizer.py:123-154): nonzero weights and their axis
    codes of all (string, qubit) cells in C order, ``counts[s, j]`` entries per cell, ascending
    axes inside a cell, no zero stored."""

    n: int
    lambdas: np.ndarray
    values: np.ndarray
    axes: np.ndarray
    counts: np.ndarray
    _offsets: np.ndarray = field(default=None, repr=False)
    _source: tuple = field(default=None, repr=False)

    layout = "ragged"

    @property
    def offsets(self) -> np.ndarray:
        if self._offsets is None:
            flat = self.counts.astype(np.int64).ravel()
            self._offsets = (np.cumsum(flat) - flat).reshape(self.counts.shape)
        return self._offsets

    def entries(self, s: int, j: int) -> tuple:
        """(axis codes, weights) of string s at qubit j."""
        lo = int(self.offsets[s, j])
        hi = lo + int(self.counts[s, j])
        return self.axes[lo:hi], self.values[lo:hi]


ComplexForm = (DenseComplexGenerator, RaggedComplexGenerator)


def _ragged_from_weights(n: int, lambdas: np.ndarray, weights: np.ndarray, source=None) -> RaggedComplexGenerator:
    nz = weights != 0.0
    return RaggedComplexGenerator(n, lambdas, weights[nz], np.nonzero(nz)[2].astype(np.uint8),
                                  nz.sum(axis=2).astype(np.uint8), None, source)


def to_ragged(g: DenseComplexGenerator) -> RaggedComplexGenerator:
    """Dense layout -> ragged layout (reference stabilizer.py:217-219)."""
    return _ragged_from_weights(g.n, g.lambdas.copy(), g.weights)


def to_dense(g: RaggedComplexGenerator) -> DenseComplexGenerator:
    """Ragged layout -> dense layout (reference stabilizer.py:222-229)."""
    s = len(g.lambdas)
    weights = np.zeros((s, g.n, 4))
    per_cell = g.counts.astype(np.int64).ravel()
    cell = np.repeat(np.arange(s * g.n), per_cell)
    weights[cell // g.n, cell % g.n, g.axes.astype(np.int64)] = g.values
    return DenseComplexGenerator(g.n, g.lambdas.copy(), weights)


def _fingerprint(arr: np.ndarray) -> tuple:
    return arr.shape, float(np.sum(arr))


def sub(g: SimpleGenerator, block: np.ndarray, layout: str = "ragged"):
    """Substitute an (n, 3, 3) operator block (reference stabilizer.py:189-206): every non-identity
    axis of every string becomes its conjugated (X, Y, Z) weight row.  The returned form also
    remembers (keys, block), so that ``flatten`` of an untouched form runs as ONE device expansion
    with per-qubit tables instead of string by string."""
    n = g.n
    block = np.asarray(block, dtype=np.float64)
    if block.shape != (n, 3, 3):
        raise ValueError(f"expected block shape ({n}, 3, 3), got {block.shape}")
    if layout not in ("dense", "ragged"):
        raise ValueError(f"unknown layout {layout!r}")
    rows = np.zeros((n, 4, 4))
    rows[:, 0, 0] = 1.0
    rows[:, 1:, 1:] = block
    weights = rows[np.arange(n)[None, :], indices_to_digits(g.indices, n)]
    if layout == "dense":
        out = DenseComplexGenerator(n, g.lambdas.copy(), weights)
        out._source = (g.keys(), block.copy(), _fingerprint(out.weights), _fingerprint(out.lambdas))
        return out
    out = _ragged_from_weights(n, g.lambdas.copy(), weights)
    out._source = (g.keys(), block.copy(), _fingerprint(out.values), _fingerprint(out.lambdas))
    return out


def branch_counts(g) -> np.ndarray:
    """Raw branches every string contributes when flattened (reference stabilizer.py:232-237)."""
    if isinstance(g, RaggedComplexGenerator):
        return g.counts.astype(np.int64).prod(axis=1)
    if isinstance(g, DenseComplexGenerator):
        return (g.weights != 0.0).sum(axis=2).astype(np.int64).prod(axis=1)
    raise TypeError(f"cannot count the branches of {type(g).__name__}")


def pad_dense(st: DeviceStore, n: int, segments) -> None:
    """Dense layout with eps = 0: a generator that went through the reference's 4**n scatter
    buffer keeps EVERY word, exact zeros included (``keep = |out| >= 0``, stabilizer.py:277-286).
    Appends one zero-coefficient term per word to the raw lists of ``segments``; the merge that
    follows adds 0.0 into the words that exist and keeps the rest as zeros.  Only reachable for
    4**n <= DENSE_FLATTEN_BUDGET; the lists take a round trip through the host (no arithmetic)."""
    segs = [(lam.copy(), keys.copy()) for lam, keys in st.segments()]
    every = np.arange(4 ** n, dtype=np.uint64)
    for g in segments:
        lam, keys = segs[g]
        segs[g] = (np.concatenate([lam, np.zeros(len(every))]), np.concatenate([keys, every]))
    st.upload(segs)


def _untouched_source(g):
    """(keys, block) of a form that still is what ``sub`` returned, else None."""
    src = getattr(g, "_source", None)
    if src is None:
        return None
    keys, block, fp_w, fp_l = src
    body = g.weights if isinstance(g, DenseComplexGenerator) else g.values
    if _fingerprint(body) != fp_w or _fingerprint(g.lambdas) != fp_l or len(keys) != len(g.lambdas):
        return None
    return keys, block


def _flatten_block(g, keys, block, eps: float, canonical: bool) -> SimpleGenerator:
    """flatten(sub(g, block)): one device expansion with per-qubit branch tables."""
    n = g.n
    dense = isinstance(g, DenseComplexGenerator)
    counts, axes, weights = _lut.operator_tables(block)
    with DeviceStore(n, 1, 2 * len(g.lambdas) + 2) as st:
        st.upload([(g.lambdas, keys)])
        if dense and canonical and 4 ** n > DENSE_FLATTEN_BUDGET:
            if st.count_operator(counts)[0] > len(g.lambdas):
                raise ResourceLimitError(
                    f"dense flatten needs a 4**{n}-element buffer (> {DENSE_FLATTEN_BUDGET}); "
                    "use the ragged layout for circuits of this size"
                )
        if not dense or not canonical:
            st.order_for_operator(counts, by_key=False)      # raw order of _flatten_ragged (:294-296)
        dense_zeros = (dense and canonical and eps == 0.0
                       and st.count_operator(counts)[0] > len(g.lambdas))
        st.apply_operator(counts, axes, weights)
        if dense_zeros:
            pad_dense(st, n, [0])
        if canonical:
            st.merge(eps)
        return _fetch(st, n)


def _flatten_cells(g: RaggedComplexGenerator, dense: bool, eps: float, canonical: bool) -> SimpleGenerator:
    """A complex form built cell by cell (every string with weights of its own, as the reference's
    unit tests do): the device expansion kernel takes per-QUBIT tables, so each string is expanded
    on its own -- its non-trivial cells become the table rows of a stand-in word -- and the raw
    lists are concatenated in the reference's order (strings grouped by their branch-count
    pattern, stable inside a group, stabilizer.py:294-296) and merged on the device."""
    n, s_count = g.n, len(g.lambdas)
    counts_all = g.counts.astype(np.int64)
    if dense and canonical and 4 ** n > DENSE_FLATTEN_BUDGET and np.any(counts_all != 1):
        raise ResourceLimitError(
            f"dense flatten needs a 4**{n}-element buffer (> {DENSE_FLATTEN_BUDGET}); "
            "use the ragged layout for circuits of this size"
        )
    if s_count:
        _, inverse = np.unique(counts_all, axis=0, return_inverse=True)
        order = np.argsort(np.asarray(inverse).reshape(-1), kind="stable")
    else:
        order = []
    raw_l, raw_k = [np.zeros(0)], [np.zeros(0, dtype=np.uint64 if n <= MAX_QUBITS else object)]
    for s in order:
        key = 0
        lam = float(g.lambdas[s])
        tab_c = np.ones((n, 3), dtype=np.int32)
        tab_a = np.tile(np.array([[1, 0, 0], [2, 0, 0], [3, 0, 0]], dtype=np.int32), (n, 1, 1))
        tab_w = np.zeros((n, 3, 3))
        tab_w[:, :, 0] = 1.0
        for j in range(n):
            ax, vals = g.entries(int(s), j)
            ax = np.asarray(ax, dtype=np.int64)
            if len(ax) == 1 and ax[0] == 0:
                lam = lam * float(vals[0])        # an identity cell: a scalar, exactly 1.0 from sub()
                continue
            if len(ax) == 0 or np.any(ax == 0):
                raise ValueError(f"cell ({s}, {j}) mixes the identity with other axes: not a conjugated Pauli row")
            key |= 1 << (2 * (n - 1 - j))         # stand-in digit X; its table row is this cell
            tab_c[j, 0] = len(ax)
            tab_a[j, 0, :len(ax)] = ax
            tab_w[j, 0, :] = 0.0
            tab_w[j, 0, :len(ax)] = vals
        keys = np.array([key], dtype=np.uint64) if n <= MAX_QUBITS else np.array([key], dtype=object)
        with DeviceStore(n, 1, 4) as st:
            st.upload([(np.array([lam]), keys)])
            st.apply_operator(tab_c, tab_a, tab_w)
            (l, k), = st.segments()
            raw_l.append(l.copy())
            raw_k.append(k.copy())
    lam_all = np.concatenate(raw_l)
    keys_all = np.concatenate(raw_k) if n <= MAX_QUBITS else np.array([int(v) for part in raw_k for v in part], dtype=object)
    raw = SimpleGenerator(n, lam_all, keys_to_indices(keys_all, n) if n <= MAX_QUBITS else keys_all)
    if not canonical:
        return raw
    if dense and eps == 0.0 and np.any(counts_all != 1):
        every = np.arange(4 ** n, dtype=np.uint64)
        raw = SimpleGenerator(n, np.concatenate([raw.lambdas, np.zeros(len(every))]),
                              keys_to_indices(np.concatenate([raw.keys(), every]), n))
    return canonicalize(raw, eps)


def flatten(cg, eps: float = DEFAULT_EPS, canonical: bool = True) -> SimpleGenerator:
    """Expand a complex form back into a simple form (reference stabilizer.py:240-256).

    ``canonical=False`` returns the raw branch list in the reference's order (strings grouped by
    branch-count pattern, stable inside a group, each string's branches in C order).  The
    dense layout keeps the reference's budget guard (stabilizer.py:272-276): it
    refuses a branching expansion when 4**n exceeds DENSE_FLATTEN_BUDGET.
    """
    if not isinstance(cg, ComplexForm):
        raise TypeError(f"cannot flatten {type(cg).__name__}")
    src = _untouched_source(cg)
    if src is not None:
        return _flatten_block(cg, src[0], src[1], eps, canonical)
    if isinstance(cg, DenseComplexGenerator):
        return _flatten_cells(to_ragged(cg), True, eps, canonical)
    return _flatten_cells(cg, False, eps, canonical)
