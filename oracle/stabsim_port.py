"""CPU oracle: numpy restatement of the reference's extended-stabilizer hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_2505_03307_b200/`` imports
this file; only ``tests/``, ``__graft_entry__.smoke()`` and the CPU legs of
``bench.py`` do, and only as the checker / CPU baseline.

Parity status: PINNED.  ``tests/test_oracle_golden.py`` checks this file against
(a) every known-answer vector the reference's own tests hold for this path
 and (b) fixtures produced by importing the reference
itself in the build container (``oracle/make_golden.py`` ->
``tests/golden/*.json|npz``), keys bit-exact and coefficients bit-exact for
v1/v3 (same numpy primitives in the same order) and <= 1e-12 for v2.

Each function cites the reference lines it restates (paths under
``/root/reference/pkg/src/stabsim/``).  Word indices are ``uint64`` for every
n <= 32 (4**32 - 1 == 2**64 - 1 fits exactly); the reference switches to Python
big-int object arrays above 31 qubits (stabilizer.py:40-59), same values.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2505_03307_b200.errors import (
    ConsistencyError,
    NumericalCollapseError,
    ResourceLimitError,
)

EPS = 1e-12                      # stabilizer.py:38
DENSE_BUDGET = 4 ** 10           # stabilizer.py:45
DENSITY_MAX_QUBITS = 12          # measure.py:23
TERM_BUDGET = 2_000_000          # measure.py:24
U64 = np.uint64


# ----------------------------------------------------------------------------
# tables (lut.py:28-52, 108-134; pauli.py:37-46)
# ----------------------------------------------------------------------------
def axis_map(gate, theta=0.0):
    """lut.py:41-52 with the fixed maps of lut.py:29-38."""
    c, s = math.cos(theta), math.sin(theta)
    table = {
        "H": [[0.0, 0.0, 1.0], [0.0, -1.0, 0.0], [1.0, 0.0, 0.0]],
        "S": [[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]],
        "X": [[1.0, 0.0, 0.0], [0.0, -1.0, 0.0], [0.0, 0.0, -1.0]],
        "SX": [[1.0, 0.0, 0.0], [0.0, 0.0, -1.0], [0.0, 1.0, 0.0]],
        "RX": [[1.0, 0.0, 0.0], [0.0, c, -s], [0.0, s, c]],
        "RY": [[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]],
        "RZ": [[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]],
    }
    if gate not in table:
        raise ValueError(f"no single-qubit conjugation rule for gate {gate!r}")
    return np.array(table[gate])


CX_C = np.array([[0, 0, 3, 3], [1, 1, 2, 2], [2, 2, 1, 1], [3, 3, 0, 0]], dtype=np.int64)
CX_T = np.array([[0, 1, 2, 3], [1, 0, 3, 2], [1, 0, 3, 2], [0, 1, 2, 3]], dtype=np.int64)
CX_S = np.array([[1, 1, 1, 1], [1, 1, 1, -1], [1, 1, -1, 1], [1, 1, 1, 1]], dtype=np.int64)
PHASE_EXP = np.array([[0, 0, 0, 0], [0, 0, 1, 3], [0, 3, 0, 1], [0, 1, 3, 0]], dtype=np.int64)
PHASE = np.array([1, 1j, -1, -1j], dtype=np.complex128)


def block_of(gates):
    """lut.py:67-74: left-multiply in circuit order, return the transpose."""
    total = np.eye(3)
    for g in gates:
        total = axis_map(g.gate, g.theta) @ total
    return total.T.copy()


# ----------------------------------------------------------------------------
# partition (circuit.py:158-182)
# ----------------------------------------------------------------------------
def partition(instructions, n):
    """Chain of ('U', {wire: gates}) / ('V', [cx, ...]) operators."""
    chain = []
    for g in instructions:
        if any(w >= n for w in g.wires):
            raise ValueError(f"wire out of range for n={n}: {g}")
        kind = "V" if len(g.wires) == 2 else "U"
        if not chain or chain[-1][0] != kind:
            chain.append((kind, [] if kind == "V" else {}))
        if kind == "V":
            chain[-1][1].append(g)
        else:
            chain[-1][1].setdefault(g.wires[0], []).append(g)
    return chain


def lut_blocks(chain, n):
    """lut.py:77-103: one (n,3,3) block per U operator."""
    out = []
    for kind, body in chain:
        if kind == "U":
            blk = np.empty((n, 3, 3))
            for j in range(n):
                blk[j] = block_of(body.get(j, ()))
            out.append(blk)
    return out


# ----------------------------------------------------------------------------
# term-level operations
# ----------------------------------------------------------------------------
def digit(idx, n, q):
    """(idx // 4**(n-1-q)) % 4 (stabilizer.py:354-355) as a shift on uint64."""
    return ((idx >> U64(2 * (n - 1 - q))) & U64(3)).astype(np.int64)


def merge(lam, idx, eps=EPS):
    """stabilizer.py:325-337: unique-sort, in-order segmented sum, keep |sum| >= eps."""
    if len(lam) == 0:
        return lam.copy(), idx.copy()
    uniq, inv = np.unique(idx, return_inverse=True)
    sums = np.zeros(len(uniq))
    np.add.at(sums, inv.reshape(-1), lam)
    keep = np.abs(sums) >= eps
    return sums[keep], uniq[keep]


def conj_cx(lam, idx, n, c, t):
    """stabilizer.py:340-363: table lookup on the (c, t) digit pair; unsorted output."""
    if c == t:
        raise ValueError(f"control and target must differ, got {c}")
    if not (0 <= c < n and 0 <= t < n):
        raise ValueError(f"wires ({c}, {t}) out of range for n={n}")
    sc, st = U64(2 * (n - 1 - c)), U64(2 * (n - 1 - t))
    dc, dt = digit(idx, n, c), digit(idx, n, t)
    nc, nt = CX_C[dc, dt], CX_T[dc, dt]
    cleared = idx & ~((U64(3) << sc) | (U64(3) << st))
    moved = cleared | (nc.astype(U64) << sc) | (nt.astype(U64) << st)
    return lam * CX_S[dc, dt], moved


def conj_1q_v1(lam, idx, n, q, m, eps=EPS):
    """engine.py:183-218: first branches of all terms, then second branches, then merge."""
    a1 = np.zeros(4, dtype=np.int64)
    a2 = np.zeros(4, dtype=np.int64)
    w1 = np.zeros(4)
    w2 = np.zeros(4)
    w1[0] = 1.0
    for d in (1, 2, 3):
        col = m[:, d - 1]
        hot = np.nonzero(col)[0]
        a1[d], w1[d] = hot[0] + 1, col[hot[0]]
        if len(hot) > 1:
            a2[d], w2[d] = hot[1] + 1, col[hot[1]]
    sh = U64(2 * (n - 1 - q))
    d = digit(idx, n, q)
    base = idx & ~(U64(3) << sh)
    idx1 = base | (a1[d].astype(U64) << sh)
    idx2 = base | (a2[d].astype(U64) << sh)
    second = w2[d] != 0.0
    raw_l = np.concatenate([lam * w1[d], lam[second] * w2[d][second]])
    raw_i = np.concatenate([idx1, idx2[second]])
    return merge(raw_l, raw_i, eps)


def expand_operator(lam, idx, n, block):
    """sub + ragged flatten, raw (unmerged) output (stabilizer.py:177-214, 289-322).

    Raw order is the reference's: strings grouped by their per-qubit width
    pattern (patterns ascending lexicographically, strings stable inside a
    group), each string's branches in C order with qubit 0 slowest, products
    taken left to right in qubit order.
    """
    s = len(lam)
    if s == 0:
        return lam.copy(), idx.copy()
    rows = np.zeros((n, 4, 4))
    rows[:, 0, 0] = 1.0
    rows[:, 1:, 1:] = block
    digs = np.stack([digit(idx, n, j) for j in range(n)], axis=1)        # (s, n)
    w = rows[np.arange(n)[None, :], digs]                                 # (s, n, 4)
    nz = w != 0.0
    counts = nz.sum(axis=2).astype(np.uint8)
    pats, inv = np.unique(counts, axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    order = np.argsort(inv, kind="stable")
    sizes = np.bincount(inv, minlength=len(pats))
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    out_l, out_i = [], []
    for gi, widths in enumerate(pats):
        members = order[bounds[gi]:bounds[gi + 1]]
        acc_l = lam[members, None].copy()
        acc_i = np.zeros((len(members), 1), dtype=U64)
        for j in range(n):
            k = int(widths[j])
            # the k nonzero axes of cell (string, j), ascending
            ax = np.argsort(~nz[members, j, :], axis=1, kind="stable")[:, :k]
            vals = np.take_along_axis(w[members, j, :], ax, axis=1)
            acc_l = (acc_l[:, :, None] * vals[:, None, :]).reshape(len(members), -1)
            acc_i = ((acc_i[:, :, None] << U64(2)) | ax.astype(U64)[:, None, :]).reshape(len(members), -1)
        out_l.append(acc_l.ravel())
        out_i.append(acc_i.ravel())
    return np.concatenate(out_l), np.concatenate(out_i)


def operator_v3(lam, idx, n, block, eps=EPS):
    """flatten(sub(g, block, 'ragged'), eps) (engine.py:114)."""
    return merge(*expand_operator(lam, idx, n, block), eps)


def operator_v2(lam, idx, n, block, eps=EPS):
    """flatten(sub(g, block, 'dense'), eps) (stabilizer.py:259-286).

    Same term set as v3; the 4**n scatter buffer is refused above the dense
    budget unless every substituted row is one-hot.  Sums are accumulated with
    ``np.add.at`` instead of the reference's chunked ``sum(axis=0)``, so
    coefficients agree to rounding (pinned at 1e-12), not bitwise.
    """
    raw_l, raw_i = expand_operator(lam, idx, n, block)
    if len(raw_l) == len(lam):            # no string branched: one-hot fast path
        return merge(raw_l, raw_i, eps)
    if 4 ** n > DENSE_BUDGET:
        raise ResourceLimitError(
            f"dense flatten needs a 4**{n}-element buffer (> {DENSE_BUDGET}); "
            "use the ragged layout for circuits of this size"
        )
    dense = np.zeros(4 ** n)
    np.add.at(dense, raw_i.astype(np.int64), raw_l)
    keep = np.abs(dense) >= eps
    return dense[keep], np.nonzero(keep)[0].astype(U64)


# ----------------------------------------------------------------------------
# engine (engine.py:89-180)
# ----------------------------------------------------------------------------
def init_z(n):
    """stabilizer.py:169-174: generator j = 1.0 * Z_j."""
    if n < 1:
        raise ValueError(f"qubit count must be positive, got {n}")
    return [(np.ones(1), np.array([3 << (2 * (n - 1 - j))], dtype=U64)) for j in range(n)]


def _collapse(rank, gi, step):
    if rank == 0:
        raise NumericalCollapseError(f"all terms of generator {gi} dropped at operator step {step}")


def run(instructions, n, mode="v3", eps=EPS, generators=None, initial=None):
    """engine.run restated.  Returns a dict with final generators and bookkeeping.

    ``generators`` restricts the evolution to a subset of generator ids (they
    are independent, engine.py:113-116) -- used by the multi-process CPU
    baseline and the shard tests.  ``initial`` overrides init_z with arbitrary
    (lambdas, indices) pairs (Heisenberg read-out checks).
    ``updates`` counts term-gate updates = sum over gates of the ranks before
    the gate; it is exact in v1 and is the work unit bench.py
    reports for every mode.
    """
    mode = str(mode).lower()
    if mode not in ("v1", "v2", "v3"):
        raise ValueError(f"'{mode}' is not a valid Mode")
    chain = partition(instructions, n)
    order = [0 if kind == "U" else 1 for kind, _ in chain]
    gens = list(initial) if initial is not None else init_z(n)
    ids = list(range(len(gens))) if generators is None else list(generators)
    live = {gi: gens[gi] for gi in ids}
    trace = [[len(live[gi][0]) for gi in ids]]
    counters = {"gates": len(instructions), "sub_flatten_ops": 0, "cx_applications": 0}
    updates = 0
    if mode == "v1":
        sizes = [len(b) if k == "V" else sum(len(v) for v in b.values()) for k, b in chain]
        boundaries = set(np.cumsum(sizes).tolist())
        for pos, g in enumerate(instructions, start=1):
            for gi in ids:
                lam, idx = live[gi]
                updates += len(lam)
                if len(g.wires) == 2:
                    lam, idx = merge(*conj_cx(lam, idx, n, *g.wires), eps)
                else:
                    lam, idx = conj_1q_v1(lam, idx, n, g.wires[0], axis_map(g.gate, g.theta), eps)
                _collapse(len(lam), gi, pos - 1)
                live[gi] = (lam, idx)
            if len(g.wires) == 2:
                counters["cx_applications"] += 1
            else:
                counters["v1_gate_applications"] = counters.get("v1_gate_applications", 0) + 1
            if pos in boundaries:
                trace.append([len(live[gi][0]) for gi in ids])
    else:
        op = operator_v2 if mode == "v2" else operator_v3
        blocks = iter(lut_blocks(chain, n))
        for step, (kind, body) in enumerate(chain):
            if kind == "U":
                blk = next(blocks)
                for gi in ids:
                    lam, idx = op(*live[gi], n, blk, eps)
                    _collapse(len(lam), gi, step)
                    live[gi] = (lam, idx)
                counters["sub_flatten_ops"] += 1
            else:
                for g in body:
                    for gi in ids:
                        live[gi] = conj_cx(*live[gi], n, *g.wires)
                    counters["cx_applications"] += 1
                for gi in ids:
                    lam, idx = merge(*live[gi], eps)
                    _collapse(len(lam), gi, step)
                    live[gi] = (lam, idx)
            trace.append([len(live[gi][0]) for gi in ids])
    k = order.count(0)
    counters["operators"] = len(order)
    return {
        "mode": mode, "n": n, "ids": ids,
        "final": [live[gi] for gi in ids],
        "rank_trace": trace, "counters": counters,
        "k": k, "k_prime": len(order) - k, "order": order,
        "updates": updates,
    }


def count_updates(instructions, n, eps=EPS):
    """Term-gate updates of a circuit (v1 definition)."""
    return run(instructions, n, "v1", eps)["updates"]


# ----------------------------------------------------------------------------
# readout (measure.py:40-123)
# ----------------------------------------------------------------------------
def word_product_phase(a, b, n):
    """Sum of PHASE_EXP over digits, mod 4, for broadcastable uint64 words (pauli.py:38-46)."""
    total = np.zeros(np.broadcast(a, b).shape, dtype=np.int64)
    for j in range(n):
        total += PHASE_EXP[digit(a, n, j), digit(b, n, j)]
    return total % 4


def density_expansion(gens, n, max_qubits=DENSITY_MAX_QUBITS, term_budget=TERM_BUDGET):
    """measure.py:40-73.  Returns (codes uint64 ascending, real coefficients already * 2**-n)."""
    if n > max_qubits:
        raise ResourceLimitError(f"density expansion capped at {max_qubits} qubits, got {n}")
    codes = np.zeros(1, dtype=U64)
    coeff = np.ones(1, dtype=np.complex128)
    for lam, idx in gens:
        prod = codes[:, None] ^ idx[None, :]                       # AXIS_PRODUCT is XOR
        ph = PHASE[word_product_phase(codes[:, None], idx[None, :], n)]
        new = coeff[:, None] * lam[None, :] * ph
        codes = np.concatenate([codes, prod.reshape(-1)])
        coeff = np.concatenate([coeff, new.ravel()])
        if len(coeff) > term_budget:
            raise ResourceLimitError(f"density expansion exceeded the term budget ({term_budget})")
        uniq, inv = np.unique(codes, return_inverse=True)          # measure.py:81-91
        sums = np.zeros(len(uniq), dtype=np.complex128)
        np.add.at(sums, inv.reshape(-1), coeff)
        keep = sums != 0.0
        codes, coeff = uniq[keep], sums[keep]
    worst = float(np.max(np.abs(coeff.imag)))
    if worst > 1e-10:
        raise ConsistencyError(f"density expansion produced a non-real coefficient (imag {worst:.3e})")
    return codes, coeff.real * 0.5 ** n


def coeff_of(expansion, word):
    codes, vals = expansion
    pos = int(np.searchsorted(codes, U64(word)))
    return float(vals[pos]) if pos < len(codes) and int(codes[pos]) == int(word) else 0.0


def prob_z(gens, n, k, expansion=None):
    """measure.py:94-111."""
    if not 0 <= k < n:
        raise ValueError(f"qubit {k} out of range for n={n}")
    if expansion is None:
        expansion = density_expansion(gens, n)
    p0 = 0.5 + 2.0 ** (n - 1) * coeff_of(expansion, 3 << (2 * (n - 1 - k)))
    if not -1e-10 <= p0 <= 1.0 + 1e-10:
        raise ConsistencyError(f"probability {p0} for qubit {k} outside [0, 1]")
    p0 = min(1.0, max(0.0, p0))
    return p0, 1.0 - p0


def expectation(gens, n, word, expansion=None):
    """measure.py:114-123."""
    if not 0 <= word < 4 ** n:
        raise ValueError(f"word index {word} out of range [0, 4**{n})")
    if expansion is None:
        expansion = density_expansion(gens, n)
    return 2.0 ** n * coeff_of(expansion, word)


# ----------------------------------------------------------------------------
# Heisenberg read-out oracle: <0| U^dagger W U |0> (SURVEY.md 5.7' option B)
# ----------------------------------------------------------------------------
class _G:
    def __init__(self, gate, wires, theta=0.0):
        self.gate, self.wires, self.theta = gate, tuple(wires), theta


def inverse_circuit(instructions):
    """Reversed gate order, each gate inverted (S^-1 = S^3, SX^-1 = SX^3, R(t)^-1 = R(-t))."""
    out = []
    for g in reversed(list(instructions)):
        if g.gate in ("S", "SX"):
            out += [_G(g.gate, g.wires)] * 3
        elif g.gate in ("RX", "RY", "RZ"):
            out.append(_G(g.gate, g.wires, -g.theta))
        else:
            out.append(_G(g.gate, g.wires))
    return out


def expectation_heisenberg(instructions, n, words, mode="v1", eps=EPS):
    """<psi|W|psi> for each word by conjugating W through the inverse circuit."""
    init = [(np.ones(1), np.array([int(w)], dtype=U64)) for w in words]
    res = run(inverse_circuit(instructions), n, mode, eps, initial=init)
    mask = U64(0x5555555555555555)
    out = []
    for lam, idx in res["final"]:
        zi_only = (((idx >> U64(1)) ^ idx) & mask) == 0          # x bit = hi ^ lo
        out.append(float(lam[zi_only].sum()))
    return out
