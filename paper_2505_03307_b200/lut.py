"""Host-side conjugation tables: 1q axis maps, composed U_k blocks, CX tables.

Stays on the host by design: the tables are O(K*n*9)
doubles, and building them with the *same* arithmetic as the reference
(``math.cos/sin`` of the full angle, numpy 3x3 ``@`` in gate order,
``lut.py:41-52,67-74``) keeps every weight the device multiplies bit-identical
to the reference's, so that only the merge's summation order can differ.

The second half packs those tables into what the kernels consume:
  * ``perm_word``   -- a 1q signed axis permutation as a 9-bit field,
  * ``branch_table`` -- per (qubit, input axis): how many output axes, which,
    and their weights, zero entries removed exactly like the reference does
    (``stabilizer.py:210``, ``engine.py:197-202``).
"""

from __future__ import annotations

import math

import numpy as np

# new_w = M @ w on (X, Y, Z) weight vectors (reference lut.py:29-38).
_H = ((0.0, 0.0, 1.0), (0.0, -1.0, 0.0), (1.0, 0.0, 0.0))      # X<->Z, Y->-Y
_S = ((0.0, -1.0, 0.0), (1.0, 0.0, 0.0), (0.0, 0.0, 1.0))      # X->Y, Y->-X
_X = ((1.0, 0.0, 0.0), (0.0, -1.0, 0.0), (0.0, 0.0, -1.0))     # Y->-Y, Z->-Z
_SX = ((1.0, 0.0, 0.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0))     # Y->Z, Z->-Y
_FIXED = {"H": _H, "S": _S, "X": _X, "SX": _SX}


def axis_map(gate: str, theta: float = 0.0) -> np.ndarray:
    """3x3 action of one gate on (X, Y, Z) weights; R_a(theta) = exp(-i theta a / 2)."""
    fixed = _FIXED.get(gate)
    if fixed is not None:
        return np.array(fixed)
    c, s = math.cos(theta), math.sin(theta)
    if gate == "RX":
        rows = ((1.0, 0.0, 0.0), (0.0, c, -s), (0.0, s, c))
    elif gate == "RY":
        rows = ((c, 0.0, s), (0.0, 1.0, 0.0), (-s, 0.0, c))
    elif gate == "RZ":
        rows = ((c, -s, 0.0), (s, c, 0.0), (0.0, 0.0, 1.0))
    else:
        raise ValueError(f"no single-qubit conjugation rule for gate {gate!r}")
    return np.array(rows)


def conjugate_axis(gate: str, theta: float, w) -> np.ndarray:
    """One gate on an (X, Y, Z) weight row (reference lut.py:55-64); the identity component never
    appears: conjugation fixes I and no axis acquires an I part."""
    w = np.asarray(w, dtype=float)
    if w.shape != (3,):
        raise ValueError(f"weight row must have 3 components, got shape {w.shape}")
    return axis_map(gate, theta) @ w


def lut_to_json(lut: np.ndarray) -> list:
    """Nested lists of a LUT tensor (reference lut.py:142-144)."""
    return np.asarray(lut).tolist()


def compose_block(gates) -> np.ndarray:
    """One U_{k,j} block: row p = image of axis p after all gates in circuit order.

    Same left-multiplication and final transpose as reference ``lut.py:67-74``;
    numpy's ``@`` is used on purpose so rounding matches the reference's.
    """
    acc = np.eye(3)
    for inst in gates:
        acc = axis_map(inst.gate, inst.theta) @ acc
    return np.ascontiguousarray(acc.T)


def _fill_axis_map(out: np.ndarray, gate: str, theta: float) -> None:
    """Write axis_map(gate, theta) into the zeroed 3x3 view ``out`` (same values, no temporaries)."""
    fixed = _FIXED_ARRAYS.get(gate)
    if fixed is not None:
        out[...] = fixed
        return
    c, s = math.cos(theta), math.sin(theta)
    if gate == "RX":
        out[0, 0] = 1.0
        out[1, 1] = c
        out[1, 2] = -s
        out[2, 1] = s
        out[2, 2] = c
    elif gate == "RY":
        out[0, 0] = c
        out[0, 2] = s
        out[1, 1] = 1.0
        out[2, 0] = -s
        out[2, 2] = c
    elif gate == "RZ":
        out[0, 0] = c
        out[0, 1] = -s
        out[1, 0] = s
        out[1, 1] = c
        out[2, 2] = 1.0
    else:
        raise ValueError(f"no single-qubit conjugation rule for gate {gate!r}")


def create_lut_1q(partition, workers=None) -> np.ndarray:
    """(K, n, 3, 3) tensor of composed blocks (reference lut.py:77-103).

    Only cells that hold gates are composed; the rest are the exact identity,
    which is what composing an empty list yields.  ``workers`` is accepted for
    signature compatibility; cells are independent so the result is the same.

    Cells with the same number of gates are composed together: their i-th gate
    matrices are stacked and multiplied with one batched ``np.matmul`` per
    position -- numpy runs the same 3x3 product per matrix as ``compose_block``
    does with ``@`` (bit-identical, tests/test_native_abi.py), without the
    per-call overhead.  The first factor is taken as is: M @ I == M.
    """
    return build_lut(partition)[0]


def build_lut(partition) -> tuple:
    """``create_lut_1q`` plus the classification the engine needs, in one walk over the cells:
    (lut[K, n, 3, 3], is_perm bool[K, n], table uint32[K, n]) with ``table`` as in
    ``classify_lut``.  Cells made of fixed gates only -- nearly all cells of a Clifford+T circuit
    -- recur with few distinct gate sequences: block and permutation word of a sequence are
    composed once (same numpy chain as ``compose_block``) and looked up afterwards."""
    lut = np.empty((partition.k, partition.n, 3, 3))
    lut[:] = np.eye(3)
    is_perm = np.ones((partition.k, partition.n), dtype=bool)
    table = np.full((partition.k, partition.n), IDENTITY_PERM, dtype=np.uint32)
    by_len: dict = {}
    fixed_k, fixed_w, fixed_b, fixed_t = [], [], [], []
    for ki, bucket in enumerate(partition.u_groups):
        for wire, gates in bucket.items():
            names = tuple([g.gate for g in gates])
            hit = _FIXED_BLOCKS.get(names)
            if hit is None and all(name in _FIXED for name in names):
                block = compose_block(gates)
                hit = (block, perm_word(block))      # products of signed permutations: always a word
                if len(_FIXED_BLOCKS) < 65536:
                    _FIXED_BLOCKS[names] = hit
            if hit is not None:
                fixed_k.append(ki)
                fixed_w.append(wire)
                fixed_b.append(hit[0])
                fixed_t.append(hit[1])
            else:
                by_len.setdefault(len(gates), []).append((ki, wire, gates))
    if fixed_k:
        lut[fixed_k, fixed_w] = np.array(fixed_b)     # one scatter instead of one assignment per cell
        table[fixed_k, fixed_w] = np.array(fixed_t, dtype=np.uint32)
    for length, cells in by_len.items():
        mats = np.zeros((length, len(cells), 3, 3))
        for ci, (_, _, gates) in enumerate(cells):
            for gi, inst in enumerate(gates):
                _fill_axis_map(mats[gi, ci], inst.gate, inst.theta)
        acc = mats[0] + 0.0                     # M @ I == M (and -0.0 -> 0.0, like the product)
        for gi in range(1, length):
            acc = np.matmul(mats[gi], acc)
        ks = [c[0] for c in cells]
        ws = [c[1] for c in cells]
        blocks = acc.transpose(0, 2, 1)
        lut[ks, ws] = blocks
        p, t = classify_lut(np.ascontiguousarray(blocks)[None])
        is_perm[ks, ws] = p[0]
        table[ks, ws] = t[0]
    return lut, is_perm, table


_FIXED_ARRAYS = {name: np.array(rows) for name, rows in _FIXED.items()}
_FIXED_BLOCKS: dict = {}


# CX tables indexed [control axis, target axis] (reference lut.py:108-134).
# Derived here from the x/z rule instead of typed in: with code bits (hi, lo),
# z = hi and x = hi ^ lo;  CX: x_t ^= x_c, z_c ^= z_t, sign = -1 iff
# x_c & z_t & ~(x_t ^ z_c) on the inputs.
def _cx_tables():
    tc = np.zeros((4, 4), dtype=np.int64)
    tt = np.zeros((4, 4), dtype=np.int64)
    ts = np.ones((4, 4), dtype=np.int64)
    for dc in range(4):
        for dt in range(4):
            zc, xc = dc >> 1, (dc >> 1) ^ (dc & 1)
            zt, xt = dt >> 1, (dt >> 1) ^ (dt & 1)
            if xc & zt & (1 ^ xt ^ zc):
                ts[dc, dt] = -1
            xt2, zc2 = xt ^ xc, zc ^ zt
            tc[dc, dt] = (zc2 << 1) | (zc2 ^ xc)
            tt[dc, dt] = (zt << 1) | (zt ^ xt2)
    return tc, tt, ts


LUT_C, LUT_T, LUT_SIGN = _cx_tables()


def cx_lookup(c: int, t: int) -> tuple:
    """(c', t', sign) of CX conjugation on one (control, target) axis pair."""
    return int(LUT_C[c, t]), int(LUT_T[c, t]), int(LUT_SIGN[c, t])


_cx_words_for = [None, None]      # (bytes of the sign table the cached words were packed from, the words)


def cx_device_words(sign_table=None) -> tuple:
    """The three CX tables packed for the kernel: 2 bits (axes) / 1 bit (sign) per entry.

    ``sign_table`` lets the tests inject a corrupted table (the reference's
    mutation check, tests/test_cli.py:198-203) and see parity fail.
    """
    sign = LUT_SIGN if sign_table is None else sign_table
    stamp = sign.tobytes()                        # every store asks; the tables only change in mutation tests
    if stamp == _cx_words_for[0]:
        return _cx_words_for[1]
    wc = wt = ws = 0
    for dc in range(4):
        for dt in range(4):
            e = dc * 4 + dt
            wc |= int(LUT_C[dc, dt]) << (2 * e)
            wt |= int(LUT_T[dc, dt]) << (2 * e)
            ws |= (1 if sign[dc, dt] < 0 else 0) << e
    _cx_words_for[0], _cx_words_for[1] = stamp, (wc, wt, ws)
    return wc, wt, ws


STANDARD_CX = cx_device_words()   # the reference's tables; folded runs and circuit programs assume them


def perm_word(block: np.ndarray):
    """Pack a 3x3 block as a signed axis permutation, or None if it is not one.

    A block qualifies only if every row has exactly one nonzero and that entry
    is exactly +1.0 or -1.0 -- then conjugation neither branches nor rescales,
    so no merge is needed after it.  Layout (12 bits, the table field of a
    ``qx_apply_clifford`` op): bits 2a..2a+1 = image axis of input axis a
    (a = 0 is the identity and maps to 0), bit 8+a = 1 for a minus sign.
    """
    word = 0
    for p in (1, 2, 3):
        row = block[p - 1]
        hot = np.flatnonzero(row)
        if len(hot) != 1:
            return None
        v = row[hot[0]]
        if v != 1.0 and v != -1.0:
            return None
        word |= (int(hot[0]) + 1) << (2 * p)
        if v < 0.0:
            word |= 1 << (8 + p)
    return word


def perm_op(n: int, qubit: int, table: int) -> int:
    """Op word of a 1q signed permutation on ``qubit`` (include/qimax_b200.h): 32 bits for n <= 32,
    the 64-bit form of qx_apply_clifford_wide above (digit positions in the high half)."""
    if n > 32:
        return 0 | (table << 16) | ((2 * (n - 1 - qubit)) << 32)
    return 0 | ((2 * (n - 1 - qubit)) << 2) | (table << 16)


def cx_op(n: int, control: int, target: int) -> int:
    """Op word of CX(control, target); see perm_op."""
    if n > 32:
        return 1 | ((2 * (n - 1 - control)) << 32) | ((2 * (n - 1 - target)) << 48)
    return 1 | ((2 * (n - 1 - control)) << 2) | ((2 * (n - 1 - target)) << 8)


def op_dtype(n: int):
    """numpy dtype of a gate program for an n-qubit store."""
    return np.uint64 if n > 32 else np.uint32


IDENTITY_PERM = perm_word(np.eye(3))


def branch_table(block3: np.ndarray) -> tuple:
    """(counts[3], axes[3][3], weights[3][3]) of one qubit's block.

    Row p-1 describes input axis p: its nonzero output weights in ascending
    axis order (the reference's ragged cell, stabilizer.py:209-214).  Unused
    slots hold axis 0 / weight 0.0.
    """
    counts = np.zeros(3, dtype=np.int32)
    axes = np.zeros((3, 3), dtype=np.int32)
    weights = np.zeros((3, 3), dtype=np.float64)
    for p in range(3):
        hot = np.flatnonzero(block3[p])
        counts[p] = len(hot)
        axes[p, : len(hot)] = hot + 1
        weights[p, : len(hot)] = block3[p, hot]
    return counts, axes, weights


def gate_branch_block(gate: str, theta: float) -> np.ndarray:
    """The block a lone gate contributes: row p = column p of its axis map.

    This is what v1's per-digit tables (reference engine.py:190-202) read:
    for input digit d the candidates are the nonzeros of column d-1.
    """
    return np.ascontiguousarray(axis_map(gate, theta).T)


def classify_lut(lut: np.ndarray) -> tuple:
    """Vectorised ``perm_word`` over a whole (K, n, 3, 3) tensor.

    Returns (is_perm bool[K, n], table uint32[K, n]); ``table`` is only
    meaningful where ``is_perm``.
    """
    nz = lut != 0.0
    one_hot = nz.sum(axis=-1) == 1                                   # (K, n, 3)
    unit = np.where(nz, np.abs(lut) == 1.0, True).all(axis=-1)       # nonzeros are exactly +-1
    is_perm = (one_hot & unit).all(axis=-1)
    image = nz.argmax(axis=-1).astype(np.uint32) + 1                  # (K, n, 3)
    minus = (lut.sum(axis=-1) < 0.0).astype(np.uint32)
    table = np.zeros(lut.shape[:2], dtype=np.uint32)
    for p in (1, 2, 3):
        table |= image[..., p - 1] << np.uint32(2 * p)
        table |= minus[..., p - 1] << np.uint32(8 + p)
    return is_perm, table


FIXED_PERMS = {name: perm_word(axis_map(name).T) for name in ("H", "S", "X", "SX")}


def operator_tables(block: np.ndarray) -> tuple:
    """Branch tables of a whole U_k: (counts[n,3], axes[n,3,3], weights[n,3,3])."""
    n = block.shape[0]
    nz = block != 0.0
    counts = nz.sum(axis=-1).astype(np.int32)
    # stable argsort of "is zero" lists the nonzero axes first, ascending
    order = np.argsort(~nz, axis=-1, kind="stable")
    weights = np.take_along_axis(block, order, axis=-1)
    axes = (order + 1).astype(np.int32)
    slot = np.arange(3)[None, None, :]
    dead = slot >= counts[..., None]
    axes[dead] = 0
    weights = np.where(dead, 0.0, weights)
    assert counts.shape == (n, 3)
    return counts, axes, np.ascontiguousarray(weights)
