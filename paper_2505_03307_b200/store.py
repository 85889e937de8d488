"""Python handle on the HBM term store (``qx_store`` in include/qimax_b200.h).

Thin by design: every method is one C-ABI call.  Host <-> device copies happen
only in ``upload`` / ``download``; everything else leaves the terms in HBM.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native as nat
from . import lut


# host threads of a narrow download: four saturate what the host memory system spares next to the DMA
# (more only contend with it: 35.4 ms with 4, 39.8 ms with 8 on a 16-core host)
PROGRAM_TERMS = 4096              # terms per generator a one-launch run can return (kPgSrcCap, csrc/program.cuh)
HOST_WIDEN_THREADS = int(os.environ.get("QX_WIDEN_THREADS", 0)) or max(1, min(4, (os.cpu_count() or 2) // 2))


class DeviceStore:
    """n_segments generators of an n-qubit system, structure-of-arrays in HBM."""

    def __init__(self, n: int, n_segments: int, capacity: int = 0, device=None):
        self.n = int(n)
        self.n_segments = int(n_segments)
        self.words = 1 if self.n <= 32 else (2 * self.n + 63) // 64       # > 1: multi-word keys (csrc/wide.cu)
        self.device = nat.default_device() if device is None else int(device)
        self._h = C.c_void_p()
        nat.check(nat.lib().qx_store_create(self.device, self.n, self.n_segments, int(capacity),
                                            C.byref(self._h)))
        self._cx = lut.cx_device_words()

    # -- lifetime ---------------------------------------------------------------
    def close(self):
        h, self._h = self._h, None
        if h is not None and h.value:
            nat.check(nat.lib().qx_store_destroy(h))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def support(self) -> list:
        """Per segment, the qubits on which some term has a non-identity digit (qx_store_support),
        as integer masks with bit q set for qubit q."""
        words = np.zeros((self.n_segments, self.words), dtype=np.uint64)
        nat.check(nat.lib().qx_store_support(self._h, nat.ptr(words)))
        out = []
        for row in words.tolist():
            key_mask = sum(int(w) << (64 * i) for i, w in enumerate(row))
            m = 0
            for q in range(self.n):
                if (key_mask >> (2 * (self.n - 1 - q))) & 1:
                    m |= 1 << q
            out.append(m)
        return out

    def compact(self, qubits, take) -> "DeviceStore":
        """A one-word store over the selected qubits holding the terms of the segments in ``take``
        (bool per segment); the other segments are empty in it."""
        sel = np.ascontiguousarray(qubits, dtype=np.int32)
        flags = np.ascontiguousarray(take, dtype=np.uint8)
        narrow = DeviceStore(len(sel), self.n_segments, 0, self.device)
        try:
            nat.check(nat.lib().qx_store_compact(self._h, nat.ptr(sel), len(sel), nat.ptr(flags), narrow._h))
        except BaseException:
            narrow.close()
            raise
        return narrow

    def expand_from(self, narrow: "DeviceStore", qubits, take):
        """Replace the segments in ``take`` by the one-word store's, spread back over the selected qubits."""
        sel = np.ascontiguousarray(qubits, dtype=np.int32)
        flags = np.ascontiguousarray(take, dtype=np.uint8)
        nat.check(nat.lib().qx_store_expand(narrow._h, nat.ptr(sel), len(sel), nat.ptr(flags), self._h))

    def mark(self) -> int:
        """A CUDA event on the store's stream (qx_store_event_record); returns its index."""
        idx = C.c_int32()
        nat.check(nat.lib().qx_store_event_record(self._h, C.byref(idx)))
        return idx.value

    def elapsed_ms(self, first: int, second: int) -> float:
        ms = C.c_double()
        nat.check(nat.lib().qx_store_event_elapsed(self._h, int(first), int(second), C.byref(ms)))
        return ms.value

    def set_stream(self, cuda_stream: int):
        nat.check(nat.lib().qx_store_set_stream(self._h, C.c_void_p(int(cuda_stream))))

    def set_cx_tables(self, sign_table):
        """Test hook: run with a (possibly corrupted) CX sign table."""
        self._cx = lut.cx_device_words(sign_table)

    # -- content ----------------------------------------------------------------
    def init_z(self, qubits=None):
        arr = None if qubits is None else np.ascontiguousarray(qubits, dtype=np.int32)
        if arr is not None and len(arr) != self.n_segments:
            raise ValueError(f"expected {self.n_segments} qubits, got {len(arr)}")
        nat.check(nat.lib().qx_store_init_z(self._h, nat.ptr(arr)))

    def upload(self, gens):
        """gens: sequence of (lambdas, keys) per segment."""
        if len(gens) != self.n_segments:
            raise ValueError(f"expected {self.n_segments} segments, got {len(gens)}")
        off = np.zeros(self.n_segments + 1, dtype=np.int64)
        for i, (lam, keys) in enumerate(gens):
            if len(lam) != len(keys):
                raise ValueError("lambdas and indices must have equal length")
            off[i + 1] = off[i] + len(lam)
        lam = np.empty(int(off[-1]), dtype=np.float64)
        if self.words > 1:
            # multi-word keys: Python ints -> little-endian 64-bit words, term-major
            words = np.zeros((int(off[-1]), self.words), dtype=np.uint64)
            mask = (1 << 64) - 1
            for i, (l, k) in enumerate(gens):
                for j, v in enumerate(k):
                    v = int(v)
                    if v < 0 or v >= 4 ** self.n:
                        raise ValueError(f"word index out of range [0, 4**{self.n})")
                    for w in range(self.words):
                        words[off[i] + j, w] = (v >> (64 * w)) & mask
                lam[off[i]:off[i + 1]] = l
            nat.check(nat.lib().qx_store_upload_wide(self._h, nat.ptr(off), nat.ptr(words), nat.ptr(lam)))
            return
        keys = np.empty(int(off[-1]), dtype=np.uint64)
        for i, (l, k) in enumerate(gens):
            keys[off[i]:off[i + 1]] = np.asarray(k, dtype=np.uint64) if not _is_object(k) else [int(v) for v in k]
            lam[off[i]:off[i + 1]] = l
        nat.check(nat.lib().qx_store_upload(self._h, nat.ptr(off), nat.ptr(keys), nat.ptr(lam)))

    def ranks(self) -> list:
        out = np.zeros(self.n_segments, dtype=np.int64)
        nat.check(nat.lib().qx_store_ranks(self._h, nat.ptr(out)))
        return out.tolist()

    def download(self, pinned: bool = False):
        """(offsets int64[n_seg+1], keys uint64[total], lambdas float64[total]) on the host."""
        off = np.zeros(self.n_segments + 1, dtype=np.int64)
        if self.words > 1:
            nat.check(nat.lib().qx_store_download_wide(self._h, nat.ptr(off), None, None, 0))
            total = int(off[-1])
            words = np.zeros((total, self.words), dtype=np.uint64)
            lam = np.empty(total, dtype=np.float64)
            nat.check(nat.lib().qx_store_download_wide(self._h, nat.ptr(off), nat.ptr(words), nat.ptr(lam), total))
            keys = np.empty(total, dtype=object)                  # Python ints, like the reference above 31 qubits
            rows = words.tolist()
            keys[:] = [sum(int(w) << (64 * i) for i, w in enumerate(row)) for row in rows]
            return off, keys, lam
        nat.check(nat.lib().qx_store_download(self._h, nat.ptr(off), None, None, 0))
        total = int(off[-1])
        if pinned and total > 0:
            buf = nat.PINNED.take(16 * total)
            keys = buf.view(np.uint64, 0, total)
            lam = buf.view(np.float64, 8 * total, total)
        else:
            keys = np.empty(total, dtype=np.uint64)
            lam = np.empty(total, dtype=np.float64)
        nat.check(nat.lib().qx_store_download(self._h, nat.ptr(off), nat.ptr(keys), nat.ptr(lam), total))
        return off, keys, lam

    def slice(self, seg_lo: int, seg_hi: int, capacity: int = 0) -> "DeviceStore":
        """A new store with copies of segments [seg_lo, seg_hi), on a CUDA stream of its own."""
        child = object.__new__(DeviceStore)
        child.n, child.n_segments, child.device = self.n, int(seg_hi) - int(seg_lo), self.device
        child.words = self.words
        child._h = C.c_void_p()
        child._cx = self._cx
        nat.check(nat.lib().qx_store_slice(self._h, int(seg_lo), int(seg_hi), int(capacity), C.byref(child._h)))
        return child

    def set_keep_narrow(self, on=True):
        """The store is only downloaded next: let the operator step leave 32-bit keys (n <= 16);
        ``on=2`` also allows the packed form (16-bit low halves + bucket tables) for large results."""
        nat.check(nat.lib().qx_store_set_keep_narrow(self._h, int(on)))
        self._keep_narrow = bool(on)

    def download_async(self, pinned: bool = True):
        """Like download, but the term copies are only queued on the store's stream: the arrays
        are valid after ``synchronize()``.  A store left with 32-bit keys ships them as such and
        host threads widen them while the copy runs (12 instead of 16 bytes per term over PCIe)."""
        off = np.zeros(self.n_segments + 1, dtype=np.int64)
        nat.check(nat.lib().qx_store_ranks(self._h, nat.ptr(off[1:])))
        np.cumsum(off[1:], out=off[1:])
        total = int(off[-1])
        if pinned and total > 0 and getattr(self, "_keep_narrow", False):
            words = total + 65537 * self.n_segments + 2            # enough for either narrow form
            buf = nat.PINNED.take(16 * total + 4 * words)
            keys = buf.view(np.uint64, 0, total)
            lam = buf.view(np.float64, 8 * total, total)
            staging = buf.view(np.uint32, 16 * total, words)
            self._staging = staging                                # alive until synchronize()
            d2h = C.c_int64()
            nat.check(nat.lib().qx_store_download_packed_async(
                self._h, nat.ptr(off), nat.ptr(keys), nat.ptr(lam), total, nat.ptr(staging), words,
                HOST_WIDEN_THREADS, C.byref(d2h)))
            self.d2h_bytes = int(d2h.value)
            return off, keys, lam
        self.d2h_bytes = 16 * total
        if pinned and total > 0:
            buf = nat.PINNED.take(16 * total)
            keys = buf.view(np.uint64, 0, total)
            lam = buf.view(np.float64, 8 * total, total)
        else:
            keys = np.empty(total, dtype=np.uint64)
            lam = np.empty(total, dtype=np.float64)
        nat.check(nat.lib().qx_store_download_async(self._h, nat.ptr(off), nat.ptr(keys), nat.ptr(lam), total))
        return off, keys, lam

    def segments(self, pinned: bool = False) -> list:
        """[(lambdas, keys)] per segment (views into one download)."""
        off, keys, lam = self.download(pinned)
        return [(lam[off[i]:off[i + 1]], keys[off[i]:off[i + 1]]) for i in range(self.n_segments)]

    def device_view(self) -> tuple:
        k, l, o = C.c_void_p(), C.c_void_p(), C.c_void_p()
        nat.check(nat.lib().qx_store_device_view(self._h, C.byref(k), C.byref(l), C.byref(o)))
        return k.value, l.value, o.value

    def capacity(self) -> tuple:
        cap, hbm = C.c_int64(), C.c_int64()
        nat.check(nat.lib().qx_store_capacity(self._h, C.byref(cap), C.byref(hbm)))
        return cap.value, hbm.value

    def synchronize(self):
        nat.check(nat.lib().qx_store_synchronize(self._h))

    # -- kernels ----------------------------------------------------------------
    def apply_clifford(self, program):
        c, t, s = self._cx
        if self.words > 1:
            prog = np.ascontiguousarray(program, dtype=np.uint64)        # lut.perm_op / cx_op wide form
            if len(prog):
                nat.check(nat.lib().qx_apply_clifford_wide(self._h, nat.ptr(prog), len(prog), c, t, s))
            return
        prog = np.ascontiguousarray(program, dtype=np.uint32)
        if len(prog):
            nat.check(nat.lib().qx_apply_clifford(self._h, nat.ptr(prog), len(prog), c, t, s))

    def apply_split(self, qubit: int, a1, w1, a2, w2):
        a1 = np.ascontiguousarray(a1, dtype=np.int32)
        a2 = np.ascontiguousarray(a2, dtype=np.int32)
        w1 = np.ascontiguousarray(w1, dtype=np.float64)
        w2 = np.ascontiguousarray(w2, dtype=np.float64)
        fn = nat.lib().qx_apply_split_wide if self.words > 1 else nat.lib().qx_apply_split
        nat.check(fn(self._h, int(qubit), nat.ptr(a1), nat.ptr(w1), nat.ptr(a2), nat.ptr(w2)))

    def apply_operator(self, counts, axes, weights, term_limit: int = 0) -> int:
        counts = np.ascontiguousarray(counts, dtype=np.int32).reshape(-1)
        axes = np.ascontiguousarray(axes, dtype=np.int32).reshape(-1)
        weights = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1)
        raw = C.c_int64()
        nat.check(nat.lib().qx_apply_operator(self._h, nat.ptr(counts), nat.ptr(axes), nat.ptr(weights),
                                              int(term_limit), C.byref(raw)))
        return raw.value

    def apply_operator_run(self, counts, axes, weights, program, eps: float, term_limit: int = 0):
        """U_k + the sign-permutation run behind it + merge in one call; returns (raw, ranks)."""
        counts = np.ascontiguousarray(counts, dtype=np.int32).reshape(-1)
        axes = np.ascontiguousarray(axes, dtype=np.int32).reshape(-1)
        weights = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1)
        prog = np.ascontiguousarray(program, dtype=np.uint32)
        raw = C.c_int64()
        ranks = np.zeros(self.n_segments, dtype=np.int64)
        c, t, s = self._cx
        nat.check(nat.lib().qx_apply_operator_run(
            self._h, nat.ptr(counts), nat.ptr(axes), nat.ptr(weights), nat.ptr(prog) if len(prog) else None,
            len(prog), c, t, s, float(eps), int(term_limit), C.byref(raw), nat.ptr(ranks)))
        return raw.value, ranks.tolist()

    def apply_operator_run_part(self, counts, axes, weights, program, eps: float, part: int, parts: int):
        """The part-th of `parts` slot ranges of U_k + run + merge (multi-GPU, last branching
        operator); returns (ranks of this share, partitioned flag)."""
        counts = np.ascontiguousarray(counts, dtype=np.int32).reshape(-1)
        axes = np.ascontiguousarray(axes, dtype=np.int32).reshape(-1)
        weights = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1)
        prog = np.ascontiguousarray(program, dtype=np.uint32)
        ranks = np.zeros(self.n_segments, dtype=np.int64)
        flag = C.c_int32()
        c, t, s = self._cx
        nat.check(nat.lib().qx_apply_operator_run_part(
            self._h, nat.ptr(counts), nat.ptr(axes), nat.ptr(weights), nat.ptr(prog) if len(prog) else None,
            len(prog), c, t, s, float(eps), int(part), int(parts), nat.ptr(ranks), C.byref(flag)))
        return ranks.tolist(), bool(flag.value)

    def run_program(self, program: "CircuitProgram", eps: float, init_qubits=None, to_host: bool = False,
                    pinned: bool = False, max_steps: int = 0):
        """The whole compiled circuit in one launch (qx_store_run_program).  Returns (fitted, ranks,
        raw, segments): ranks[row][g] after the row-th branching step; fitted False = the store is
        untouched (or holds init_z if init_qubits was given).  init_qubits: start from Z words made in
        the kernel instead of the store's content.  to_host: the kernel also writes the result into
        page-locked host memory; segments = [(lambdas, keys)] then (views of the pinned block if
        ``pinned``, fresh arrays otherwise), else None.  max_steps > 0: only the first max_steps steps."""
        ranks = np.zeros((max(program.rows, 1), self.n_segments), dtype=np.int64)
        raw, fitted, filled = C.c_int64(), C.c_int32(), C.c_int32()
        off = np.zeros(self.n_segments + 1, dtype=np.int64)
        init = None if init_qubits is None else np.ascontiguousarray(init_qubits, dtype=np.int32)
        keys = lam = None
        cap = 0
        if to_host:
            # room for every generator at the kernel's limit, but never more than 64 MB of pinned
            # memory: a result that does not fit is downloaded the ordinary way
            cap = min(self.n_segments * PROGRAM_TERMS, 1 << 22)
            buf = nat.PINNED.take(16 * cap)
            keys = buf.view(np.uint64, 0, cap)
            lam = buf.view(np.float64, 8 * cap, cap)
        dev_ms, stopped = C.c_double(), C.c_int32()
        nat.check(nat.lib().qx_store_run_program(self._h, program.handle, nat.ptr(init), float(eps), nat.ptr(ranks),
                                                 C.byref(raw), C.byref(fitted), nat.ptr(off), nat.ptr(keys), nat.ptr(lam),
                                                 cap, C.byref(filled), C.byref(dev_ms), int(max_steps), C.byref(stopped)))
        self.program_ms = dev_ms.value         # duration of the launch on the GPU's clock
        self.program_stopped = stopped.value   # not fitted: the first step that outgrew shared memory
        segs = None
        if fitted.value and filled.value:
            o = off.tolist()
            if pinned:
                segs = [(lam[o[i]:o[i + 1]], keys[o[i]:o[i + 1]]) for i in range(self.n_segments)]
            else:
                total = o[-1]
                k2, l2 = keys[:total].copy(), lam[:total].copy()
                segs = [(l2[o[i]:o[i + 1]], k2[o[i]:o[i + 1]]) for i in range(self.n_segments)]
        return bool(fitted.value), ranks[:program.rows].tolist(), raw.value, segs

    def count_operator(self, counts) -> list:
        counts = np.ascontiguousarray(counts, dtype=np.int32).reshape(-1)
        out = np.zeros(self.n_segments, dtype=np.int64)
        nat.check(nat.lib().qx_count_operator(self._h, nat.ptr(counts), nat.ptr(out)))
        return out.tolist()

    def order_for_operator(self, counts, by_key: bool = True):
        """Source order of the reference's ragged flatten (qx_store_order_for_operator)."""
        counts = np.ascontiguousarray(counts, dtype=np.int32).reshape(-1)
        nat.check(nat.lib().qx_store_order_for_operator(self._h, nat.ptr(counts), 1 if by_key else 0))

    def merge(self, eps: float) -> list:
        out = np.zeros(self.n_segments, dtype=np.int64)
        nat.check(nat.lib().qx_merge(self._h, float(eps), nat.ptr(out)))
        return out.tolist()

    def sort(self):
        nat.check(nat.lib().qx_sort(self._h))

    def zi_sums(self) -> np.ndarray:
        out = np.zeros(self.n_segments, dtype=np.float64)
        nat.check(nat.lib().qx_store_zi_sums(self._h, nat.ptr(out)))
        return out

    def norms(self) -> np.ndarray:
        out = np.zeros(self.n_segments, dtype=np.float64)
        nat.check(nat.lib().qx_store_norms(self._h, nat.ptr(out)))
        return out

    def partition_by_owner(self, world: int) -> np.ndarray:
        out = np.zeros((int(world), self.n_segments), dtype=np.int64)
        nat.check(nat.lib().qx_store_partition_by_owner(self._h, int(world), nat.ptr(out)))
        return out

    def assemble(self, d_keys: int, d_lambdas: int, recv_counts):
        rc = np.ascontiguousarray(recv_counts, dtype=np.int64)
        nat.check(nat.lib().qx_store_assemble(self._h, C.c_void_p(int(d_keys)), C.c_void_p(int(d_lambdas)),
                                              rc.shape[0], nat.ptr(rc.reshape(-1))))


def _is_object(arr) -> bool:
    return isinstance(arr, np.ndarray) and arr.dtype == object


class CircuitProgram:
    """Device-resident step list of a circuit plan (``qx_program`` in include/qimax_b200.h).
    steps: ("clifford", ops) | ("oprun", order, counts, axes, weights, ops) | ("sort",)."""

    KINDS = {"clifford": 0, "oprun": 1, "sort": 2}

    def __init__(self, n: int, steps, device=None):
        self.n, self.device = int(n), nat.default_device() if device is None else int(device)
        ns = len(steps)
        kinds = np.zeros(ns, dtype=np.int32)
        order = np.zeros(ns, dtype=np.int32)
        counts = np.ones((ns, n, 3), dtype=np.int32)
        axes = np.zeros((ns, n, 3, 3), dtype=np.int32)
        weights = np.zeros((ns, n, 3, 3), dtype=np.float64)
        ops, off = [], [0]
        for i, st in enumerate(steps):
            kinds[i] = self.KINDS[st[0]]
            if st[0] == "clifford":
                ops.extend(st[1])
            elif st[0] == "oprun":
                order[i] = 1 if st[1] else 0
                counts[i] = np.asarray(st[2], dtype=np.int32).reshape(n, 3)
                axes[i] = np.asarray(st[3], dtype=np.int32).reshape(n, 3, 3)
                weights[i] = np.asarray(st[4], dtype=np.float64).reshape(n, 3, 3)
                ops.extend(st[5])
            off.append(len(ops))
        ops = np.asarray(ops, dtype=np.uint32)
        off = np.asarray(off, dtype=np.int64)
        self.rows = int((kinds == 1).sum())
        self.steps = ns
        self.fit_steps = None         # None: all steps fit one launch (as far as known); K: only the first K do
        self._h = C.c_void_p()
        nat.check(nat.lib().qx_program_create(self.device, self.n, ns, nat.ptr(kinds), nat.ptr(order), nat.ptr(counts),
                                              nat.ptr(axes), nat.ptr(weights), nat.ptr(ops) if len(ops) else None,
                                              nat.ptr(off), C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def close(self):
        h, self._h = self._h, None
        if h is not None and h.value:
            nat.check(nat.lib().qx_program_destroy(h))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
