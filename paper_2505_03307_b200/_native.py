"""ctypes binding of ``libqimax_b200.so`` (``include/qimax_b200.h``).

This is the only place the package touches native code.  There is no CPU
fallback: if the library is missing or no CUDA device is usable, every compute
entry point raises :class:`NativeError`.
"""

from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

from .errors import ConsistencyError, NativeError, ResourceLimitError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QX_LIB") or os.path.join(HERE, "lib", "libqimax_b200.so")   # QX_LIB: A/B builds (tools/build_variant.sh)
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "qimax_b200.h")

QX_OK, QX_ERR_INVALID, QX_ERR_RESOURCE, QX_ERR_CUDA, QX_ERR_UNSUPPORTED, QX_ERR_CONSISTENCY = range(6)

KERNEL_CLASSES = (
    "clifford", "split", "expand_count", "expand_emit", "sort_hist", "sort_pass",
    "reduce", "small_merge", "readout_product", "readout_reduce", "partition",
    "dense_prep", "dense_emit", "bucket_emit",
)

_i32, _i64, _u32, _u64, _f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
_p = C.c_void_p
_P = C.POINTER

# name -> (restype, argtypes); must list every function declared in the header
SIGNATURES = {
    "qx_abi_version": (C.c_int, []),
    "qx_last_error": (C.c_char_p, []),
    "qx_device_count": (C.c_int, [_P(C.c_int)]),
    "qx_device_info": (C.c_int, [C.c_int, C.c_char_p, C.c_int, _P(C.c_int), _P(C.c_int), _P(C.c_int),
                                 _P(_i64), _P(_i64)]),
    "qx_host_alloc": (C.c_int, [_i64, _P(_p)]),
    "qx_host_free": (C.c_int, [_p]),
    "qx_trim": (C.c_int, []),
    "qx_store_create": (C.c_int, [C.c_int, C.c_int, C.c_int, _i64, _P(_p)]),
    "qx_store_destroy": (C.c_int, [_p]),
    "qx_store_set_stream": (C.c_int, [_p, _p]),
    "qx_store_init_z": (C.c_int, [_p, _p]),
    "qx_store_upload": (C.c_int, [_p, _p, _p, _p]),
    "qx_store_ranks": (C.c_int, [_p, _p]),
    "qx_store_download": (C.c_int, [_p, _p, _p, _p, _i64]),
    "qx_store_device_view": (C.c_int, [_p, _P(_p), _P(_p), _P(_p)]),
    "qx_store_capacity": (C.c_int, [_p, _P(_i64), _P(_i64)]),
    "qx_store_synchronize": (C.c_int, [_p]),
    "qx_store_event_record": (C.c_int, [_p, _P(_i32)]),
    "qx_store_event_elapsed": (C.c_int, [_p, _i32, _i32, _P(_f64)]),
    "qx_store_slice": (C.c_int, [_p, _i32, _i32, _i64, _P(_p)]),
    "qx_store_words": (C.c_int, [_p, _P(_i32)]),
    "qx_store_upload_wide": (C.c_int, [_p, _p, _p, _p]),
    "qx_store_download_wide": (C.c_int, [_p, _p, _p, _p, _i64]),
    "qx_store_support": (C.c_int, [_p, _p]),
    "qx_store_compact": (C.c_int, [_p, _p, _i32, _p, _p]),
    "qx_store_expand": (C.c_int, [_p, _p, _i32, _p, _p]),
    "qx_apply_clifford_wide": (C.c_int, [_p, _p, _i32, _u32, _u32, _u32]),
    "qx_apply_split_wide": (C.c_int, [_p, _i32, _p, _p, _p, _p]),
    "qx_store_download_async": (C.c_int, [_p, _p, _p, _p, _i64]),
    "qx_store_set_keep_narrow": (C.c_int, [_p, C.c_int]),
    "qx_store_download_narrow_async": (C.c_int, [_p, _p, _p, _p, _i64, _p, _i32]),
    "qx_store_download_packed_async": (C.c_int, [_p, _p, _p, _p, _i64, _p, _i64, _i32, _p]),
    "qx_apply_clifford": (C.c_int, [_p, _p, _i32, _u32, _u32, _u32]),
    "qx_apply_split": (C.c_int, [_p, _i32, _p, _p, _p, _p]),
    "qx_apply_operator": (C.c_int, [_p, _p, _p, _p, _i64, _P(_i64)]),
    "qx_apply_operator_run": (C.c_int, [_p, _p, _p, _p, _p, _i32, _u32, _u32, _u32, _f64, _i64, _P(_i64), _p]),
    "qx_apply_operator_run_part": (C.c_int, [_p, _p, _p, _p, _p, _i32, _u32, _u32, _u32, _f64, _i32, _i32, _p, _P(_i32)]),
    "qx_count_operator": (C.c_int, [_p, _p, _p]),
    "qx_store_order_for_operator": (C.c_int, [_p, _p, C.c_int32]),
    "qx_operator_classes": (C.c_int, [_i32, _p, _p, _p, _p, _p, _p, _p]),
    "qx_bucket_last": (C.c_int, [_P(_i64)]),
    "qx_bucket_enable": (C.c_int, [_i32]),
    "qx_dense_last": (C.c_int, [_P(_i64)]),
    "qx_program_create": (C.c_int, [C.c_int, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _P(_p)]),
    "qx_program_destroy": (C.c_int, [_p]),
    "qx_program_rows": (C.c_int, [_p, _P(_i32)]),
    "qx_store_run_program": (C.c_int, [_p, _p, _p, _f64, _p, _P(_i64), _P(_i32), _p, _p, _p, _i64, _P(_i32), _P(_f64),
                                       _i32, _P(_i32)]),
    "qx_merge": (C.c_int, [_p, _f64, _p]),
    "qx_sort": (C.c_int, [_p]),
    "qx_store_zi_sums": (C.c_int, [_p, _p]),
    "qx_store_norms": (C.c_int, [_p, _p]),
    "qx_expansion_create": (C.c_int, [C.c_int, C.c_int, _i64, _P(_p)]),
    "qx_expansion_destroy": (C.c_int, [_p]),
    "qx_expansion_reset": (C.c_int, [_p]),
    "qx_expansion_multiply": (C.c_int, [_p, _p, _p, _i64, _i64]),
    "qx_expansion_multiply_segment": (C.c_int, [_p, _p, _i32, _i64]),
    "qx_expansion_size": (C.c_int, [_p, _P(_i64)]),
    "qx_expansion_max_abs_imag": (C.c_int, [_p, _P(_f64)]),
    "qx_expansion_download": (C.c_int, [_p, _p, _p, _p, _i64]),
    "qx_expansion_lookup": (C.c_int, [_p, _p, _i64, _p]),
    "qx_store_partition_by_owner": (C.c_int, [_p, _i32, _p]),
    "qx_store_assemble": (C.c_int, [_p, _p, _p, _i32, _p]),
    "qx_profile_enable": (C.c_int, [C.c_int]),
    "qx_profile_reset": (C.c_int, []),
    "qx_profile_read": (C.c_int, [C.c_int, _P(_i64), _P(_f64), _P(_f64)]),
    "qx_launch_count": (C.c_int, [_P(_i64)]),
}

_lib = None


def header_symbols() -> list:
    """Function names declared in include/qimax_b200.h."""
    with open(HEADER_PATH) as fh:
        text = re.sub(r"/\*.*?\*/", "", fh.read(), flags=re.S)
    return sorted(set(re.findall(r"\b(qx_[a-z0-9_]+)\s*\(", text)))


def lib():
    """The loaded library (loads on first use; never falls back)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(nvcc, sm_100a). There is no CPU fallback."
            )
        try:
            handle = C.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeError(f"cannot load {LIB_PATH}: {exc}") from None
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype, fn.argtypes = res, args
        if handle.qx_abi_version() != 1:
            raise NativeError(f"ABI version {handle.qx_abi_version()} != 1")
        _lib = handle
    return _lib


def last_error() -> str:
    return lib().qx_last_error().decode("utf-8", "replace")


def check(status: int) -> None:
    """Raise the reference's exception class for a non-zero qx_status."""
    if status == QX_OK:
        return
    msg = last_error()
    if status == QX_ERR_INVALID:
        raise ValueError(msg)
    if status == QX_ERR_RESOURCE:
        raise ResourceLimitError(msg)
    if status == QX_ERR_CONSISTENCY:
        raise ConsistencyError(msg)
    raise NativeError(msg)


def ptr(arr) -> C.c_void_p:
    """Raw data pointer of a C-contiguous numpy array (None -> NULL)."""
    if arr is None:
        return C.c_void_p(0)
    assert arr.flags["C_CONTIGUOUS"]
    return C.c_void_p(arr.ctypes.data)


def device_count() -> int:
    n = C.c_int(0)
    check(lib().qx_device_count(C.byref(n)))
    return n.value


def default_device() -> int:
    """QX_DEVICE, else LOCAL_RANK (one process per GPU under torchrun), else 0."""
    for var in ("QX_DEVICE", "LOCAL_RANK"):
        if os.environ.get(var, "") != "":
            return int(os.environ[var])
    return 0


def device_info(device: int = 0) -> dict:
    name = C.create_string_buffer(256)
    sm, major, minor = C.c_int(), C.c_int(), C.c_int()
    total, free = _i64(), _i64()
    check(lib().qx_device_info(device, name, 256, C.byref(sm), C.byref(major), C.byref(minor),
                               C.byref(total), C.byref(free)))
    return {"name": name.value.decode(), "sm_count": sm.value, "cc": (major.value, minor.value),
            "total_bytes": total.value, "free_bytes": free.value}


class PinnedBuffer:
    """Page-locked host allocation exposed as numpy views (keeps itself alive via .base)."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        raw = C.c_void_p()
        check(lib().qx_host_alloc(self.nbytes, C.byref(raw)))
        self._raw = raw
        self._ctype = (C.c_uint8 * max(self.nbytes, 8)).from_address(raw.value)
        # numpy views keep the ctypes array alive; the array keeps this object alive, so the
        # pinned block is only released once the last view is gone
        self._ctype._qx_owner = self

    def view(self, dtype, offset: int, count: int) -> np.ndarray:
        return np.frombuffer(self._ctype, dtype=dtype, count=count, offset=offset)

    def __del__(self):
        raw, self._raw = getattr(self, "_raw", None), None
        if raw is not None and raw.value and _lib is not None:
            try:
                _lib.qx_host_free(raw)
            except Exception:
                pass


class PinnedPool:
    """Reuses page-locked blocks across downloads: pinning gigabytes costs far more than the
    copy itself.  A block is handed out again only when no numpy view of it is alive."""

    def __init__(self, keep: int = 4):
        self.keep, self.blocks = keep, []

    def take(self, nbytes: int) -> PinnedBuffer:
        import sys

        best = None
        for blk in self.blocks:
            idle = sys.getrefcount(blk._ctype) <= 2          # blk._ctype + getrefcount's argument
            if idle and blk.nbytes >= nbytes and (best is None or blk.nbytes < best.nbytes):
                best = blk
        if best is None:
            best = PinnedBuffer(nbytes + nbytes // 16)
            self.blocks.append(best)
            if len(self.blocks) > self.keep:                 # forget the oldest; it frees itself
                self.blocks.pop(0)                           # once its last view is gone
        return best


PINNED = PinnedPool()


def profile_enable(on: bool = True) -> None:
    check(lib().qx_profile_enable(1 if on else 0))


def profile_reset() -> None:
    check(lib().qx_profile_reset())


def profile_read() -> dict:
    """{kernel class: {"launches", "ms", "alg_bytes"}} since the last reset."""
    out = {}
    for i, name in enumerate(KERNEL_CLASSES):
        n, ms, by = _i64(), _f64(), _f64()
        check(lib().qx_profile_read(i, C.byref(n), C.byref(ms), C.byref(by)))
        out[name] = {"launches": n.value, "ms": ms.value, "alg_bytes": by.value}
    return out


def trim() -> None:
    """Give cached device blocks back to the driver."""
    check(lib().qx_trim())


def launch_count() -> int:
    n = _i64()
    check(lib().qx_launch_count(C.byref(n)))
    return n.value


def bucket_enable(on: bool) -> bool:
    """Switch the bucketed operator step (csrc/bucket.cuh) on/off; returns the previous setting."""
    return bool(lib().qx_bucket_enable(1 if on else 0))


def dense_last() -> dict:
    """What the last grouped operator step did: groups, and how many had their sums formed mode by mode."""
    out = (_i64 * 4)()
    check(lib().qx_dense_last(out))
    return dict(zip(("groups", "kron_groups", "kron_slots", "kron_sources"), (int(v) for v in out)))


def bucket_last() -> dict:
    """Geometry of the last bucketed operator step (cap == 0: it fell back to grouped step + sort)."""
    out = (_i64 * 8)()
    check(lib().qx_bucket_last(out))
    keys = ("groups", "tiles", "buckets", "max_bucket", "slots", "ell", "cap", "ctas_per_sm")
    return dict(zip(keys, (int(v) for v in out)))
