"""ctypes binding of include/kk_spgemm.h (argument marshalling only).

Every function here has the name of the C entry point it forwards to.  No step of
the SpGEMM path runs in Python: if libkk_spgemm.so is missing, load() raises.
"""
from __future__ import annotations

import ctypes
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libkk_spgemm.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "kk_spgemm.h")

KK_OK, KK_ERR_INVALID_ARG, KK_ERR_DIM_MISMATCH, KK_ERR_UNSUPPORTED_TYPE = 0, 1, 2, 3
KK_ERR_INDEX_OVERFLOW, KK_ERR_STALE_HANDLE, KK_ERR_OUT_OF_MEMORY, KK_ERR_CUDA = 4, 5, 6, 7
KK_I32, KK_I64 = 0, 1
KK_F32, KK_F64 = 0, 1
KK_STATS_MAX_BINS = 24  # include/kk_spgemm.h

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64


class kk_csr_t(ctypes.Structure):
    _fields_ = [("nrows", _i64), ("ncols", _i64), ("nnz", _i64), ("offset_type", ctypes.c_int),
                ("value_type", ctypes.c_int), ("row_map", _vp), ("entries", _vp), ("values", _vp)]


ALLOC_FN = ctypes.CFUNCTYPE(_vp, ctypes.c_size_t, _vp, _vp)
FREE_FN = ctypes.CFUNCTYPE(None, _vp, ctypes.c_size_t, _vp, _vp)


class kk_spgemm_opts_t(ctypes.Structure):
    _fields_ = [("sort_rows", ctypes.c_int), ("compression", ctypes.c_int), ("validate", ctypes.c_int),
                ("num_streams", ctypes.c_int), ("timing", ctypes.c_int),
                ("patterns", ctypes.c_int), ("deterministic", ctypes.c_int), ("alloc", ALLOC_FN), ("free", FREE_FN),
                ("alloc_ctx", _vp)]


class kk_spgemm_stats_t(ctypes.Structure):
    _fields_ = [("muladds", _i64), ("nnz_c", _i64), ("compressed_words", _i64), ("compression_used", ctypes.c_int),
                ("b_sorted", ctypes.c_int), ("b_strict", ctypes.c_int), ("num_symbolic_bins", ctypes.c_int),
                ("num_numeric_bins", ctypes.c_int), ("symbolic_bin_rows", _i64 * KK_STATS_MAX_BINS),
                ("numeric_bin_rows", _i64 * KK_STATS_MAX_BINS), ("kernel_launches", _i64), ("workspace_bytes", _i64)]


class kk_kernel_time_t(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 48), ("launches", _i64), ("total_ms", ctypes.c_double),
                ("max_ms", ctypes.c_double)]


class KKError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{status_string(status)}: {detail}")
        self.status = status
        self.detail = detail


_lib = None


def load() -> ctypes.CDLL:
    """Load libkk_spgemm.so (built by `python -m paper_2103_11991_b200.build`)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2103_11991_b200.build` "
                               "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        H = ctypes.c_void_p
        P = ctypes.POINTER
        lib.kk_spgemm_opts_default.argtypes = [P(kk_spgemm_opts_t)]
        lib.kk_spgemm_opts_default.restype = None
        lib.kk_spgemm_create.argtypes = [P(H), ctypes.c_int, P(kk_spgemm_opts_t)]
        lib.kk_spgemm_destroy.argtypes = [H]
        lib.kk_spgemm_row_flops.argtypes = [H, P(kk_csr_t), P(kk_csr_t), _vp, _vp, P(_i64), _vp]
        lib.kk_spgemm_compress.argtypes = [H, P(kk_csr_t), _vp, _vp, _vp]
        lib.kk_spgemm_symbolic.argtypes = [H, P(kk_csr_t), P(kk_csr_t), _vp, P(_i64), _vp]
        lib.kk_spgemm_numeric.argtypes = [H, P(kk_csr_t), P(kk_csr_t), _vp, _vp, _vp, _vp]
        lib.kk_spgemm_jacobi_numeric.argtypes = [H, ctypes.c_double, _vp, P(kk_csr_t), P(kk_csr_t), _vp, _vp, _vp,
                                                 _vp]
        lib.kk_spadd_symbolic.argtypes = [H, P(kk_csr_t), P(kk_csr_t), _vp, P(_i64), _vp]
        lib.kk_spadd_numeric.argtypes = [H, ctypes.c_double, P(kk_csr_t), ctypes.c_double, P(kk_csr_t), _vp, _vp,
                                         _vp, _vp]
        lib.kk_spgemm_stats.argtypes = [H, P(kk_spgemm_stats_t)]
        lib.kk_spgemm_multiply_host.argtypes = [H, P(kk_csr_t), P(kk_csr_t), _vp, P(_i64),
                                                P(ctypes.POINTER(ctypes.c_int32)), P(_vp), ctypes.c_int, _vp]
        lib.kk_spgemm_rap_symbolic.argtypes = [H, P(kk_csr_t), P(kk_csr_t), P(kk_csr_t), _vp, P(_i64), _vp]
        lib.kk_spgemm_rap_numeric.argtypes = [H, P(kk_csr_t), P(kk_csr_t), P(kk_csr_t), _vp, _vp, _vp, _vp]
        lib.kk_spgemm_kernel_times.argtypes = [H, P(kk_kernel_time_t), P(ctypes.c_int)]
        lib.kk_spgemm_timing_reset.argtypes = [H]
        for fn in ("kk_spgemm_create", "kk_spgemm_destroy", "kk_spgemm_row_flops", "kk_spgemm_compress",
                   "kk_spgemm_symbolic", "kk_spgemm_numeric", "kk_spgemm_jacobi_numeric", "kk_spgemm_stats",
                   "kk_spadd_symbolic", "kk_spadd_numeric", "kk_spgemm_multiply_host",
                   "kk_spgemm_rap_symbolic", "kk_spgemm_rap_numeric",
                   "kk_spgemm_kernel_times",
                   "kk_spgemm_timing_reset"):
            getattr(lib, fn).restype = ctypes.c_int
        lib.kk_status_string.argtypes = [ctypes.c_int]
        lib.kk_status_string.restype = ctypes.c_char_p
        lib.kk_last_error_detail.argtypes = [H]
        lib.kk_last_error_detail.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def header_functions() -> list:
    """Names of the functions include/kk_spgemm.h declares."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kk_\w+)\s*\(", src)) - {"kk_alloc_fn", "kk_free_fn"})


def status_string(status: int) -> str:
    return load().kk_status_string(int(status)).decode()


def _check(h, status: int):
    if status != KK_OK:
        detail = load().kk_last_error_detail(h).decode() if h else ""
        raise KKError(status, detail)


def kk_spgemm_opts_default() -> kk_spgemm_opts_t:
    o = kk_spgemm_opts_t()
    load().kk_spgemm_opts_default(ctypes.byref(o))
    return o


def kk_spgemm_create(device: int, opts: kk_spgemm_opts_t | None = None) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    st = load().kk_spgemm_create(ctypes.byref(h), int(device), ctypes.byref(opts) if opts is not None else None)
    if st != KK_OK:
        raise KKError(st, "kk_spgemm_create failed")
    return h


def kk_spgemm_destroy(h) -> None:
    _check(None, load().kk_spgemm_destroy(h))


def kk_spgemm_row_flops(h, A: kk_csr_t, B: kk_csr_t, flops_ptr: int, scan_ptr: int, want_total: bool,
                        stream: int) -> int | None:
    tot = _i64(0)
    st = load().kk_spgemm_row_flops(h, ctypes.byref(A), ctypes.byref(B), flops_ptr or None, scan_ptr or None,
                                    ctypes.byref(tot) if want_total else None, stream or None)
    _check(h, st)
    return int(tot.value) if want_total else None


def kk_spgemm_compress(h, B: kk_csr_t, len_ptr: int, pairs_ptr: int, stream: int) -> None:
    _check(h, load().kk_spgemm_compress(h, ctypes.byref(B), len_ptr or None, pairs_ptr or None, stream or None))


def kk_spgemm_symbolic(h, A: kk_csr_t, B: kk_csr_t, c_row_map_ptr: int, stream: int) -> int:
    nnz = _i64(0)
    _check(h, load().kk_spgemm_symbolic(h, ctypes.byref(A), ctypes.byref(B), c_row_map_ptr or None,
                                        ctypes.byref(nnz), stream or None))
    return int(nnz.value)


def kk_spgemm_numeric(h, A: kk_csr_t, B: kk_csr_t, c_row_map_ptr: int, c_entries_ptr: int, c_values_ptr: int,
                      stream: int) -> None:
    _check(h, load().kk_spgemm_numeric(h, ctypes.byref(A), ctypes.byref(B), c_row_map_ptr or None,
                                       c_entries_ptr or None, c_values_ptr or None, stream or None))


def kk_spgemm_jacobi_numeric(h, omega: float, dinv_ptr: int, A: kk_csr_t, B: kk_csr_t, c_row_map_ptr: int,
                             c_entries_ptr: int, c_values_ptr: int, stream: int) -> None:
    _check(h, load().kk_spgemm_jacobi_numeric(h, float(omega), dinv_ptr or None, ctypes.byref(A), ctypes.byref(B),
                                              c_row_map_ptr or None, c_entries_ptr or None, c_values_ptr or None,
                                              stream or None))


def kk_spadd_symbolic(h, A: kk_csr_t, B: kk_csr_t, c_row_map_ptr: int, stream: int) -> int:
    nnz = _i64(0)
    _check(h, load().kk_spadd_symbolic(h, ctypes.byref(A), ctypes.byref(B), c_row_map_ptr, ctypes.byref(nnz),
                                       stream or None))
    return int(nnz.value)


def kk_spadd_numeric(h, alpha: float, A: kk_csr_t, beta: float, B: kk_csr_t, c_row_map_ptr: int,
                     c_entries_ptr: int, c_values_ptr: int, stream: int) -> None:
    _check(h, load().kk_spadd_numeric(h, float(alpha), ctypes.byref(A), float(beta), ctypes.byref(B),
                                      c_row_map_ptr or None, c_entries_ptr or None, c_values_ptr or None,
                                      stream or None))


def kk_spgemm_stats(h) -> dict:
    s = kk_spgemm_stats_t()
    _check(h, load().kk_spgemm_stats(h, ctypes.byref(s)))
    d = {f: getattr(s, f) for f, _ in kk_spgemm_stats_t._fields_}
    d["symbolic_bin_rows"] = list(s.symbolic_bin_rows)
    d["numeric_bin_rows"] = list(s.numeric_bin_rows)
    return d


def kk_spgemm_multiply_host(h, A: kk_csr_t, B: kk_csr_t, c_row_map_ptr: int, blocks: int, stream: int):
    """-> (nnz, entries address, values address): host arrays owned by the handle."""
    nnz = _i64(0)
    ent = ctypes.POINTER(ctypes.c_int32)()
    val = _vp()
    _check(h, load().kk_spgemm_multiply_host(h, ctypes.byref(A), ctypes.byref(B), c_row_map_ptr or None,
                                             ctypes.byref(nnz), ctypes.byref(ent), ctypes.byref(val), int(blocks),
                                             stream or None))
    return int(nnz.value), ctypes.cast(ent, _vp).value or 0, val.value or 0


def kk_spgemm_rap_symbolic(h, R: kk_csr_t, A: kk_csr_t, P: kk_csr_t, c_row_map_ptr: int, stream: int) -> int:
    nnz = _i64(0)
    _check(h, load().kk_spgemm_rap_symbolic(h, ctypes.byref(R), ctypes.byref(A), ctypes.byref(P),
                                            c_row_map_ptr or None, ctypes.byref(nnz), stream or None))
    return int(nnz.value)


def kk_spgemm_rap_numeric(h, R: kk_csr_t, A: kk_csr_t, P: kk_csr_t, c_row_map_ptr: int, c_entries_ptr: int,
                          c_values_ptr: int, stream: int) -> None:
    _check(h, load().kk_spgemm_rap_numeric(h, ctypes.byref(R), ctypes.byref(A), ctypes.byref(P),
                                           c_row_map_ptr or None, c_entries_ptr or None, c_values_ptr or None,
                                           stream or None))


def kk_spgemm_kernel_times(h) -> list:
    """[(name, launches, total_ms, max_ms)] accumulated since the last reset (opts.timing=1)."""
    n = ctypes.c_int(0)
    _check(h, load().kk_spgemm_kernel_times(h, None, ctypes.byref(n)))
    arr = (kk_kernel_time_t * max(n.value, 1))()
    n2 = ctypes.c_int(n.value)
    _check(h, load().kk_spgemm_kernel_times(h, arr, ctypes.byref(n2)))
    return [(arr[i].name.decode(), int(arr[i].launches), float(arr[i].total_ms), float(arr[i].max_ms))
            for i in range(min(n.value, n2.value))]


def kk_spgemm_timing_reset(h) -> None:
    _check(h, load().kk_spgemm_timing_reset(h))
