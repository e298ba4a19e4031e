"""Plain CPU oracle for two-phase SpGEMM (ctypes binding of oracle/kk_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs are the only callers.  The product package
(paper_2103_11991_b200/) never imports this module and shares no code with it.

Each function names the passage of /root/reference/PAPER.md it follows; the C
source header lists the readings taken where the paper is silent.  Pins for every
function live in tests/test_oracle.py (brute force, closed forms, SPEC.md worked
examples, invariants).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kk_oracle.c")
_LIB = os.path.join(_HERE, "libkk_oracle.so")
_lock = threading.Lock()
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_f64p = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile the oracle: gcc -O2 -ffp-contract=off -fopenmp (R5: no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            lib.kko_row_flops.restype = ctypes.c_int64
            lib.kko_row_flops.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i32p, _i64p, _i64p]
            lib.kko_compress.restype = ctypes.c_int
            lib.kko_compress.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i32p, _i64p, _i32p, _u32p]
            lib.kko_symbolic.restype = ctypes.c_int
            lib.kko_symbolic.argtypes = [ctypes.c_int64] * 3 + [_i64p, _i32p, _i64p, _i32p, _i64p]
            lib.kko_numeric.restype = ctypes.c_int
            lib.kko_numeric.argtypes = [ctypes.c_int64] * 3 + [_i64p, _i32p, _f64p, _i64p, _i32p, _f64p, _i64p,
                                                               _i32p, _f64p, _f64p]
            lib.kko_jacobi_counts.restype = ctypes.c_int
            lib.kko_jacobi_counts.argtypes = [ctypes.c_int64] * 2 + [_i64p, _i32p, _i64p, _i32p, _i64p]
            lib.kko_jacobi_fill.restype = ctypes.c_int
            lib.kko_jacobi_fill.argtypes = [ctypes.c_int64] * 2 + [_i64p, _i32p, _f64p, _i64p, _i32p, _f64p,
                                                                   ctypes.c_double, _f64p, _i64p, _i32p, _f64p,
                                                                   _f64p]
            lib.kko_spadd_counts.restype = ctypes.c_int
            lib.kko_spadd_counts.argtypes = [ctypes.c_int64] * 2 + [_i64p, _i32p, _i64p, _i32p, _i64p]
            lib.kko_spadd_fill.restype = ctypes.c_int
            lib.kko_spadd_fill.argtypes = [ctypes.c_int64] * 2 + [_i64p, _i32p, _f64p, _i64p, _i32p, _f64p,
                                                                  ctypes.c_double, ctypes.c_double, _i64p, _i32p,
                                                                  _f64p, _f64p]
            lib.kko_num_threads.restype = ctypes.c_int
            lib.kko_set_num_threads.argtypes = [ctypes.c_int]
            _lib = lib
    return _lib


def _np(x, dtype):
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(x), dtype=dtype)


def _p(a, t):
    return a.ctypes.data_as(t)


def _csr(M):
    return (int(M.nrows), int(M.ncols), _np(M.row_map, np.int64), _np(M.entries, np.int32),
            _np(M.values, np.float64))


def num_threads() -> int:
    return int(_load().kko_num_threads())


def set_num_threads(t: int) -> None:
    _load().kko_set_num_threads(int(t))


def row_flops(A, B):
    """flops_i = sum_{j in A(i,:)} nnz(B(j,:)). Returns (flops[m], total)."""
    lib = _load()
    m, n, arm, aent, _ = _csr(A)
    brm = _np(B.row_map, np.int64)
    out = np.zeros(m, dtype=np.int64)
    tot = lib.kko_row_flops(m, n, _p(arm, _i64p), _p(aent, _i32p), _p(brm, _i64p), _p(out, _i64p))
    if tot < 0:
        raise ValueError("oracle row_flops: column index out of range")
    return out, int(tot)


def compress(B):
    """B -> B_C: per row, sorted distinct (col//32, OR of bits). Returns
    (bc_row_map[n+1], words[], masks[])."""
    lib = _load()
    n, k, brm, bent, _ = _csr(B)
    rm = np.zeros(n + 1, dtype=np.int64)
    w = np.zeros(max(len(bent), 1), dtype=np.int32)
    mk = np.zeros(max(len(bent), 1), dtype=np.uint32)
    if lib.kko_compress(n, k, _p(brm, _i64p), _p(bent, _i32p), _p(rm, _i64p), _p(w, _i32p), _p(mk, _u32p)) != 0:
        raise ValueError("oracle compress: bad input")
    return rm, w[: rm[-1]], mk[: rm[-1]]


def symbolic(A, B):
    """Row pointers of C: exclusive prefix of distinct-column counts."""
    lib = _load()
    m, n, arm, aent, _ = _csr(A)
    nb, k, brm, bent, _ = _csr(B)
    if n != nb:
        raise ValueError("dimension mismatch")
    out = np.zeros(m + 1, dtype=np.int64)
    if lib.kko_symbolic(m, n, k, _p(arm, _i64p), _p(aent, _i32p), _p(brm, _i64p), _p(bent, _i32p),
                        _p(out, _i64p)) != 0:
        raise ValueError("oracle symbolic: bad input")
    return out


def numeric(A, B, c_row_map):
    """Columns (sorted) and fp64 values of C = A*B (Eq. 1), plus the
    per-entry bound sum |a||b| used by the tolerance."""
    lib = _load()
    m, n, arm, aent, aval = _csr(A)
    nb, k, brm, bent, bval = _csr(B)
    crm = _np(c_row_map, np.int64)
    nnz = int(crm[-1])
    ent = np.zeros(max(nnz, 1), dtype=np.int32)
    val = np.zeros(max(nnz, 1), dtype=np.float64)
    bnd = np.zeros(max(nnz, 1), dtype=np.float64)
    rc = lib.kko_numeric(m, n, k, _p(arm, _i64p), _p(aent, _i32p), _p(aval, _f64p), _p(brm, _i64p),
                         _p(bent, _i32p), _p(bval, _f64p), _p(crm, _i64p), _p(ent, _i32p), _p(val, _f64p),
                         _p(bnd, _f64p))
    if rc != 0:
        raise ValueError("oracle numeric: bad input or row map inconsistent with A*B")
    return ent[:nnz], val[:nnz], bnd[:nnz]


def spgemm(A, B):
    """Both phases: returns (row_map[int64], entries[int32], values[f64], bound[f64])."""
    rm = symbolic(A, B)
    ent, val, bnd = numeric(A, B, rm)
    return rm, ent, val, bnd


def jacobi(omega, dinv, A, B):
    """Jacobi-fused SpGEMM reference C = (I - omega D^-1 A) B (Sec. 2.2.2),
    written as the paper's three-kernel composition E = AB, F = D^-1 E, C = B - omega F
    (MSAK), row by row.  A is m x m, B is m x k, dinv has m entries.
    Returns (row_map[int64], entries[int32], values[f64], bound[f64]) with
    bound = |b| + |omega| |dinv_i| sum |a||b|; C's pattern = pattern(B) U pattern(E)."""
    lib = _load()
    m, n, arm, aent, aval = _csr(A)
    nb, k, brm, bent, bval = _csr(B)
    if n != m or nb != m:
        raise ValueError("Jacobi SpGEMM needs A m x m and B m x k")
    d = _np(dinv, np.float64)
    if len(d) != m:
        raise ValueError("dinv must have m entries")
    counts = np.zeros(max(m, 1), dtype=np.int64)
    if lib.kko_jacobi_counts(m, k, _p(arm, _i64p), _p(aent, _i32p), _p(brm, _i64p), _p(bent, _i32p),
                             _p(counts, _i64p)) != 0:
        raise ValueError("oracle jacobi: bad input")
    rm = np.zeros(m + 1, dtype=np.int64)
    rm[1:] = np.cumsum(counts[:m])
    nnz = int(rm[-1])
    ent = np.zeros(max(nnz, 1), dtype=np.int32)
    val = np.zeros(max(nnz, 1), dtype=np.float64)
    bnd = np.zeros(max(nnz, 1), dtype=np.float64)
    if lib.kko_jacobi_fill(m, k, _p(arm, _i64p), _p(aent, _i32p), _p(aval, _f64p), _p(brm, _i64p),
                           _p(bent, _i32p), _p(bval, _f64p), float(omega), _p(d, _f64p), _p(rm, _i64p),
                           _p(ent, _i32p), _p(val, _f64p), _p(bnd, _f64p)) != 0:
        raise ValueError("oracle jacobi: bad input")
    return rm, ent[:nnz], val[:nnz], bnd[:nnz]


def spadd(alpha, A, beta, B):
    """SpAdd reference C = alpha A + beta B (Sec. 2.3): entries of equal
    (row, column) merged, duplicates inside A or B included; rows sorted; structural pattern.
    Returns (row_map[int64], entries[int32], values[f64], bound[f64]) with
    bound = |alpha| sum|a| + |beta| sum|b|."""
    lib = _load()
    m, k, arm, aent, aval = _csr(A)
    mb, kb, brm, bent, bval = _csr(B)
    if m != mb or k != kb:
        raise ValueError("SpAdd needs A and B of the same shape")
    counts = np.zeros(max(m, 1), dtype=np.int64)
    if lib.kko_spadd_counts(m, k, _p(arm, _i64p), _p(aent, _i32p), _p(brm, _i64p), _p(bent, _i32p),
                            _p(counts, _i64p)) != 0:
        raise ValueError("oracle spadd: bad input")
    rm = np.zeros(m + 1, dtype=np.int64)
    rm[1:] = np.cumsum(counts[:m])
    nnz = int(rm[-1])
    ent = np.zeros(max(nnz, 1), dtype=np.int32)
    val = np.zeros(max(nnz, 1), dtype=np.float64)
    bnd = np.zeros(max(nnz, 1), dtype=np.float64)
    if lib.kko_spadd_fill(m, k, _p(arm, _i64p), _p(aent, _i32p), _p(aval, _f64p), _p(brm, _i64p), _p(bent, _i32p),
                          _p(bval, _f64p), float(alpha), float(beta), _p(rm, _i64p), _p(ent, _i32p),
                          _p(val, _f64p), _p(bnd, _f64p)) != 0:
        raise ValueError("oracle spadd: bad input")
    return rm, ent[:nnz], val[:nnz], bnd[:nnz]
