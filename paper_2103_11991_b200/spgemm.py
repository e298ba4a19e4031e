"""Python front end of the C ABI: torch tensors in, torch tensors out.

PyTorch supplies device memory and the current CUDA stream; every step of the
SpGEMM runs in libkk_spgemm.so (include/kk_spgemm.h).  There is no CPU path.

    A = CsrMatrix(m, n, row_map, entries, values)   # CUDA tensors
    C = spgemm(A, B)                                  # symbolic + numeric

or, following the paper's two-phase protocol:

    h = SpGEMM()
    c_row_map, nnz = h.symbolic(A, B)       # fills the row pointers; nnz(C) on host
    c_entries, c_values = h.numeric(A, B, c_row_map)
"""
from __future__ import annotations

import ctypes

from dataclasses import dataclass
from typing import Optional

import torch

from . import _ffi


@dataclass
class CsrMatrix:
    """CSR matrix on a CUDA device.  row_map: int32/int64 (nrows+1);
    entries: int32 column indices; values: float32/float64 (or None for patterns)."""

    nrows: int
    ncols: int
    row_map: torch.Tensor
    entries: torch.Tensor
    values: Optional[torch.Tensor] = None

    @property
    def nnz(self) -> int:
        return int(self.entries.numel())

    @staticmethod
    def from_any(M) -> "CsrMatrix":
        if isinstance(M, CsrMatrix):
            return M
        return CsrMatrix(int(M.nrows), int(M.ncols), M.row_map, M.entries, getattr(M, "values", None))


_OFF = {torch.int32: _ffi.KK_I32, torch.int64: _ffi.KK_I64}
_VAL = {torch.float32: _ffi.KK_F32, torch.float64: _ffi.KK_F64}


def _kk_csr(M: CsrMatrix, need_values: bool, host: bool = False) -> _ffi.kk_csr_t:
    """kk_csr_t of M: device tensors, or host tensors for kk_spgemm_multiply_host (host=True;
    the library copies them to the device -- there is no CPU compute path)."""
    for name, t in (("row_map", M.row_map), ("entries", M.entries)):
        if t.is_cuda == host:
            raise ValueError(f"{name} must be a {'host' if host else 'CUDA'} tensor")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    if M.row_map.dtype not in _OFF:
        raise TypeError("row_map must be int32 or int64")
    if M.entries.dtype != torch.int32:
        raise TypeError("entries must be int32")
    if M.row_map.numel() != M.nrows + 1:
        raise ValueError("row_map must have nrows+1 entries")
    c = _ffi.kk_csr_t()
    c.nrows, c.ncols, c.nnz = int(M.nrows), int(M.ncols), int(M.entries.numel())
    c.offset_type = _OFF[M.row_map.dtype]
    c.row_map = M.row_map.data_ptr()
    c.entries = M.entries.data_ptr() if M.entries.numel() else None
    if M.values is not None:
        if M.values.is_cuda == host or not M.values.is_contiguous() or M.values.dtype not in _VAL:
            raise TypeError(f"values must be a contiguous {'host' if host else 'CUDA'} float32/float64 tensor")
        c.value_type = _VAL[M.values.dtype]
        c.values = M.values.data_ptr() if M.values.numel() else None
    else:
        if need_values:
            raise ValueError("values are required for the numeric phase")
        c.value_type = _ffi.KK_F64
        c.values = None
    return c


def _stream_ptr(device, stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


class SpGEMM:
    """Kernel handle: options + the symbolic state reused by numeric."""

    def __init__(self, device=None, sort_rows: bool = True, compression="auto", validate: bool = False,
                 num_streams: int = 2, timing: bool = False, patterns: bool = True, deterministic: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2103_11991_b200 needs a CUDA device (there is no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        o = _ffi.kk_spgemm_opts_default()
        o.sort_rows = int(bool(sort_rows))
        o.compression = {"auto": -1, "off": 0, "on": 1, -1: -1, 0: 0, 1: 1, True: 1, False: 0}[compression]
        o.validate = int(bool(validate))
        o.num_streams = int(num_streams)
        o.timing = int(bool(timing))
        o.deterministic = int(bool(deterministic))
        o.patterns = int(bool(patterns))
        self._h = _ffi.kk_spgemm_create(self.device.index, o)

    # -- phases ------------------------------------------------------------------------
    def symbolic(self, A, B, c_row_map: Optional[torch.Tensor] = None, stream=None):
        """Fill C's row pointers; returns (c_row_map, nnz(C)).  Synchronises the stream once."""
        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        a, b = _kk_csr(A, False), _kk_csr(B, False)
        if c_row_map is None:
            c_row_map = torch.empty(A.nrows + 1, dtype=A.row_map.dtype, device=A.row_map.device)
        nnz = _ffi.kk_spgemm_symbolic(self._h, a, b, c_row_map.data_ptr(), _stream_ptr(self.device, stream))
        return c_row_map, nnz

    def numeric(self, A, B, c_row_map: torch.Tensor, nnz: Optional[int] = None,
                c_entries: Optional[torch.Tensor] = None, c_values: Optional[torch.Tensor] = None, stream=None):
        """Column indices and values of C (asynchronous on the stream)."""
        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        a, b = _kk_csr(A, True), _kk_csr(B, True)
        if nnz is None:
            nnz = self.stats()["nnz_c"]
        if c_entries is None:
            c_entries = torch.empty(nnz, dtype=torch.int32, device=A.row_map.device)
        if c_values is None:
            c_values = torch.empty(nnz, dtype=A.values.dtype, device=A.row_map.device)
        _ffi.kk_spgemm_numeric(self._h, a, b, c_row_map.data_ptr(), c_entries.data_ptr() if nnz else 0,
                               c_values.data_ptr() if nnz else 0, _stream_ptr(self.device, stream))
        return c_entries, c_values

    def jacobi_numeric(self, omega: float, dinv: torch.Tensor, A, B, c_row_map: torch.Tensor,
                       nnz: Optional[int] = None, c_entries: Optional[torch.Tensor] = None,
                       c_values: Optional[torch.Tensor] = None, stream=None):
        """Jacobi-fused numeric C = (I - omega D^-1 A) B after
        symbolic(A, B); dinv: device vector of D^-1 (A's value dtype)."""
        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        a, b = _kk_csr(A, True), _kk_csr(B, True)
        if nnz is None:
            nnz = self.stats()["nnz_c"]
        if dinv.dtype != A.values.dtype or dinv.device != A.values.device or not dinv.is_contiguous():
            raise ValueError("dinv must be a contiguous device vector of A's value dtype")
        if c_entries is None:
            c_entries = torch.empty(nnz, dtype=torch.int32, device=A.row_map.device)
        if c_values is None:
            c_values = torch.empty(nnz, dtype=A.values.dtype, device=A.row_map.device)
        _ffi.kk_spgemm_jacobi_numeric(self._h, omega, dinv.data_ptr() if A.nrows else 0, a, b, c_row_map.data_ptr(),
                                      c_entries.data_ptr() if nnz else 0, c_values.data_ptr() if nnz else 0,
                                      _stream_ptr(self.device, stream))
        return c_entries, c_values

    def jacobi(self, omega: float, dinv: torch.Tensor, A, B, stream=None) -> CsrMatrix:
        """Both phases of the Jacobi-fused product (usual symbolic, fused numeric)."""
        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        rm, nnz = self.symbolic(A, B, stream=stream)
        ent, val = self.jacobi_numeric(omega, dinv, A, B, rm, nnz=nnz, stream=stream)
        return CsrMatrix(A.nrows, B.ncols, rm, ent, val)

    # -- SpAdd ---------------------------------------------------------
    def spadd_symbolic(self, A, B, c_row_map: Optional[torch.Tensor] = None, stream=None):
        """Row pointers of C = alpha A + beta B and nnz(C); keeps the scatter positions."""
        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        a, b = _kk_csr(A, False), _kk_csr(B, False)
        if c_row_map is None:
            c_row_map = torch.empty(A.nrows + 1, dtype=A.row_map.dtype, device=A.row_map.device)
        nnz = _ffi.kk_spadd_symbolic(self._h, a, b, c_row_map.data_ptr(), _stream_ptr(self.device, stream))
        return c_row_map, nnz

    def spadd_numeric(self, alpha: float, A, beta: float, B, c_row_map: torch.Tensor, nnz: int,
                      c_entries: Optional[torch.Tensor] = None, c_values: Optional[torch.Tensor] = None, stream=None):
        """Sorted columns and values alpha*a + beta*b of C (asynchronous)."""
        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        a, b = _kk_csr(A, True), _kk_csr(B, True)
        if c_entries is None:
            c_entries = torch.empty(nnz, dtype=torch.int32, device=A.row_map.device)
        if c_values is None:
            c_values = torch.empty(nnz, dtype=A.values.dtype, device=A.row_map.device)
        _ffi.kk_spadd_numeric(self._h, alpha, a, beta, b, c_row_map.data_ptr(), c_entries.data_ptr() if nnz else 0,
                              c_values.data_ptr() if nnz else 0, _stream_ptr(self.device, stream))
        return c_entries, c_values

    def spadd(self, alpha: float, A, beta: float, B, stream=None) -> CsrMatrix:
        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        rm, nnz = self.spadd_symbolic(A, B, stream=stream)
        ent, val = self.spadd_numeric(alpha, A, beta, B, rm, nnz, stream=stream)
        return CsrMatrix(A.nrows, A.ncols, rm, ent, val)

    def __call__(self, A, B, stream=None) -> CsrMatrix:
        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        rm, nnz = self.symbolic(A, B, stream=stream)
        ent, val = self.numeric(A, B, rm, nnz=nnz, stream=stream)
        return CsrMatrix(A.nrows, B.ncols, rm, ent, val)

    # -- fused Galerkin triple product (NEXT-4) --------------------------------------------
    def rap_symbolic(self, R, A, P, c_row_map: Optional[torch.Tensor] = None, stream=None):
        """Row map and nnz of Ac = R*A*P (one pass, A*P never formed)."""
        R, A, P = (CsrMatrix.from_any(M) for M in (R, A, P))
        if c_row_map is None:
            c_row_map = torch.empty(R.nrows + 1, dtype=R.row_map.dtype, device=R.row_map.device)
        nnz = _ffi.kk_spgemm_rap_symbolic(self._h, _kk_csr(R, False), _kk_csr(A, False), _kk_csr(P, False),
                                          c_row_map.data_ptr(), _stream_ptr(self.device, stream))
        return c_row_map, nnz

    def rap_numeric(self, R, A, P, c_row_map: torch.Tensor, nnz: int, c_entries: Optional[torch.Tensor] = None,
                    c_values: Optional[torch.Tensor] = None, stream=None):
        R, A, P = (CsrMatrix.from_any(M) for M in (R, A, P))
        dev = R.row_map.device
        if c_entries is None:
            c_entries = torch.empty(nnz, dtype=torch.int32, device=dev)
        if c_values is None:
            c_values = torch.empty(nnz, dtype=R.values.dtype, device=dev)
        _ffi.kk_spgemm_rap_numeric(self._h, _kk_csr(R, True), _kk_csr(A, True), _kk_csr(P, True),
                                   c_row_map.data_ptr(), c_entries.data_ptr() if nnz else 0,
                                   c_values.data_ptr() if nnz else 0, _stream_ptr(self.device, stream))
        return c_entries, c_values

    def rap(self, R, A, P, stream=None) -> CsrMatrix:
        """Ac = R*A*P, fused (kk_spgemm_rap_symbolic + kk_spgemm_rap_numeric)."""
        rm, nnz = self.rap_symbolic(R, A, P, stream=stream)
        ent, val = self.rap_numeric(R, A, P, rm, nnz, stream=stream)
        R = CsrMatrix.from_any(R)
        return CsrMatrix(R.nrows, CsrMatrix.from_any(P).ncols, rm, ent, val)

    # -- end to end from host memory ------------------------------------------------------
    def multiply_host(self, A, B, stream=None, blocks: Optional[int] = None) -> "CsrMatrix":
        """C = A*B for CSR operands in (pinned) HOST memory, C returned in HOST memory, through
        the C ABI's kk_spgemm_multiply_host (B copied once in row chunks; A in row blocks whose
        copies in both PCIe directions overlap the kernels -- `blocks` fixes their number, None
        plans them from the first block's output; pass the same matrix twice for A*A and it
        crosses PCIe once; the global row map assembled in the library).  C's entries and
        values are the handle's pinned buffers: valid until the next call on this handle (copy
        them to keep them)."""
        import numpy as np

        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        a, b = _kk_csr(A, True, host=True), _kk_csr(B, True, host=True)
        cache = self.__dict__.setdefault("_host_cache", {})
        rm = cache.get("h_crm")
        if rm is None or rm.numel() < A.nrows + 1 or rm.dtype != A.row_map.dtype:
            rm = torch.empty(A.nrows + 1, dtype=A.row_map.dtype, pin_memory=True)
            cache["h_crm"] = rm
        rm = rm[:A.nrows + 1]
        nnz, pe, pv = _ffi.kk_spgemm_multiply_host(self._h, a, b, rm.data_ptr(), blocks or 0,
                                                   _stream_ptr(self.device, stream))
        vt = np.float64 if A.values.dtype == torch.float64 else np.float32
        if nnz:
            ent = torch.from_numpy(np.ctypeslib.as_array((ctypes.c_int32 * nnz).from_address(pe)))
            val = torch.from_numpy(np.frombuffer((ctypes.c_char * (nnz * np.dtype(vt).itemsize)).from_address(pv),
                                                 dtype=vt))
        else:
            ent = torch.zeros(0, dtype=torch.int32)
            val = torch.zeros(0, dtype=A.values.dtype)
        return CsrMatrix(A.nrows, B.ncols, rm, ent, val)

    # -- individual steps ----------------------------------------------------------------
    def row_flops(self, A, B, scan: bool = True, total: bool = True, stream=None):
        """a1+a2: per-row multiply-adds, their exclusive scan, and the total."""
        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        a, b = _kk_csr(A, False), _kk_csr(B, False)
        dev = A.row_map.device
        f = torch.empty(A.nrows, dtype=torch.int64, device=dev)
        F = torch.empty(A.nrows + 1, dtype=torch.int64, device=dev) if scan else None
        tot = _ffi.kk_spgemm_row_flops(self._h, a, b, f.data_ptr() if A.nrows else 0,
                                       F.data_ptr() if F is not None else 0, total,
                                       _stream_ptr(self.device, stream))
        return f, F, tot

    def compress(self, B, stream=None):
        """a4: B -> B_C; returns (len[n] int32, words[nnzB] int32, masks[nnzB] int32) with the
        pairs of row j at B.row_map[j] .. + len[j]."""
        B = CsrMatrix.from_any(B)
        b = _kk_csr(B, False)
        dev = B.row_map.device
        ln = torch.zeros(max(B.nrows, 1), dtype=torch.int32, device=dev)
        pairs = torch.zeros(max(B.nnz, 1), 2, dtype=torch.int32, device=dev)
        _ffi.kk_spgemm_compress(self._h, b, ln.data_ptr() if B.nrows else 0, pairs.data_ptr() if B.nnz else 0,
                                _stream_ptr(self.device, stream))
        return ln[:B.nrows], pairs[:B.nnz, 0], pairs[:B.nnz, 1]

    def kernel_times(self) -> list:
        """Per-kernel CUDA-event times since the last reset (needs timing=True)."""
        return _ffi.kk_spgemm_kernel_times(self._h)

    def timing_reset(self) -> None:
        _ffi.kk_spgemm_timing_reset(self._h)

    def stats(self) -> dict:
        return _ffi.kk_spgemm_stats(self._h)

    def close(self):
        if getattr(self, "_h", None):
            _ffi.kk_spgemm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def spgemm(A, B, **opts) -> CsrMatrix:
    """C = A*B (both phases) with a temporary handle."""
    h = SpGEMM(**opts)
    try:
        return h(A, B)
    finally:
        torch.cuda.current_stream(h.device).synchronize()
        h.close()


def spgemm_jacobi(omega: float, dinv: torch.Tensor, A, B, **opts) -> CsrMatrix:
    """One-shot Jacobi-fused product C = (I - omega D^-1 A) B on the device
    (PAPER.md:188-217): usual symbolic, fused numeric."""
    h = SpGEMM(**opts)
    try:
        return h.jacobi(omega, dinv, A, B)
    finally:
        torch.cuda.current_stream(h.device).synchronize()
        h.close()


def spadd(alpha: float, A, beta: float, B, **opts) -> CsrMatrix:
    """One-shot SpAdd C = alpha A + beta B on the device."""
    h = SpGEMM(**opts)
    try:
        return h.spadd(alpha, A, beta, B)
    finally:
        torch.cuda.current_stream(h.device).synchronize()
        h.close()
