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


def _kk_csr(M: CsrMatrix, need_values: bool) -> _ffi.kk_csr_t:
    for name, t in (("row_map", M.row_map), ("entries", M.entries)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
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
        if not M.values.is_cuda or not M.values.is_contiguous() or M.values.dtype not in _VAL:
            raise TypeError("values must be a contiguous CUDA float32/float64 tensor")
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
                 num_streams: int = 2, timing: bool = False, patterns: bool = True):
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

    # -- end to end from host memory ------------------------------------------------------
    def multiply_host(self, A, B, stream=None, blocks: Optional[int] = None) -> "CsrMatrix":
        """C = A*B for CSR operands in (pinned) HOST memory, C returned in pinned HOST memory.

        B is copied to the device once; A is processed in `blocks` contiguous row blocks
        (default 8 when A has >= 64K rows): block b's host->device copy, its symbolic and
        numeric phases and the device->host copy of its rows of C run on three streams, so
        the copies of neighbouring blocks (both PCIe directions) overlap the kernels.  Row
        blocks are independent products (Eq. 1); the host assembles the
        global row map from the blocks' row maps and nnz.  Device and pinned staging buffers
        are cached on the handle.  The result is valid until the next call on this handle."""
        A, B = CsrMatrix.from_any(A), CsrMatrix.from_any(B)
        dev = self.device
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        cache = self.__dict__.setdefault("_host_cache", {})
        m = A.nrows
        if blocks is None:
            blocks = 8 if m >= 65536 else 1
        blocks = max(1, min(int(blocks), max(m, 1)))
        if "s_in" not in cache:
            cache["s_in"] = torch.cuda.Stream(dev)
            cache["s_out"] = torch.cuda.Stream(dev)
        s_in, s_out = cache["s_in"], cache["s_out"]

        def dbuf(key, n, dtype):
            t = cache.get(key)
            if t is None or t.numel() < n or t.dtype != dtype:
                t = torch.empty(max(n, 1), dtype=dtype, device=dev)
                cache[key] = t
            return t[:n]

        def hbuf(key, n, dtype):
            t = cache.get(key)
            if t is None or t.numel() < n or t.dtype != dtype:
                t = torch.empty(max(n, 1), dtype=dtype, pin_memory=True)
                cache[key] = t
            return t[:n]

        def h2d(key, t):
            d = dbuf(key, t.numel(), t.dtype)
            d.copy_(t, non_blocking=True)
            return d

        # B once (every block reads all of it)
        ev_b = torch.cuda.Event()
        with torch.cuda.stream(s_in):
            Bd = CsrMatrix(B.nrows, B.ncols, h2d("brm", B.row_map), h2d("bent", B.entries), h2d("bval", B.values))
            ev_b.record(s_in)
        # A's row blocks; their row maps rebased to 0 in a pinned staging buffer
        rm = A.row_map
        cuts = [m * q // blocks for q in range(blocks + 1)]
        reb = hbuf("a_rm_reb", m + blocks, rm.dtype)
        roffs = []
        for q in range(blocks):
            r0, r1 = cuts[q], cuts[q + 1]
            o = q + r0
            torch.sub(rm[r0:r1 + 1], rm[r0], out=reb[o:o + r1 - r0 + 1])
            roffs.append(o)
        ev_in = [torch.cuda.Event() for _ in range(blocks)]
        ev_c = [torch.cuda.Event() for _ in range(blocks)]
        ev_out = [torch.cuda.Event() for _ in range(blocks)]

        def load_block(q):
            r0, r1 = cuts[q], cuts[q + 1]
            e0, e1 = int(rm[r0]), int(rm[r1])
            sl = q % 2
            with torch.cuda.stream(s_in):
                if q >= 2:
                    s_in.wait_event(ev_c[q - 2])
                Ab = CsrMatrix(r1 - r0, A.ncols, h2d(f"arm{sl}", reb[roffs[q]:roffs[q] + r1 - r0 + 1]),
                               h2d(f"aent{sl}", A.entries[e0:e1]), h2d(f"aval{sl}", A.values[e0:e1]))
                ev_in[q].record(s_in)
            return Ab

        h_rm = hbuf("h_crm", m + 1, rm.dtype)
        pending = [load_block(q) for q in range(min(2, blocks))]
        nnz_off = [0] * (blocks + 1)
        for q in range(blocks):
            r0, r1 = cuts[q], cuts[q + 1]
            Ab = pending[q]
            sl = q % 2
            st.wait_event(ev_in[q])
            st.wait_event(ev_b)
            if q >= 2:
                st.wait_event(ev_out[q - 2])
            crm = dbuf(f"crm{sl}", r1 - r0 + 1, rm.dtype)
            crm, nnz = self.symbolic(Ab, Bd, c_row_map=crm, stream=st)
            cent = dbuf(f"cent{sl}", nnz, torch.int32)
            cval = dbuf(f"cval{sl}", nnz, A.values.dtype)
            self.numeric(Ab, Bd, crm, nnz=nnz, c_entries=cent, c_values=cval, stream=st)
            ev_c[q].record(st)
            nnz_off[q + 1] = nnz_off[q] + nnz
            # host output capacity (grows only on a first, larger call: earlier blocks are kept)
            for key, dt in (("h_cent", torch.int32), ("h_cval", A.values.dtype)):
                t = cache.get(key)
                if t is None or t.numel() < nnz_off[q + 1] or t.dtype != dt:
                    s_out.synchronize()
                    nt = torch.empty(max(int(nnz_off[q + 1] * 1.25), 1), dtype=dt, pin_memory=True)
                    if t is not None and t.dtype == dt and nnz_off[q]:
                        nt[:nnz_off[q]].copy_(t[:nnz_off[q]])
                    cache[key] = nt
            h_ent, h_val = cache["h_cent"], cache["h_cval"]
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_c[q])
                h_rm[r0:r1 + 1].copy_(crm, non_blocking=True)
                h_ent[nnz_off[q]:nnz_off[q + 1]].copy_(cent, non_blocking=True)
                h_val[nnz_off[q]:nnz_off[q + 1]].copy_(cval, non_blocking=True)
                ev_out[q].record(s_out)
            if q + 2 < blocks:
                pending.append(load_block(q + 2))
        s_out.synchronize()
        # global row map: block q's local offsets + the nnz of the blocks before it (block
        # q+1's copy overwrote the shared boundary entry with its local 0; restored here)
        for q in range(blocks):
            r0, r1 = cuts[q], cuts[q + 1]
            if nnz_off[q]:
                h_rm[r0 + 1:r1 + 1] += nnz_off[q]
            h_rm[r0] = nnz_off[q]
        h_rm[m] = nnz_off[blocks]
        tot = nnz_off[blocks]
        return CsrMatrix(m, B.ncols, h_rm, cache["h_cent"][:tot], cache["h_cval"][:tot])

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
