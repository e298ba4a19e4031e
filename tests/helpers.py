"""Test helpers: run the CUDA path through the C ABI and compare with the oracle.

Tolerance (north star): |c_gpu - c_ref| <= tau * sum|a||b| with
tau = 1e-12 (fp64) / 1e-5 (fp32); row maps and sorted column indices bit-exact.
"""
from __future__ import annotations

import numpy as np
import torch

from workloads import generators as g

TAU = {torch.float64: 1e-12, torch.float32: 1e-5}


def to_device(M, device="cuda", value_dtype=torch.float64, offset_dtype=torch.int64):
    return M.to(device=device, value_dtype=value_dtype, offset_dtype=offset_dtype)


def gpu_spgemm(A, B, value_dtype=torch.float64, offset_dtype=torch.int64, **opts):
    """C = A*B on cuda:0 through paper_2103_11991_b200 (C ABI). Returns numpy arrays + stats."""
    from paper_2103_11991_b200 import SpGEMM

    Ad, Bd = to_device(A, "cuda", value_dtype, offset_dtype), to_device(B, "cuda", value_dtype, offset_dtype)
    h = SpGEMM(**opts)
    rm, nnz = h.symbolic(Ad, Bd)
    ent, val = h.numeric(Ad, Bd, rm, nnz=nnz)
    torch.cuda.synchronize()
    st = h.stats()
    if opts.get("timing"):
        st["kernels"] = [k[0] for k in h.kernel_times()]
    h.close()
    return rm.cpu().numpy().astype(np.int64), ent.cpu().numpy(), val.cpu().to(torch.float64).numpy(), st


def sample_rows(A: g.CSR, rows) -> g.CSR:
    """CSR with A's rows `rows` kept and all other rows empty (same shape)."""
    rows = torch.as_tensor(np.sort(np.unique(np.asarray(rows))), dtype=torch.int64)
    rm = A.row_map.to(torch.int64).cpu()
    lens = torch.zeros(A.nrows, dtype=torch.int64)
    lens[rows] = rm[rows + 1] - rm[rows]
    nrm = torch.zeros(A.nrows + 1, dtype=torch.int64)
    nrm[1:] = torch.cumsum(lens, 0)
    idx = torch.cat([torch.arange(int(rm[r]), int(rm[r + 1])) for r in rows.tolist()]) if len(rows) else \
        torch.zeros(0, dtype=torch.int64)
    return g.CSR(A.nrows, A.ncols, nrm, A.entries.cpu()[idx], A.values.cpu()[idx])


def assert_parity(oracle_mod, A, B, got, value_dtype=torch.float64, rows=None, exact=False, sorted_rows=True):
    """Compare (row_map, entries, values) from the GPU with the oracle.

    rows=None: whole matrix; else only the listed rows (oracle on a row sample)."""
    grm, gent, gval = got[0], got[1], got[2]
    if rows is None:
        orm, oent, oval, obnd = oracle_mod.spgemm(A, B)
        assert np.array_equal(grm, orm), "row map differs"
        check_rows = range(A.nrows)
        o_off = orm
    else:
        As = sample_rows(A, rows)
        orm, oent, oval, obnd = oracle_mod.spgemm(As, B)
        check_rows = sorted(set(int(r) for r in rows))
        o_off = orm
        for r in check_rows:
            assert grm[r + 1] - grm[r] == orm[r + 1] - orm[r], f"row {r}: nnz differs"
    tau = TAU[value_dtype]
    worst = 0.0
    if rows is None and sorted_rows:
        assert np.array_equal(gent, oent), "column indices differ"
        diff = np.abs(gval - oval)
        if exact:
            assert np.array_equal(gval, oval), "values differ (integer-valued config must be exact)"
        ok = diff <= tau * obnd
        assert ok.all(), f"{(~ok).sum()} values out of tolerance; worst {np.max(diff - tau * obnd)}"
        nz = obnd > 0
        worst = float(np.max(diff[nz] / obnd[nz])) if nz.any() else 0.0
        return worst
    for r in check_rows:
        g0, g1 = grm[r], grm[r + 1]
        o0, o1 = o_off[r], o_off[r + 1]
        ge, gv = gent[g0:g1], gval[g0:g1]
        if not sorted_rows:
            order = np.argsort(ge, kind="stable")
            ge, gv = ge[order], gv[order]
        assert np.array_equal(ge, oent[o0:o1]), f"row {r}: columns differ"
        diff = np.abs(gv - oval[o0:o1])
        if exact:
            assert np.array_equal(gv, oval[o0:o1]), f"row {r}: values differ"
        bnd = obnd[o0:o1]
        assert (diff <= tau * bnd).all(), f"row {r}: value out of tolerance"
        nz = bnd > 0
        if nz.any():
            worst = max(worst, float(np.max(diff[nz] / bnd[nz])))
    return worst
