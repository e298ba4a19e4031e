"""SpAdd C = alpha A + beta B on the GPU (Sec. 2.3) against the oracle
(oracle.spadd): row map and sorted columns bit-exact; values within tau * (|alpha| sum|a| +
|beta| sum|b|) (two roundings per term at most, so tau = 1e-12 / 1e-5 is generous)."""
import numpy as np
import pytest
import torch

from workloads import generators as g

from .helpers import TAU, to_device

pytestmark = pytest.mark.gpu


def _run(alpha, A, beta, B, vt=torch.float64, ot=torch.int64):
    from paper_2103_11991_b200 import SpGEMM

    Ad, Bd = to_device(A, "cuda", vt, ot), to_device(B, "cuda", vt, ot)
    h = SpGEMM()
    C = h.spadd(alpha, Ad, beta, Bd)
    torch.cuda.synchronize()
    h.close()
    return C.row_map.cpu().numpy().astype(np.int64), C.entries.cpu().numpy(), C.values.cpu().double().numpy()


def _check(oracle_mod, alpha, A, beta, B, got, vt=torch.float64):
    rm, ent, val = got
    orm, oent, oval, obnd = oracle_mod.spadd(alpha, A, beta, B)
    assert np.array_equal(rm, orm), "row map"
    assert np.array_equal(ent, oent), "columns"
    bad = np.abs(val - oval) > TAU[vt] * obnd
    assert not bad.any(), f"{bad.sum()} values outside tolerance"


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("ma,mb", [(6, 9), (20, 30), (40, 60), (100, 120)])
@pytest.mark.parametrize("kw", [{}, dict(sorted_rows=False), dict(duplicates=True, sorted_rows=False)])
@pytest.mark.parametrize("vt,ot", [(torch.float64, torch.int64), (torch.float32, torch.int32)])
def test_spadd_random(oracle_mod, seed, ma, mb, kw, vt, ot):
    """Rows of every sort-width class (<= 32, 64, 128, 256 keys), sorted, unsorted and
    unmerged inputs, empty rows."""
    m, k = 300, 500
    A = g.random_csr(m, k, ma, seed=seed, **kw)
    B = g.random_csr(m, k, mb, seed=seed + 40, **kw)
    _check(oracle_mod, 0.5, A, -2.0, B, _run(0.5, A, -2.0, B, vt, ot), vt)


def test_spadd_paper_workload(oracle_mod):
    """The paper's SpAdd test shape: square, 30 random entries per row."""
    m = 20000
    A = g.random_csr(m, m, 30, seed=3, empty_row_frac=0.0)
    B = g.random_csr(m, m, 30, seed=4, empty_row_frac=0.0)
    _check(oracle_mod, 1.0, A, 1.0, B, _run(1.0, A, 1.0, B))


def test_spadd_symbolic_reuse_and_errors(oracle_mod):
    from paper_2103_11991_b200 import SpGEMM
    from paper_2103_11991_b200._ffi import KKError

    A = g.random_csr(200, 150, 12, seed=5)
    B = g.random_csr(200, 150, 12, seed=6)
    Ad, Bd = to_device(A, "cuda"), to_device(B, "cuda")
    h = SpGEMM()
    rm, nnz = h.spadd_symbolic(Ad, Bd)
    for al, be in ((1.0, 1.0), (3.0, -0.25)):  # numeric reuse with new scalars (same patterns)
        ent, val = h.spadd_numeric(al, Ad, be, Bd, rm, nnz)
        torch.cuda.synchronize()
        _check(oracle_mod, al, A, be, B, (rm.cpu().numpy().astype(np.int64), ent.cpu().numpy(), val.cpu().numpy()))
    with pytest.raises(KKError):  # shape mismatch
        h.spadd_symbolic(Ad, to_device(g.random_csr(200, 151, 3, seed=7), "cuda"))
    with pytest.raises(KKError):  # a row over the CTA tier's 16,384-key sort
        n = 9000  # one row of 9,000 entries: A + A has 18,000 keys
        row = g.CSR(1, 40000, torch.tensor([0, n]), torch.arange(0, 4 * n, 4, dtype=torch.int32),
                    torch.ones(n, dtype=torch.float64))
        L = to_device(row, "cuda")
        h.spadd_symbolic(L, L)
    h.close()


@pytest.mark.parametrize("kw", [{}, dict(sorted_rows=False), dict(sorted_rows=False, duplicates=True)])
@pytest.mark.parametrize("vt", [torch.float64, torch.float32])
def test_spadd_long_rows(oracle_mod, kw, vt):
    """Rows with nnz(A_i) + nnz(B_i) > 256 (the CTA tier: shared-memory bitonic sort), mixed
    with short rows (warp tier), sorted, unsorted and unmerged."""
    A = g.random_csr(60, 30000, 3000, seed=61, **kw)
    B = g.random_csr(60, 30000, 5000, seed=62, **kw)
    got = _run(0.75, A, -1.5, B, vt=vt)
    _check(oracle_mod, 0.75, A, -1.5, B, got, vt=vt)
