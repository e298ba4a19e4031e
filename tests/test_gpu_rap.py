"""Fused Galerkin triple product Ac = R*A*P (NEXT-4) on the GPU against the
oracle's two products R*(A*P): row map and sorted columns bit-exact; values exact on integer
data (C3) and within tau * sum|r||a||p| otherwise (the bound from the oracle's
product of the absolute matrices)."""
import numpy as np
import pytest
import torch

from workloads import generators as g

from .helpers import TAU, to_device

pytestmark = pytest.mark.gpu


def _oracle_rap(oracle_mod, R, A, P):
    orm, oent, oval, _ = oracle_mod.spgemm(A, P)
    T = g.CSR(A.nrows, P.ncols, torch.tensor(orm), torch.tensor(oent), torch.tensor(oval))
    crm, cent, cval, _ = oracle_mod.spgemm(R, T)

    def absm(M):
        return g.CSR(M.nrows, M.ncols, M.row_map, M.entries, M.values.abs())

    arm, aent, aval, _ = oracle_mod.spgemm(absm(A), absm(P))
    Ta = g.CSR(A.nrows, P.ncols, torch.tensor(arm), torch.tensor(aent), torch.tensor(aval))
    _, _, bnd, _ = oracle_mod.spgemm(absm(R), Ta)
    return crm, cent, cval, bnd


def _gpu_rap(R, A, P, vt=torch.float64, ot=torch.int64):
    from paper_2103_11991_b200 import SpGEMM

    Rd, Ad, Pd = (to_device(M, "cuda", vt, ot) for M in (R, A, P))
    h = SpGEMM()
    C = h.rap(Rd, Ad, Pd)
    torch.cuda.synchronize()
    h.close()
    return C.row_map.cpu().numpy().astype(np.int64), C.entries.cpu().numpy(), C.values.cpu().double().numpy()


@pytest.mark.parametrize("n", [12, 33])
@pytest.mark.parametrize("ot", [torch.int32, torch.int64])
def test_rap_galerkin_exact(oracle_mod, n, ot):
    A, P, R = g.config("C3", size=n)
    got = _gpu_rap(R, A, P, ot=ot)
    crm, cent, cval, _ = _oracle_rap(oracle_mod, R, A, P)
    assert np.array_equal(got[0], crm) and np.array_equal(got[1], cent)
    assert np.array_equal(got[2], cval), "integer-valued Galerkin product must be exact"


@pytest.mark.parametrize("vt", [torch.float64, torch.float32])
@pytest.mark.parametrize("case", range(4))
def test_rap_random(oracle_mod, vt, case):
    cases = [(30, 50, 40, 20, 6, 5, 3), (80, 200, 150, 60, 20, 8, 6), (5, 9, 7, 3, 4, 4, 4), (40, 300, 300, 200, 12, 10, 10)]
    mc, m, n, nc, mr, ma, mp = cases[case]
    R = g.random_csr(mc, m, mr, seed=10 + case)
    A = g.random_csr(m, n, ma, seed=20 + case, sorted_rows=(case % 2 == 0), duplicates=(case == 3))
    P = g.random_csr(n, nc, mp, seed=30 + case)
    got = _gpu_rap(R, A, P, vt=vt)
    crm, cent, cval, bnd = _oracle_rap(oracle_mod, R, A, P)
    assert np.array_equal(got[0], crm) and np.array_equal(got[1], cent)
    assert np.all(np.abs(got[2] - cval) <= TAU[vt] * bnd)


def test_rap_errors():
    from paper_2103_11991_b200 import SpGEMM
    from paper_2103_11991_b200._ffi import KKError, KK_ERR_DIM_MISMATCH, KK_ERR_STALE_HANDLE, KK_ERR_UNSUPPORTED_TYPE

    h = SpGEMM()
    R = to_device(g.random_csr(10, 20, 3, seed=1))
    A = to_device(g.random_csr(20, 30, 3, seed=2))
    P = to_device(g.random_csr(31, 5, 3, seed=3))
    with pytest.raises(KKError) as e:
        h.rap(R, A, P)
    assert e.value.status == KK_ERR_DIM_MISMATCH
    P = to_device(g.random_csr(30, 5, 3, seed=3))
    rm, nnz = h.rap_symbolic(R, A, P)
    with pytest.raises(KKError) as e:
        h.rap_numeric(R, to_device(g.random_csr(20, 30, 3, seed=4)), P, rm, nnz)
    assert e.value.status == KK_ERR_STALE_HANDLE
    # a coarse row with more than 256 distinct columns
    W = to_device(g.random_csr(2, 400, 400, seed=5, empty_row_frac=0.0))
    I = to_device(g.random_csr(400, 400, 30, seed=6, empty_row_frac=0.0))
    with pytest.raises(KKError) as e:
        h.rap(W, I, I)
    assert e.value.status == KK_ERR_UNSUPPORTED_TYPE
    h.close()
