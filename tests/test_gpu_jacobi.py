"""Jacobi-fused SpGEMM C = (I - w D^-1 A) B on the GPU (Sec. 2.2.2)
against the oracle's MSAK composition (oracle.jacobi): row map and sorted columns
bit-exact, values within tau * (|b| + |w dinv_i| sum|a||b|) (SURVEY R5 applied to Eq. 2)."""
import numpy as np
import pytest
import torch

from workloads import generators as g

from .helpers import TAU, to_device

pytestmark = pytest.mark.gpu


def _square_with_diag(m, maxr, seed, sorted_rows=True):
    A = g.random_csr(m, m, maxr, seed=seed, sorted_rows=sorted_rows)
    rm = A.row_map.tolist()
    rows, cols, vals = [], [], []
    for i in range(m):
        c = A.entries[rm[i]:rm[i + 1]].tolist()
        v = A.values[rm[i]:rm[i + 1]].tolist()
        if i not in c:
            c.append(i)
            v.append(2.0 + (i % 5))
        order = np.argsort(c) if sorted_rows else np.arange(len(c))
        cols += [c[t] for t in order]
        vals += [v[t] for t in order]
        rows.append(len(c))
    row_map = torch.zeros(m + 1, dtype=torch.int64)
    row_map[1:] = torch.cumsum(torch.tensor(rows), 0)
    return g.CSR(m, m, row_map, torch.tensor(cols, dtype=torch.int32), torch.tensor(vals, dtype=torch.float64))


def _run(A, B, dinv, w, vt=torch.float64, ot=torch.int64, **opts):
    from paper_2103_11991_b200 import SpGEMM

    Ad, Bd = to_device(A, "cuda", vt, ot), to_device(B, "cuda", vt, ot)
    h = SpGEMM(**opts)
    C = h.jacobi(w, torch.as_tensor(dinv, dtype=vt).cuda(), Ad, Bd)
    torch.cuda.synchronize()
    h.close()
    return C.row_map.cpu().numpy().astype(np.int64), C.entries.cpu().numpy(), C.values.cpu().double().numpy()


def _check(oracle_mod, A, B, dinv, w, got, vt=torch.float64):
    rm, ent, val = got
    orm, oent, oval, obnd = oracle_mod.jacobi(w, np.asarray(dinv, dtype=np.float64), A, B)
    assert np.array_equal(rm, orm), "row map"
    assert np.array_equal(ent, oent), "columns"
    tau = TAU[vt]
    bad = np.abs(val - oval) > tau * obnd + (0 if vt == torch.float64 else 1e-30)
    assert not bad.any(), f"{bad.sum()} values outside tolerance, worst {np.max(np.abs(val - oval) / (obnd + 1e-300))}"


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("m,k,ma,mb", [(70, 40, 6, 8), (300, 120, 12, 30), (200, 500, 40, 45)])
@pytest.mark.parametrize("vt", [torch.float64, torch.float32])
def test_jacobi_random(oracle_mod, seed, m, k, ma, mb, vt):
    A = _square_with_diag(m, ma, seed)
    B = g.random_csr(m, k, mb, seed=seed + 10)
    dinv = np.random.default_rng(seed).uniform(-1.5, 1.5, size=m)
    _check(oracle_mod, A, B, dinv, 0.7, _run(A, B, dinv, 0.7, vt), vt)


@pytest.mark.parametrize("opts", [dict(compression="off"), dict(patterns=False), dict(compression="on")])
def test_jacobi_paths(oracle_mod, opts):
    """Pattern (num_rank), hash (num_strict) and general (num_warp) tiers all fuse."""
    A = _square_with_diag(400, 10, 3)
    B = g.random_csr(400, 300, 20, seed=4)
    dinv = np.random.default_rng(5).uniform(0.1, 1.0, size=400)
    _check(oracle_mod, A, B, dinv, 0.5, _run(A, B, dinv, 0.5, **opts))


def test_jacobi_unsorted(oracle_mod):
    A = _square_with_diag(150, 8, 6, sorted_rows=False)
    B = g.random_csr(150, 90, 12, seed=7, sorted_rows=False)
    dinv = np.random.default_rng(8).uniform(-1, 1, size=150)
    _check(oracle_mod, A, B, dinv, 1.3, _run(A, B, dinv, 1.3))


@pytest.mark.parametrize("ot", [torch.int32, torch.int64])
def test_jacobi_smoothed_prolongator(oracle_mod, ot):
    """(I - w D^-1 A) P for the 7-point Laplacian with 3x3x3 aggregates (SURVEY NEXT-1
    workload, C3J) at 24^3 and 25^3 (a ragged last aggregate), integer A/P, w = 2/3."""
    for n in (24, 25):
        A, P, dinv, w = g.config("C3J", size=n)
        _check(oracle_mod, A, P, dinv.numpy(), w, _run(A, P, dinv, w, ot=ot))


def test_jacobi_stencil_square(oracle_mod):
    """A*A-shaped Jacobi product on the 27-point Laplacian (pattern rows, B rows of 27)."""
    A, B = g.config("C2", size=14)
    dinv = g.diagonal_inverse(A).numpy()
    _check(oracle_mod, A, B, dinv, 0.8, _run(A, B, dinv, 0.8))


def test_jacobi_errors():
    from paper_2103_11991_b200 import SpGEMM
    from paper_2103_11991_b200._ffi import KKError

    A = to_device(g.random_csr(20, 30, 4, seed=1), "cuda")
    B = to_device(g.random_csr(30, 10, 4, seed=2), "cuda")
    h = SpGEMM()
    with pytest.raises(KKError):
        h.jacobi(0.5, torch.ones(20, dtype=torch.float64, device="cuda"), A, B)  # A not square
    h.close()
    # missing diagonal under validate
    A = to_device(g.random_csr(30, 30, 4, seed=3), "cuda")
    h = SpGEMM(validate=True)
    with pytest.raises(KKError, match="A\\(i,i\\)"):
        h.jacobi(0.5, torch.ones(30, dtype=torch.float64, device="cuda"), A, B)
    h.close()


@pytest.mark.parametrize("k", [200000, 20000])
@pytest.mark.parametrize("det", [False, True])
def test_jacobi_long_rows(oracle_mod, k, det):
    """Rows with nnz(C_i) > 512: the fused form in the long-row tiers -- the CTA bit-vector
    tier (k = 200K, values in shared memory or, above its capacity, at L2) and the windowed
    dense tier (k = 20K); deterministic mode too."""
    m = 300
    A = _square_with_diag(m, 60, 7)
    B = g.random_csr(m, k, 300, seed=8, empty_row_frac=0.0)
    dinv = 1.0 / (2.0 + np.arange(m) % 7)
    got = _run(A, B, dinv, 2.0 / 3.0, deterministic=det)
    _check(oracle_mod, A, B, dinv, 2.0 / 3.0, got)
