"""Pins for the CPU oracle (oracle/kk_oracle.c) against things other than itself.

* brute force: dense fp64 products and integer pattern products on tiny matrices
  (SURVEY.md §4 T0), including rectangular shapes (catches transposed operands),
  empty rows, explicit zeros, exact cancellations, duplicate and unsorted entries;
* closed forms for the stencil workloads (SURVEY.md §8 size table, derived below
  independently by counting lattice points);
* SPEC.md worked examples (tests/golden/spec_examples.json);
* invariants: flops identity sum_j nnz(A(:,j)) nnz(B(j,:)), symbolic nnz =
  numeric nnz, A*I = A, Kronecker identity (L (x) M)^2 = L^2 (x) M^2.
"""
import json
import os

import numpy as np
import pytest
import torch

from workloads import generators as g

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def dense_to_csr(D):
    D = np.asarray(D, dtype=np.float64)
    m, k = D.shape
    rm = [0]
    ent, val = [], []
    for i in range(m):
        for c in range(k):
            if D[i, c] != 0:
                ent.append(c)
                val.append(D[i, c])
        rm.append(len(ent))
    return g.CSR(m, k, torch.tensor(rm, dtype=torch.int64), torch.tensor(ent, dtype=torch.int32),
                 torch.tensor(val, dtype=torch.float64))


def brute(A, B):
    """Dense brute force: values (duplicates summed), bound sum|a||b|, pattern counts."""
    Ad, Bd = A.to_dense().numpy(), B.to_dense().numpy()
    absA = g.CSR(A.nrows, A.ncols, A.row_map, A.entries, A.values.abs()).to_dense().numpy()
    absB = g.CSR(B.nrows, B.ncols, B.row_map, B.entries, B.values.abs()).to_dense().numpy()
    pa = g.CSR(A.nrows, A.ncols, A.row_map, A.entries, torch.ones(A.nnz, dtype=torch.float64)).to_dense().numpy()
    pb = g.CSR(B.nrows, B.ncols, B.row_map, B.entries, torch.ones(B.nnz, dtype=torch.float64)).to_dense().numpy()
    return Ad @ Bd, absA @ absB, (pa @ pb)


def csr_to_dense_np(m, k, rm, ent, val):
    D = np.zeros((m, k))
    for i in range(m):
        for p in range(rm[i], rm[i + 1]):
            D[i, ent[p]] += val[p]
    return D


CASES = [
    # (m, n, k, maxA, maxB, kwargs)
    (17, 23, 31, 6, 5, {}),
    (40, 40, 40, 8, 8, {}),
    (64, 9, 64, 5, 40, {}),
    (5, 64, 3, 40, 3, {}),
    (33, 20, 50, 7, 9, dict(sorted_rows=False)),
    (30, 25, 45, 10, 10, dict(duplicates=True, sorted_rows=False)),
    (30, 25, 45, 10, 10, dict(explicit_zeros=True)),
    (20, 1, 20, 3, 20, dict(duplicates=True)),
    (0, 5, 7, 3, 3, {}),
    (6, 0, 7, 3, 3, {}),
    (6, 5, 0, 3, 3, {}),
]


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_oracle_vs_bruteforce(oracle_mod, case, seed):
    m, n, k, ma, mb, kw = CASES[case]
    A = g.random_csr(m, n, ma, seed=seed, **kw)
    B = g.random_csr(n, k, mb, seed=seed + 100, **kw)
    C, bound, pat = brute(A, B)
    rm, ent, val, bnd = oracle_mod.spgemm(A, B)
    # row map = structural counts of the Boolean product (R1)
    counts = (pat > 0).sum(1)
    assert np.array_equal(np.diff(rm), counts)
    for i in range(m):
        cols = ent[rm[i]:rm[i + 1]]
        assert np.all(np.diff(cols) > 0), "rows sorted, distinct (R4)"
        assert np.array_equal(cols, np.nonzero(pat[i] > 0)[0])
    D = csr_to_dense_np(m, k, rm, ent, val)
    Bd = csr_to_dense_np(m, k, rm, ent, bnd)
    assert np.all(np.abs(D - C) <= 1e-12 * bound + 1e-300)
    assert np.allclose(Bd, bound, rtol=1e-13, atol=0)
    # flops identity via an independent column count of A (SURVEY §8c muladds pin)
    fl, tot = oracle_mod.row_flops(A, B)
    colcnt = np.bincount(A.entries.numpy().astype(np.int64), minlength=n) if A.nnz else np.zeros(n, np.int64)
    assert tot == int(np.dot(colcnt, B.row_lengths().numpy()))
    assert np.array_equal(fl, pat.sum(1).astype(np.int64)) if m else True


@pytest.mark.parametrize("seed", [4, 5])
def test_oracle_integer_exact(oracle_mod, seed):
    A = g.random_csr(50, 50, 8, seed=seed, integer_values=True)
    B = g.random_csr(50, 50, 8, seed=seed + 7, integer_values=True, duplicates=True)
    C, _, _ = brute(A, B)
    rm, ent, val, _ = oracle_mod.spgemm(A, B)
    assert np.array_equal(csr_to_dense_np(50, 50, rm, ent, val), C)


def test_spec_examples(oracle_mod):
    gold = json.load(open(GOLD))
    for ex in gold["compress"]:
        row = ex["row"]
        B = g.CSR(1, 128, torch.tensor([0, len(row)]), torch.tensor(row, dtype=torch.int32),
                  torch.ones(len(row), dtype=torch.float64))
        rm, w, mk = oracle_mod.compress(B)
        assert [[int(a), int(b)] for a, b in zip(w, mk)] == ex["pairs"], ex["cite"]
    for ex in gold["symbolic"]:
        rm = oracle_mod.symbolic(dense_to_csr(ex["A"]), dense_to_csr(ex["B"]))
        assert list(np.diff(rm)) == ex["counts"], ex["cite"]
    for ex in gold["numeric"]:
        A, B = dense_to_csr(ex["A"]), dense_to_csr(ex["B"])
        rm, ent, val, _ = oracle_mod.spgemm(A, B)
        assert int(rm[-1]) == ex["nnz"], ex["cite"]
        Cd = np.asarray(ex["C"], dtype=np.float64)
        assert np.array_equal(csr_to_dense_np(A.nrows, B.ncols, rm, ent, val), Cd), ex["cite"]


def test_structural_zero_kept(oracle_mod):
    # R1: C3a-like cancellation: [[1,1]] * [[1],[-1]] stores a 0 (SURVEY §8c pins)
    A = g.CSR(1, 2, torch.tensor([0, 2]), torch.tensor([0, 1], dtype=torch.int32), torch.tensor([1.0, 1.0]).double())
    B = g.CSR(2, 1, torch.tensor([0, 1, 2]), torch.tensor([0, 0], dtype=torch.int32), torch.tensor([1.0, -1.0]).double())
    rm, ent, val, bnd = oracle_mod.spgemm(A, B)
    assert list(rm) == [0, 1] and list(ent) == [0] and val[0] == 0.0 and bnd[0] == 2.0


def _lattice_square_counts(dims, offsets):
    """Independent count of nnz(A^2) and muladds for a stencil matrix A by enumerating
    two-hop lattice paths in pure Python (small grids only)."""
    import itertools
    dims = list(dims)
    nd = len(dims)

    def inbox(p):
        return all(0 <= p[a] < dims[a] for a in range(nd))

    nnz = 0
    muladds = 0
    for p in itertools.product(*[range(d) for d in dims]):
        reach = set()
        for o1 in offsets:
            q = tuple(p[a] + o1[a] for a in range(nd))
            if not inbox(q):
                continue
            for o2 in offsets:
                r = tuple(q[a] + o2[a] for a in range(nd))
                if inbox(r):
                    reach.add(r)
                    muladds += 1
        nnz += len(reach)
    return nnz, muladds


def test_closed_forms_C1(oracle_mod):
    A, B = g.config("C1")
    rm, ent, val, _ = oracle_mod.spgemm(A, B)
    _, tot = oracle_mod.row_flops(A, B)
    assert int(rm[-1]) == 12676 and tot == 24456  # SURVEY §8 size table, C1
    nnz, mul = _lattice_square_counts((32, 32), g._box_offsets(2, 1, "cross"))
    assert (nnz, mul) == (12676, 24456)
    lens = np.diff(rm)
    assert int((lens == 13).sum()) == (32 - 4) ** 2
    # interior values: diag 20, +-e -8, +-2e 1, diagonal neighbours 2, row sum 0
    n = 32
    i = 10 + n * 12
    cols = ent[rm[i]:rm[i + 1]]
    vals = dict(zip(cols.tolist(), val[rm[i]:rm[i + 1]].tolist()))
    assert vals[i] == 20 and vals[i + 1] == -8 and vals[i - n] == -8 and vals[i + 2] == 1 and vals[i - 2 * n] == 1
    assert vals[i + 1 + n] == 2 and vals[i - 1 + n] == 2 and sum(vals.values()) == 0


@pytest.mark.parametrize("n", [3, 5, 8])
def test_closed_forms_27pt(oracle_mod, n):
    A, B = g.config("C2", size=n)
    rm, ent, val, _ = oracle_mod.spgemm(A, B)
    _, tot = oracle_mod.row_flops(A, B)
    assert int(rm[-1]) == (5 * n - 6) ** 3 and tot == (9 * n - 10) ** 3
    if n <= 5:
        assert _lattice_square_counts((n, n, n), g._box_offsets(3, 1, "box")) == ((5 * n - 6) ** 3, (9 * n - 10) ** 3)
    if n >= 5:
        c = 2 + n * (2 + n * 2)  # an interior row (all 125 neighbours within the box)
        cols = ent[rm[c]:rm[c + 1]]
        assert len(cols) == 125
        vals = dict(zip(cols.tolist(), val[rm[c]:rm[c + 1]].tolist()))
        assert vals[c] == 702 and sum(vals.values()) == 0
        # |d|_inf = 1: -52 + (N(d) - 2), N(d) = prod(3 - |d_i|): face -36, edge -42, corner -46
        assert vals[c + 1] == -36 and vals[c + 1 + n] == -42 and vals[c + 1 + n + n * n] == -46
        # |d|_inf = 2: value N(d) = prod over axes of the number of ways to split d_i into two
        # steps in {-1,0,1}: 1 if |d_i| = 2, 2 if |d_i| = 1, 3 if d_i = 0 -> {9, 6, 4, 3, 2, 1}
        assert vals[c + 2] == 9 and vals[c + 2 + n] == 6 and vals[c + 2 + n + n * n] == 4
        assert vals[c + 2 + 2 * n] == 3 and vals[c + 2 + 2 * n + n * n] == 2 and vals[c + 2 + 2 * n + 2 * n * n] == 1


def test_closed_forms_block_kron(oracle_mod):
    # (L27 (x) M)^2 = L27^2 (x) M^2: nnz 9(5n-6)^3, muladds 27(9n-10)^3
    n = 4
    A, B = g.config("C5", size=n)
    rm, ent, val, _ = oracle_mod.spgemm(A, B)
    _, tot = oracle_mod.row_flops(A, B)
    assert int(rm[-1]) == 9 * (5 * n - 6) ** 3 and tot == 27 * (9 * n - 10) ** 3
    L, L2 = g.config("C2", size=n)
    lrm, lent, lval, _ = oracle_mod.spgemm(L, L2)
    Ld = csr_to_dense_np(n ** 3, n ** 3, lrm, lent, lval)
    M = np.array(g._BLOCK_M)
    K = np.kron(Ld, M @ M)
    D = csr_to_dense_np(A.nrows, A.nrows, rm, ent, val)
    assert np.array_equal(D, K)


def test_galerkin_C3_small(oracle_mod):
    # R*A*P on a 9^3 grid with 3x3x3 aggregates: coarse operator is the 7-point pattern
    # on 3^3 with interior row [54, -9 x 6] (SURVEY §8c pins, C3b interior values)
    n = 9
    A, P, R = g.config("C3", size=n)
    trm, tent, tval, _ = oracle_mod.spgemm(A, P)
    T = g.CSR(A.nrows, P.ncols, torch.tensor(trm), torch.tensor(tent), torch.tensor(tval))
    assert int(trm[-1]) == int(np.count_nonzero(brute(A, P)[2]))  # structural count (R1)
    crm, cent, cval, _ = oracle_mod.spgemm(R, T)
    nc = 3
    c = 1 + nc * (1 + nc * 1)
    cols = cent[crm[c]:crm[c + 1]].tolist()
    vals = dict(zip(cols, cval[crm[c]:crm[c + 1]].tolist()))
    assert sorted(cols) == sorted([c, c - 1, c + 1, c - nc, c + nc, c - nc * nc, c + nc * nc])
    assert vals[c] == 54 and all(vals[x] == -9 for x in cols if x != c)
    Rd, Ad, Pd = R.to_dense().numpy(), A.to_dense().numpy(), P.to_dense().numpy()
    assert np.array_equal(csr_to_dense_np(R.nrows, P.ncols, crm, cent, cval), Rd @ Ad @ Pd)


def test_rmat_paths(oracle_mod):
    # unit-valued RMAT: C(i,j) = number of length-2 paths (SURVEY §8c pins, C4)
    A = g.rmat(scale=8, edge_factor=8, seed=3)
    B = A.clone()
    rm, ent, val, _ = oracle_mod.spgemm(A, B)
    Ad = A.to_dense().numpy()
    assert np.array_equal(csr_to_dense_np(A.nrows, A.nrows, rm, ent, val), Ad @ Ad)
    assert np.array_equal(np.diff(rm), ((Ad @ Ad) > 0).sum(1))


def test_identity_and_symmetry(oracle_mod):
    A = g.random_csr(30, 30, 6, seed=9)
    I = g.CSR(30, 30, torch.arange(31), torch.arange(30, dtype=torch.int32), torch.ones(30, dtype=torch.float64))
    rm, ent, val, _ = oracle_mod.spgemm(A, I)
    assert np.array_equal(rm, A.row_map.numpy()) and np.array_equal(ent, A.entries.numpy())
    assert np.array_equal(val, A.values.numpy())
    S, S2 = g.config("C2", size=4)
    rm, ent, _, _ = oracle_mod.spgemm(S, S2)
    P = csr_to_dense_np(64, 64, rm, ent, np.ones(len(ent)))
    assert np.array_equal(P, P.T)


def test_compress_roundtrip(oracle_mod):
    B = g.random_csr(40, 200, 30, seed=5, sorted_rows=False, duplicates=True)
    rm, w, mk = oracle_mod.compress(B)
    for j in range(B.nrows):
        cols = set(B.entries[B.row_map[j]:B.row_map[j + 1]].tolist())
        rec = set()
        ws = w[rm[j]:rm[j + 1]]
        assert np.all(np.diff(ws) > 0)
        for ww, mm in zip(ws, mk[rm[j]:rm[j + 1]]):
            assert mm != 0
            for b in range(32):
                if (int(mm) >> b) & 1:
                    rec.add(int(ww) * 32 + b)
        assert rec == cols


# ---- Jacobi-fused SpGEMM reference (Sec. 2.2.2) ----------------------

def _square_with_diag(m, maxr, seed, diag=True):
    A = g.random_csr(m, m, maxr, seed=seed)
    D = A.to_dense().numpy()
    if diag:
        rng = np.random.default_rng(seed + 7)
        for i in range(m):
            D[i, i] = rng.uniform(1.0, 3.0) * (1 if rng.random() < 0.5 else -1)
    return dense_to_csr(D)


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("diag", [True, False])
def test_jacobi_oracle_vs_dense(oracle_mod, seed, diag):
    """C = (I - w D^-1 A) B against a dense evaluation of the formula; pattern = the
    Boolean union of B's and A*B's patterns (pattern(C) = pattern(E) when A's diagonal is
    stored)."""
    m, k = 30, 17
    A = _square_with_diag(m, 6, seed, diag)
    B = g.random_csr(m, k, 5, seed=seed + 50)
    rng = np.random.default_rng(seed)
    dinv = rng.uniform(-2, 2, size=m)
    w = 0.7
    rm, ent, val, bnd = oracle_mod.jacobi(w, dinv, A, B)
    Ad, Bd = A.to_dense().numpy(), B.to_dense().numpy()
    want = Bd - w * np.diag(dinv) @ (Ad @ Bd)
    pa = (Ad != 0).astype(float)
    pb = (Bd != 0).astype(float)
    pat = ((pa @ pb) + pb) > 0
    assert np.array_equal(np.diff(rm), pat.sum(1))
    if diag:
        rmE, entE, _, _ = oracle_mod.spgemm(A, B)
        assert np.array_equal(rm, rmE) and np.array_equal(ent, entE)
    got = csr_to_dense_np(m, k, rm, ent, val)
    bound = np.abs(Bd) + abs(w) * np.abs(dinv)[:, None] * (np.abs(Ad) @ np.abs(Bd))
    assert np.all(np.abs(got - want) <= 1e-12 * bound + 1e-300)
    assert np.allclose(csr_to_dense_np(m, k, rm, ent, bnd), bound, rtol=1e-13, atol=0)


def test_jacobi_oracle_special_cases(oracle_mod):
    """omega = 0 gives B on E's pattern (E-only entries are explicit zeros); A = D with
    dinv = 1/diag gives (1 - omega) B exactly."""
    m, k = 12, 9
    A = _square_with_diag(m, 4, 11)
    B = g.random_csr(m, k, 4, seed=12)
    rm, ent, val, _ = oracle_mod.jacobi(0.0, np.ones(m), A, B)
    got = csr_to_dense_np(m, k, rm, ent, val)
    assert np.array_equal(got, B.to_dense().numpy())
    assert len(val) > B.nnz and np.count_nonzero(val) == np.count_nonzero(B.to_dense().numpy())
    Dg = np.diag([2.0, 4.0, 0.5, 8.0] * 3)
    rm, ent, val, _ = oracle_mod.jacobi(0.5, 1.0 / np.diag(Dg), dense_to_csr(Dg), B)
    assert np.array_equal(csr_to_dense_np(m, k, rm, ent, val), 0.5 * B.to_dense().numpy())


def test_jacobi_oracle_smoothed_aggregation_1d(oracle_mod):
    """Textbook smoothed aggregation in 1D: A = tridiag(-1, 2, -1), aggregates of 3 nodes,
    omega = 2/3, D^-1 = 1/2: each column of (I - w D^-1 A) P is the hat (1/3, 2/3, 1, 2/3, 1/3)
    around its aggregate (interior aggregates)."""
    n, na = 30, 10
    A = np.diag(2.0 * np.ones(n)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1)
    P = np.zeros((n, na))
    P[np.arange(n), np.arange(n) // 3] = 1.0
    rm, ent, val, _ = oracle_mod.jacobi(2.0 / 3.0, np.full(n, 0.5), dense_to_csr(A), dense_to_csr(P))
    S = csr_to_dense_np(n, na, rm, ent, val)
    for c in range(1, na - 1):
        col = S[3 * c - 1: 3 * c + 4, c]
        assert np.allclose(col, [1 / 3, 2 / 3, 1.0, 2 / 3, 1 / 3], rtol=0, atol=1e-15)
        assert np.count_nonzero(S[:, c]) == 5


# ---- SpAdd reference (Sec. 2.3) ------------------------------------------

@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("kw", [{}, dict(sorted_rows=False), dict(duplicates=True, sorted_rows=False),
                                dict(explicit_zeros=True)])
def test_spadd_oracle_vs_dense(oracle_mod, seed, kw):
    """alpha A + beta B against dense evaluation; pattern = Boolean union (structural, R1);
    duplicates inside A or B merged."""
    m, k = 40, 33
    A = g.random_csr(m, k, 9, seed=seed, **kw)
    B = g.random_csr(m, k, 12, seed=seed + 20, **kw)
    al, be = 0.75, -1.5
    rm, ent, val, bnd = oracle_mod.spadd(al, A, be, B)
    Ad, Bd = A.to_dense().numpy(), B.to_dense().numpy()
    pa = g.CSR(m, k, A.row_map, A.entries, torch.ones(A.nnz, dtype=torch.float64)).to_dense().numpy()
    pb = g.CSR(m, k, B.row_map, B.entries, torch.ones(B.nnz, dtype=torch.float64)).to_dense().numpy()
    pat = (pa + pb) > 0
    assert np.array_equal(np.diff(rm), pat.sum(1))
    for i in range(m):
        assert np.array_equal(ent[rm[i]:rm[i + 1]], np.nonzero(pat[i])[0])
    got = csr_to_dense_np(m, k, rm, ent, val)
    absA = g.CSR(m, k, A.row_map, A.entries, A.values.abs()).to_dense().numpy()
    absB = g.CSR(m, k, B.row_map, B.entries, B.values.abs()).to_dense().numpy()
    bound = abs(al) * absA + abs(be) * absB
    assert np.all(np.abs(got - (al * Ad + be * Bd)) <= 1e-15 * bound + 1e-300)
    assert np.allclose(csr_to_dense_np(m, k, rm, ent, bnd), bound, rtol=1e-14, atol=0)


def test_spadd_oracle_special_cases(oracle_mod):
    """A + A = 2A on A's pattern; A - A keeps the structural zeros; adding an empty matrix
    returns the merged, sorted A; empty shapes."""
    A = g.random_csr(25, 30, 7, seed=9, duplicates=True, sorted_rows=False)
    Z = g.random_csr(25, 30, 0, seed=1)
    rmz, entz, valz, _ = oracle_mod.spadd(1.0, A, 1.0, Z)
    rm2, ent2, val2, _ = oracle_mod.spadd(1.0, A, 1.0, A)
    assert np.array_equal(rm2, rmz) and np.array_equal(ent2, entz) and np.array_equal(val2, 2 * valz)
    rm0, ent0, val0, _ = oracle_mod.spadd(1.0, A, -1.0, A)
    assert np.array_equal(rm0, rmz) and np.all(val0 == 0)
    D = A.to_dense().numpy()
    assert np.array_equal(csr_to_dense_np(25, 30, rmz, entz, valz), D)
    rm, ent, val, _ = oracle_mod.spadd(2.0, g.random_csr(0, 5, 3, seed=1), 3.0, g.random_csr(0, 5, 3, seed=2))
    assert list(rm) == [0] and len(ent) == 0
