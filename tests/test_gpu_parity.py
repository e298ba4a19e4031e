"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Row maps and sorted column indices must be bit-exact; values within the north-star
bound |c - c_ref| <= tau * sum|a||b| (tau 1e-12 fp64, 1e-5 fp32), and exactly equal on
integer-valued workloads.
"""
import numpy as np
import pytest
import torch

from workloads import generators as g

from .helpers import assert_parity, gpu_spgemm, to_device

pytestmark = pytest.mark.gpu

RANDOM_CASES = [
    (17, 23, 31, 6, 5, {}),
    (40, 40, 40, 8, 8, {}),
    (64, 9, 64, 5, 40, {}),
    (5, 64, 3, 40, 3, {}),
    (33, 20, 50, 7, 9, dict(sorted_rows=False)),
    (30, 25, 45, 10, 10, dict(duplicates=True, sorted_rows=False)),
    (30, 25, 45, 10, 10, dict(explicit_zeros=True)),
    (20, 1, 20, 3, 20, dict(duplicates=True)),
    (300, 200, 5000, 12, 60, {}),
    (0, 5, 7, 3, 3, {}),
    (6, 0, 7, 3, 3, {}),
    (6, 5, 0, 3, 3, {}),
]


@pytest.mark.parametrize("vt", [torch.float64, torch.float32])
@pytest.mark.parametrize("ot", [torch.int32, torch.int64])
@pytest.mark.parametrize("case", range(len(RANDOM_CASES)))
def test_random_small(oracle_mod, case, ot, vt):
    m, n, k, ma, mb, kw = RANDOM_CASES[case]
    A = g.random_csr(m, n, ma, seed=case + 1, **kw)
    B = g.random_csr(n, k, mb, seed=case + 101, **kw)
    got = gpu_spgemm(A, B, value_dtype=vt, offset_dtype=ot)
    assert_parity(oracle_mod, A, B, got, value_dtype=vt)


@pytest.mark.parametrize("compression", ["auto", "on", "off"])
@pytest.mark.parametrize("sort_rows", [True, False])
def test_options_same_result(oracle_mod, compression, sort_rows):
    A, B = g.config("C2", size=12)
    got = gpu_spgemm(A, B, compression=compression, sort_rows=sort_rows)
    assert_parity(oracle_mod, A, B, got, exact=True, sorted_rows=sort_rows)
    st = got[3]
    assert st["compression_used"] == (compression != "off")


@pytest.mark.parametrize("vt", [torch.float64, torch.float32])
def test_C1(oracle_mod, vt):
    A, B = g.config("C1")
    got = gpu_spgemm(A, B, value_dtype=vt, offset_dtype=torch.int32)
    assert_parity(oracle_mod, A, B, got, value_dtype=vt, exact=True)
    assert got[3]["muladds"] == 24456 and got[3]["nnz_c"] == 12676


@pytest.mark.parametrize("values", ["int", "random"])
def test_C2_small(oracle_mod, values):
    A, B = g.config("C2", size=22, values=values)
    got = gpu_spgemm(A, B, offset_dtype=torch.int32)
    assert_parity(oracle_mod, A, B, got, exact=(values == "int"))
    n = 22
    assert got[3]["nnz_c"] == (5 * n - 6) ** 3 and got[3]["muladds"] == (9 * n - 10) ** 3


def test_C2_f32_random(oracle_mod):
    A, B = g.config("C2", size=16, values="random")
    got = gpu_spgemm(A, B, value_dtype=torch.float32, offset_dtype=torch.int32)
    assert_parity(oracle_mod, A, B, got, value_dtype=torch.float32)


def test_C3_galerkin(oracle_mod):
    n = 33
    A, P, R = g.config("C3", size=n)
    from paper_2103_11991_b200 import SpGEMM, CsrMatrix

    Ad, Pd, Rd = (to_device(M) for M in (A, P, R))
    h = SpGEMM()
    T = h(Ad, Pd)
    h2 = SpGEMM()
    Ac = h2(Rd, T)
    torch.cuda.synchronize()
    # T parity
    got_T = (T.row_map.cpu().numpy(), T.entries.cpu().numpy(), T.values.cpu().numpy())
    assert_parity(oracle_mod, A, P, got_T, exact=True)
    # Ac parity against the oracle's R*(A*P), computed entirely on the CPU
    orm, oent, oval, _ = oracle_mod.spgemm(A, P)
    To = g.CSR(A.nrows, P.ncols, torch.tensor(orm), torch.tensor(oent), torch.tensor(oval))
    got_Ac = (Ac.row_map.cpu().numpy(), Ac.entries.cpu().numpy(), Ac.values.cpu().numpy())
    assert_parity(oracle_mod, R, To, got_Ac, exact=True)


def test_C4_rmat_small(oracle_mod):
    A, B = g.config("C4", size=13)
    got = gpu_spgemm(A, B, offset_dtype=torch.int64)
    assert_parity(oracle_mod, A, B, got, exact=True)


def test_C5_block(oracle_mod):
    A, B = g.config("C5", size=10)
    got = gpu_spgemm(A, B, offset_dtype=torch.int64)
    assert_parity(oracle_mod, A, B, got, exact=True)
    assert got[3]["nnz_c"] == 9 * (5 * 10 - 6) ** 3


def _long_rows(seed, m=40, n=400, k=200000, sorted_rows=True, dup=False):
    """A few rows with thousands of products over a wide column range: exercises the
    dense (windowed) symbolic and numeric tiers, cursors and multiple windows."""
    A = g.random_csr(m, n, 120, seed=seed, empty_row_frac=0.0)
    B = g.random_csr(n, k, 400, seed=seed + 9, sorted_rows=sorted_rows, duplicates=dup, empty_row_frac=0.0)
    return A, B


@pytest.mark.parametrize("sorted_rows", [True, False])
@pytest.mark.parametrize("vt", [torch.float64, torch.float32])
def test_dense_tiers(oracle_mod, sorted_rows, vt):
    A, B = _long_rows(7, sorted_rows=sorted_rows)
    got = gpu_spgemm(A, B, value_dtype=vt)
    st = got[3]
    assert st["numeric_bin_rows"][6] > 0 and st["symbolic_bin_rows"][8] > 0, st
    assert_parity(oracle_mod, A, B, got, value_dtype=vt)


@pytest.mark.parametrize("k", [20000, 1600000])
def test_dense_windows_small_and_wide_k(oracle_mod, k):
    """Long rows where the CTA bit-vector tier (k_num_hub, 25.6K < k <= ~1.4M) does not
    apply: k <= 25.6K (one dense column window) and k = 1.6M (several windows, cursors)."""
    A = g.random_csr(24, 300, 100, seed=11, empty_row_frac=0.0)
    B = g.random_csr(300, k, 300, seed=12, empty_row_frac=0.0)
    got = gpu_spgemm(A, B)
    assert got[3]["numeric_bin_rows"][6] > 0
    assert_parity(oracle_mod, A, B, got)


def test_dense_tiers_duplicates(oracle_mod):
    A, B = _long_rows(8, sorted_rows=True, dup=True)
    got = gpu_spgemm(A, B)
    assert_parity(oracle_mod, A, B, got)


def test_symbolic_dense_multiwindow(oracle_mod):
    # k > 1.6M bits: the symbolic bit vector needs several windows
    A = g.random_csr(30, 300, 80, seed=3, empty_row_frac=0.0)
    B = g.random_csr(300, 3_500_000, 300, seed=4, empty_row_frac=0.0)
    for comp in ("on", "off"):
        got = gpu_spgemm(A, B, compression=comp)
        assert got[3]["symbolic_bin_rows"][8] > 0
        assert_parity(oracle_mod, A, B, got)


def test_row_flops_and_compress(oracle_mod):
    from paper_2103_11991_b200 import SpGEMM

    A, B = g.config("C4", size=12)
    Ad, Bd = to_device(A), to_device(B)
    h = SpGEMM()
    f, F, tot = h.row_flops(Ad, Bd)
    of, otot = oracle_mod.row_flops(A, B)
    assert tot == otot and np.array_equal(f.cpu().numpy(), of)
    assert np.array_equal(F.cpu().numpy(), np.concatenate([[0], np.cumsum(of)]))
    ln, w, mk = h.compress(Bd)
    torch.cuda.synchronize()
    brm, ow, om = oracle_mod.compress(B)
    ln, w, mk = ln.cpu().numpy(), w.cpu().numpy(), mk.cpu().numpy().view(np.uint32)
    assert np.array_equal(ln, np.diff(brm))
    rm = B.row_map.numpy()
    got_w = np.concatenate([w[rm[j]:rm[j] + ln[j]] for j in range(B.nrows)])
    got_m = np.concatenate([mk[rm[j]:rm[j] + ln[j]] for j in range(B.nrows)])
    assert np.array_equal(got_w, ow) and np.array_equal(got_m, om)


def test_symbolic_reuse_new_values(oracle_mod):
    from paper_2103_11991_b200 import SpGEMM

    A, B = g.config("C2", size=10, values="random")
    Ad, Bd = to_device(A), to_device(B)
    h = SpGEMM()
    rm, nnz = h.symbolic(Ad, Bd)
    h.numeric(Ad, Bd, rm, nnz=nnz)
    Ad.values.mul_(2.0)  # new values, same pattern
    ent, val = h.numeric(Ad, Bd, rm, nnz=nnz)
    torch.cuda.synchronize()
    A2 = g.CSR(A.nrows, A.ncols, A.row_map, A.entries, A.values * 2.0)
    assert_parity(oracle_mod, A2, B, (rm.cpu().numpy(), ent.cpu().numpy(), val.cpu().numpy()))


def test_errors():
    from paper_2103_11991_b200 import SpGEMM, CsrMatrix
    from paper_2103_11991_b200._ffi import KKError, KK_ERR_DIM_MISMATCH, KK_ERR_STALE_HANDLE, \
        KK_ERR_UNSUPPORTED_TYPE, KK_ERR_INDEX_OVERFLOW

    A = to_device(g.random_csr(10, 8, 3, seed=1))
    B = to_device(g.random_csr(9, 8, 3, seed=2))
    h = SpGEMM()
    with pytest.raises(KKError) as e:
        h.symbolic(A, B)
    assert e.value.status == KK_ERR_DIM_MISMATCH
    B2 = to_device(g.random_csr(8, 8, 3, seed=2))
    rm, nnz = h.symbolic(A, B2)
    B3 = to_device(g.random_csr(8, 8, 3, seed=3))
    with pytest.raises(KKError) as e:
        h.numeric(A, B3, rm, nnz=nnz)
    assert e.value.status == KK_ERR_STALE_HANDLE
    B4 = to_device(g.random_csr(8, 8, 3, seed=2), offset_dtype=torch.int32)
    with pytest.raises(KKError) as e:
        h.symbolic(A, B4)
    assert e.value.status == KK_ERR_UNSUPPORTED_TYPE
    # int32 offsets cannot hold nnz(C) > 2^31-1 -> caught on a large product only; here
    # check validate catches an out-of-range column instead
    bad = g.random_csr(8, 8, 3, seed=5)
    bad.entries[0] = 100
    hv = SpGEMM(validate=True)
    with pytest.raises(KKError) as e:
        hv.symbolic(A, to_device(bad))
    assert e.value.status == KK_ERR_INDEX_OVERFLOW


@pytest.mark.slow
def test_C2_full(oracle_mod):
    """BASELINE configs[1] at full size in the bench's launch configuration (int32 offsets,
    fp64, integer values): the whole product against the oracle -- row map and columns
    bit-exact, values exactly equal."""
    A, B = g.config("C2", device="cuda")
    from paper_2103_11991_b200 import SpGEMM

    Ad, Bd = A.to(offset_dtype=torch.int32), B.to(offset_dtype=torch.int32)
    h = SpGEMM()
    rm, nnz = h.symbolic(Ad, Bd)
    ent, val = h.numeric(Ad, Bd, rm, nnz=nnz)
    torch.cuda.synchronize()
    assert nnz == 120553784 and h.stats()["muladds"] == 704969000
    Ac, Bc = A.to(device="cpu"), B.to(device="cpu")
    got = (rm.cpu().numpy().astype(np.int64), ent.cpu().numpy(), val.cpu().numpy())
    h.close()
    del ent, val
    assert_parity(oracle_mod, Ac, Bc, got, exact=True)
    lens = np.diff(got[0])
    assert lens.max() == 125 and int((lens == 125).sum()) == 96 ** 3


def _diag_first(M):
    """The same matrix with each row's diagonal entry stored first (rows otherwise in
    column order): a partly unsorted B of the kind FEM assemblies produce."""
    rm = M.row_map.to(torch.int64)
    ent, val = M.entries.clone(), M.values.clone()
    for i in range(M.nrows):
        a, b = int(rm[i]), int(rm[i + 1])
        row = ent[a:b]
        d = (row == i).nonzero()
        if len(d) == 0:
            continue
        p = int(d[0])
        order = torch.cat([torch.tensor([p]), torch.arange(0, p), torch.arange(p + 1, b - a)])
        ent[a:b] = row[order]
        val[a:b] = val[a:b][order]
    return g.CSR(M.nrows, M.ncols, M.row_map, ent, val)


@pytest.mark.parametrize("compression", ["auto", "on", "off"])
@pytest.mark.parametrize("values", ["int", "random"])
def test_unsorted_diagonal_first(oracle_mod, compression, values):
    """27-point stencil with the diagonal stored first in every row of A and B: rows of ~27
    entries with one out-of-order word.  Compression must not be used on an unsorted B (the
    compressor merges adjacent equal words only), whatever the option says."""
    A, B = g.config("C2", size=12, values=values)
    A, B = _diag_first(A), _diag_first(B)
    for ot in (torch.int32, torch.int64):
        got = gpu_spgemm(A, B, offset_dtype=ot, compression=compression)
        assert_parity(oracle_mod, A, B, got, exact=(values == "int"))
        assert got[3]["b_sorted"] == 0 and got[3]["compression_used"] == 0


def test_index_overflow_int32():
    """nnz(C) = 46,341^2 = 2,147,488,281 > INT32_MAX: the outer product of a 46,341 x 1
    column of ones and a 1 x 46,341 row of ones.  int32 offsets -> KK_ERR_INDEX_OVERFLOW
    from the i64 scan; int64 offsets -> the exact count and a correct C."""
    from paper_2103_11991_b200 import SpGEMM, CsrMatrix
    from paper_2103_11991_b200._ffi import KKError, KK_ERR_INDEX_OVERFLOW

    n = 46341
    dev = "cuda"

    def col_ones(ot):
        return CsrMatrix(n, 1, torch.arange(n + 1, device=dev, dtype=ot),
                         torch.zeros(n, dtype=torch.int32, device=dev), torch.ones(n, dtype=torch.float64, device=dev))

    def row_ones(ot):
        return CsrMatrix(1, n, torch.tensor([0, n], device=dev, dtype=ot),
                         torch.arange(n, dtype=torch.int32, device=dev), torch.ones(n, dtype=torch.float64, device=dev))

    h = SpGEMM()
    with pytest.raises(KKError) as e:
        h.symbolic(col_ones(torch.int32), row_ones(torch.int32))
    assert e.value.status == KK_ERR_INDEX_OVERFLOW
    A, B = col_ones(torch.int64), row_ones(torch.int64)
    rm, nnz = h.symbolic(A, B)
    assert nnz == n * n == 2147488281
    assert torch.equal(rm, torch.arange(n + 1, device=dev, dtype=torch.int64) * n)
    ent, val = h.numeric(A, B, rm, nnz=nnz)
    torch.cuda.synchronize()
    cols = torch.arange(n, dtype=torch.int32, device=dev)
    for r in (0, 1, n // 2, n - 2, n - 1):
        assert torch.equal(ent[r * n:(r + 1) * n], cols), r
        assert bool((val[r * n:(r + 1) * n] == 1.0).all()), r
    # every entry: columns cycle 0..n-1, every value is 1 (blocks of rows, no 2^31-long temp)
    for r0 in range(0, n, 4096):
        r1 = min(n, r0 + 4096)
        blk = ent[r0 * n:r1 * n].view(r1 - r0, n)
        assert bool((blk == cols).all())
        assert bool((val[r0 * n:r1 * n] == 1.0).all())
    h.close()


def test_hub_long_entry_list_overflow(oracle_mod):
    """A hub row (k_num_hub, k > 25.6K) with more than HUB_LIST = 1,024 A entries whose B rows
    each exceed HUB_LONG = 256 entries: the CTA-walked long-entry list overflows and the
    remaining long rows take the overflow branch."""
    rng = np.random.default_rng(17)
    n, k, na, nb = 1300, 120000, 1100, 300
    # A: row 0 references B rows 0..1099, row 1 a few, row 2 empty
    a_rows = [np.arange(na), np.sort(rng.choice(n, 40, replace=False)), np.zeros(0, dtype=np.int64)]
    arm = np.cumsum([0] + [len(r) for r in a_rows])
    A = g.CSR(3, n, torch.tensor(arm), torch.tensor(np.concatenate(a_rows), dtype=torch.int32),
              torch.tensor(rng.uniform(-1, 1, arm[-1])))
    b_rows = [np.sort(rng.choice(k, nb + (j % 7), replace=False)) for j in range(n)]
    brm = np.cumsum([0] + [len(r) for r in b_rows])
    B = g.CSR(n, k, torch.tensor(brm), torch.tensor(np.concatenate(b_rows), dtype=torch.int32),
              torch.tensor(rng.uniform(-1, 1, brm[-1])))
    for ot in (torch.int32, torch.int64):
        got = gpu_spgemm(A, B, offset_dtype=ot)
        assert got[3]["numeric_bin_rows"][6] > 0
        assert_parity(oracle_mod, A, B, got)


def _banded(m, k, per_row, band, seed, values="random"):
    """Sorted rows with `per_row` distinct columns drawn in [i*k/m - band, i*k/m + band]."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(m):
        c = int(i * k // max(m, 1))
        lo, hi = max(0, c - band), min(k, c + band + 1)
        n = min(per_row, hi - lo)
        sel = np.sort(rng.choice(np.arange(lo, hi), size=n, replace=False))
        rows.append(np.full(n, i))
        cols.append(sel)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    rm = np.zeros(m + 1, dtype=np.int64)
    np.add.at(rm, rows + 1, 1)
    rm = np.cumsum(rm)
    vals = rng.uniform(-1, 1, size=len(cols)) if values == "random" else np.ones(len(cols))
    return g.CSR(m, k, torch.tensor(rm), torch.tensor(cols, dtype=torch.int32), torch.tensor(vals))


@pytest.mark.parametrize("band,per_a,per_b", [(300, 20, 30), (6000, 12, 60), (30000, 6, 40), (40, 30, 30)])
@pytest.mark.parametrize("vt", [torch.float64, torch.float32])
def test_window_and_pattern_paths(oracle_mod, band, per_a, per_b, vt):
    """Banded rows: symbolic bit-vector windows of every width class, rows whose pattern is
    kept (<= 64 words) and rows whose pattern is not (numeric falls back to the hash)."""
    n = 3000
    A = _banded(1500, n, per_a, band // 4, seed=band)
    B = _banded(n, n, per_b, band, seed=band + 1)
    for ot in (torch.int32, torch.int64):
        got = gpu_spgemm(A, B, value_dtype=vt, offset_dtype=ot)
        assert_parity(oracle_mod, A, B, got, value_dtype=vt)
        got = gpu_spgemm(A, B, value_dtype=vt, offset_dtype=ot, patterns=False)
        assert_parity(oracle_mod, A, B, got, value_dtype=vt)


@pytest.mark.parametrize("band,binid", [(45000, 14), (75000, 15)])
def test_wide_symbolic_windows(oracle_mod, band, binid):
    """Rows whose columns span 64K-192K (C5's 3-dof stencil rows span ~155K): the symbolic
    bit-vector windows of 128K and 192K bits (bins 14, 15) instead of the hash table."""
    n, k = 3000, 600000
    A = _banded(1200, n, 16, 40, seed=band)
    B = _banded(n, k, 40, band, seed=band + 1)
    for ot in (torch.int32, torch.int64):
        got = gpu_spgemm(A, B, offset_dtype=ot)
        assert_parity(oracle_mod, A, B, got)
        assert got[3]["symbolic_bin_rows"][binid] > 0, got[3]["symbolic_bin_rows"]


@pytest.mark.parametrize("ot", [torch.int32, torch.int64])
def test_speculative_symbolic_tables(oracle_mod, ot):
    """Rows bound for the large symbolic hash tables (ub > 512 words, columns spread past
    the widest window) first run with a 256-slot table: rows whose B rows overlap (few
    distinct words) finish there, rows with more than 128 distinct words are abandoned and
    redone from the retry list with the 8192-slot table; C equals the oracle."""
    rng = np.random.default_rng(31)
    k, nb = 1_000_000, 400
    base = np.sort(rng.choice(k, 30, replace=False))
    b_rows = []
    for j in range(nb):
        if j < 200:  # near-identical rows: the shared 30 columns, two of them moved
            r = base.copy()
            r[rng.choice(30, 2, replace=False)] = rng.choice(k, 2, replace=False)
            b_rows.append(np.unique(r))
        else:
            b_rows.append(np.sort(rng.choice(k, 30, replace=False)))
    brm = np.cumsum([0] + [len(r) for r in b_rows])
    B = g.CSR(nb, k, torch.tensor(brm), torch.tensor(np.concatenate(b_rows), dtype=torch.int32),
              torch.tensor(rng.uniform(-1, 1, brm[-1])))
    a_rows = [np.sort(rng.choice(200, 40, replace=False)) if i < 150 else
              np.sort(200 + rng.choice(200, 40, replace=False)) for i in range(300)]
    arm = np.cumsum([0] + [len(r) for r in a_rows])
    A = g.CSR(300, nb, torch.tensor(arm), torch.tensor(np.concatenate(a_rows), dtype=torch.int32),
              torch.tensor(rng.uniform(-1, 1, arm[-1])))
    got = gpu_spgemm(A, B, offset_dtype=ot, timing=True)
    assert_parity(oracle_mod, A, B, got)
    names = " ".join(got[3]["kernels"])
    assert "sym_rows_spec" in names and "sym_rows_retry" in names, names


def test_pattern_pool_overflow(oracle_mod):
    """Rows of ~60 words each overflow the 48-pairs-per-row pattern pool: the rows that do
    not get a slot are computed by the hash kernels; the result is unchanged."""
    n = 4000
    A = _banded(800, n, 24, 900, seed=5)
    B = _banded(n, n, 40, 1000, seed=6)
    got = gpu_spgemm(A, B)
    assert_parity(oracle_mod, A, B, got)


@pytest.mark.parametrize("blocks", [1, 3, 8, None])
@pytest.mark.parametrize("ot", [torch.int32, torch.int64])
def test_multiply_host_blocks(oracle_mod, blocks, ot):
    """Host-buffer path (the e2e API): A in row blocks pipelined over three streams; the
    assembled host C equals the oracle (row map, columns bit-exact)."""
    from paper_2103_11991_b200 import CsrMatrix, SpGEMM

    A, B = g.config("C2", size=11, values="random")

    def host(M):
        return CsrMatrix(M.nrows, M.ncols, M.row_map.to(ot).pin_memory(), M.entries.pin_memory(),
                         M.values.pin_memory())

    h = SpGEMM()
    for _ in range(2):  # second call reuses the cached staging buffers
        C = h.multiply_host(host(A), host(B), blocks=blocks)
        got = (C.row_map.numpy().astype(np.int64), C.entries.numpy().copy(), C.values.numpy().copy())
        assert_parity(oracle_mod, A, B, got)
    # A*A from ONE host matrix (A's row blocks copied from B's device copy), first block a
    # quarter of the others (blocks >= 4), values changed between calls
    Ah = host(A)
    for trial in range(2):
        if trial:
            Ah.values.mul_(-0.5)
        C = h.multiply_host(Ah, Ah, blocks=blocks)
        Ad = g.CSR(A.nrows, A.ncols, Ah.row_map.to(torch.int64), Ah.entries, Ah.values.clone())
        got = (C.row_map.numpy().astype(np.int64), C.entries.numpy().copy(), C.values.numpy().copy())
        assert_parity(oracle_mod, Ad, Ad, got)
    # a row block count above the row count, and an empty A
    E = g.random_csr(0, B.nrows, 3, seed=1)
    C = h.multiply_host(host(E), host(B), blocks=4)
    assert C.row_map.numel() == 1 and int(C.row_map[0]) == 0 and C.entries.numel() == 0
    h.close()


@pytest.mark.parametrize("square", [True, False])
def test_multiply_host_planned(oracle_mod, square, monkeypatch):
    """Host-buffer path with the block plan (A of >= 65,536 rows, no block count): a small first
    block, the rest planned from its output size (a small KK_HOST_BLOCK_BYTES forces many
    blocks, several B chunks per block and slot reuse); A*A from one host matrix and A*B from
    two; C equals the oracle."""
    from paper_2103_11991_b200 import CsrMatrix, SpGEMM

    monkeypatch.setenv("KK_HOST_BLOCK_BYTES", "1500000")
    A = g.laplacian_3d_27pt(41, values="random", seed=3)  # 68,921 rows

    def host(M):
        return CsrMatrix(M.nrows, M.ncols, M.row_map.to(torch.int32).pin_memory(), M.entries.pin_memory(),
                         M.values.pin_memory())

    Ah = host(A)
    Bh = Ah if square else host(A)
    h = SpGEMM()
    for _ in range(2):
        C = h.multiply_host(Ah, Bh)
        got = (C.row_map.numpy().astype(np.int64), C.entries.numpy().copy(), C.values.numpy().copy())
        assert_parity(oracle_mod, A, A, got)
    h.close()


def test_multiply_host_edges(oracle_mod, monkeypatch):
    """Host-buffer path: int64 offsets and fp32 values with planned blocks; B with unsorted
    rows (B_C off, the sortedness flags carried across the blocks' B prefixes); a column out of
    range under validate fails with KK_ERR_INDEX_OVERFLOW mid-pipeline and the handle stays
    usable."""
    from paper_2103_11991_b200 import CsrMatrix, SpGEMM
    from paper_2103_11991_b200._ffi import KKError

    monkeypatch.setenv("KK_HOST_BLOCK_BYTES", "1000000")
    A = g.laplacian_3d_27pt(41, values="random", seed=4)  # 68,921 rows

    def host(M, ot=torch.int32, vt=torch.float64):
        return CsrMatrix(M.nrows, M.ncols, M.row_map.to(ot).pin_memory(), M.entries.pin_memory(),
                         M.values.to(vt).pin_memory())

    h = SpGEMM(validate=True)
    # int64 offsets, fp32 values
    C = h.multiply_host(host(A, torch.int64, torch.float32), host(A, torch.int64, torch.float32))
    got = (C.row_map.numpy().astype(np.int64), C.entries.numpy().copy(), C.values.numpy().copy())
    assert_parity(oracle_mod, A, A, got, value_dtype=torch.float32)
    # B with reversed rows (unsorted)
    rm = A.row_map.numpy()
    ent = A.entries.numpy().copy()
    for r in range(0, A.nrows, 7):
        ent[rm[r]:rm[r + 1]] = ent[rm[r]:rm[r + 1]][::-1].copy()
    val = A.values.numpy().copy()
    for r in range(0, A.nrows, 7):
        val[rm[r]:rm[r + 1]] = val[rm[r]:rm[r + 1]][::-1].copy()
    Bu = g.CSR(A.nrows, A.ncols, A.row_map, torch.tensor(ent), torch.tensor(val))
    C = h.multiply_host(host(A), host(Bu))
    got = (C.row_map.numpy().astype(np.int64), C.entries.numpy().copy(), C.values.numpy().copy())
    assert_parity(oracle_mod, A, Bu, got)
    # a bad column in the last rows of A
    ent2 = A.entries.clone()
    ent2[-3] = A.ncols + 5
    Ab = g.CSR(A.nrows, A.ncols, A.row_map, ent2, A.values)
    with pytest.raises(KKError, match="INDEX_OVERFLOW|out of range"):
        h.multiply_host(host(Ab), host(A))
    C = h.multiply_host(host(A), host(A))
    got = (C.row_map.numpy().astype(np.int64), C.entries.numpy().copy(), C.values.numpy().copy())
    assert_parity(oracle_mod, A, A, got)
    h.close()


@pytest.mark.parametrize("vt", [torch.float64, torch.float32])
def test_wide_pattern_hashed_word_table(oracle_mod, vt):
    """Rows whose kept pattern (<= 64 words) spans more than the dense word index (2,048
    words): the numeric rank kernel with the hashed word table (num_rank_hash)."""
    n, k = 4000, 400000
    A = _banded(1200, n, 4, 40, seed=21)
    B = _banded(n, k, 14, 60000, seed=22)
    got = gpu_spgemm(A, B, value_dtype=vt, offset_dtype=torch.int32)
    assert_parity(oracle_mod, A, B, got, value_dtype=vt)
    st = got[3]
    assert sum(st["numeric_bin_rows"][12:16]) > 0, "expected rows in the hashed-pattern bins"


def test_cluster_tier_windows(oracle_mod):
    """Rows far above one CTA's value array on a wide k (k = 1M): the cluster tier (column
    slices across the CTAs of a thread-block cluster, slice offsets through distributed
    shared memory), slices with several rank windows, B-row segments long enough to be
    walked by the whole CTA, and more of them than its list holds (CL_LIST = 512)."""
    rng = np.random.default_rng(23)
    k, nb, per = 1_000_000, 700, 20000
    b_rows = [np.sort(rng.choice(k, per - (j % 13), replace=False)) for j in range(nb)]
    brm = np.cumsum([0] + [len(r) for r in b_rows])
    B = g.CSR(nb, k, torch.tensor(brm), torch.tensor(np.concatenate(b_rows), dtype=torch.int32),
              torch.tensor(rng.uniform(-1, 1, brm[-1])))
    a_rows = [np.arange(600), np.sort(rng.choice(nb, 50, replace=False)), np.sort(rng.choice(nb, 10, replace=False)),
              np.array([3, 500, 699]), np.array([7])]
    arm = np.cumsum([0] + [len(r) for r in a_rows])
    A = g.CSR(len(a_rows), nb, torch.tensor(arm), torch.tensor(np.concatenate(a_rows), dtype=torch.int32),
              torch.tensor(rng.uniform(-1, 1, arm[-1])))
    for vt in (torch.float64, torch.float32):
        got = gpu_spgemm(A, B, value_dtype=vt, offset_dtype=torch.int64, timing=True)
        assert "num_hub" in got[3]["kernels"], got[3]["kernels"]
        assert_parity(oracle_mod, A, B, got, value_dtype=vt)


@pytest.mark.parametrize("kind", ["hub", "dense_window", "short_b_rows", "C2"])
def test_deterministic_mode(oracle_mod, kind):
    """opts.deterministic (handle-selected variant): random values, tiers
    that add with atomics by default; two runs are bitwise equal and within the parity bound."""
    if kind == "hub":
        A, B = _long_rows(31)  # k = 200K: the CTA bit-vector tier
    elif kind == "dense_window":
        A = g.random_csr(24, 300, 100, seed=41, empty_row_frac=0.0)
        B = g.random_csr(300, 20000, 300, seed=42, empty_row_frac=0.0)  # k <= 25.6K: windowed
    elif kind == "short_b_rows":
        A = g.random_csr(400, 300, 40, seed=43)
        B = g.random_csr(300, 500, 2, seed=44)  # ~1 entry per B row: sub-warp groups otherwise
    else:
        A, B = g.config("C2", size=14, values="random")
    runs = [gpu_spgemm(A, B, deterministic=True) for _ in range(2)]
    assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])
    assert np.array_equal(runs[0][2].view(np.int64), runs[1][2].view(np.int64)), "values differ between runs"
    # products rounded before the add (-fmad=false) and added in A-entry order, as the
    # oracle does: the deterministic result is the oracle's bit for bit
    assert_parity(oracle_mod, A, B, runs[0], exact=True)


def test_deterministic_needs_strict_b():
    from paper_2103_11991_b200._ffi import KKError, KK_ERR_UNSUPPORTED_TYPE

    A = g.random_csr(30, 25, 10, seed=51, sorted_rows=False)
    B = g.random_csr(25, 45, 10, seed=52, sorted_rows=False, duplicates=True)
    with pytest.raises(KKError) as e:
        gpu_spgemm(A, B, deterministic=True)
    assert e.value.status == KK_ERR_UNSUPPORTED_TYPE
