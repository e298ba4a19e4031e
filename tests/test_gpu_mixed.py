"""One product whose rows land in every symbolic and numeric tier at once (tiny rows, bit-vector
windows of every width including 128K/192K bits, speculative hash tables that finish and that
retry, the CTA dense tiers, kept and unkept patterns), on the device path and the host-buffer
path with several block plans; every case against the oracle.  The tiers share the handle's
workspace, bins and pattern pool in one call, which the per-tier tests do not exercise."""
import numpy as np
import pytest
import torch

from workloads import generators as g

from .helpers import assert_parity, gpu_spgemm

pytestmark = pytest.mark.gpu

K = 1_000_000


def _rows_to_csr(rows, ncols, rng):
    rm = np.cumsum([0] + [len(r) for r in rows])
    ent = np.concatenate([np.asarray(r, dtype=np.int64) for r in rows]) if rm[-1] else np.zeros(0, np.int64)
    return g.CSR(len(rows), ncols, torch.tensor(rm), torch.tensor(ent, dtype=torch.int32),
                 torch.tensor(rng.uniform(-1, 1, rm[-1])))


def _mixed(seed):
    rng = np.random.default_rng(seed)
    b_rows, groups = [], {}

    def add(name, rows):
        groups[name] = (len(b_rows), len(b_rows) + len(rows))
        b_rows.extend(rows)

    # B row groups (sorted, distinct columns)
    add("band", [np.sort(rng.choice(np.arange(max(0, c - 3000), min(K, c + 3000)), 20, replace=False))
                 for c in np.linspace(1000, 60000, 300).astype(int)])
    add("wide", [np.sort(rng.choice(np.arange(max(0, c - 60000), min(K, c + 60000)), 30, replace=False))
                 for c in np.linspace(200000, 400000, 200).astype(int)])
    base = np.sort(rng.choice(K, 30, replace=False))
    clus = []
    for _ in range(200):
        r = base.copy()
        r[rng.choice(30, 2, replace=False)] = rng.choice(K, 2, replace=False)
        clus.append(np.unique(r))
    add("clus", clus)
    add("rand", [np.sort(rng.choice(K, 30, replace=False)) for _ in range(200)])
    add("long", [np.sort(rng.choice(K, 3000, replace=False)) for _ in range(40)])
    add("short", [np.sort(rng.choice(K, 8, replace=False)) for _ in range(100)])
    B = _rows_to_csr(b_rows, K, rng)

    def pick(name, n, size):
        lo, hi = groups[name]
        return [np.sort(lo + rng.choice(hi - lo, size, replace=False)) for _ in range(n)]

    a_rows = []
    a_rows += pick("band", 300, 12)          # window bins
    a_rows += pick("wide", 150, 10)          # 128K / 192K-bit windows
    a_rows += pick("clus", 150, 40)          # speculative tables that finish
    a_rows += pick("rand", 150, 40)          # speculative tables that retry
    a_rows += pick("long", 20, 30)           # CTA dense tiers (rows of ~85K outputs)
    a_rows += pick("short", 200, 2)          # tiny rows (<= 16 products)
    a_rows += [np.zeros(0, dtype=np.int64) for _ in range(30)]  # empty rows
    order = rng.permutation(len(a_rows))    # interleave the row types
    A = _rows_to_csr([a_rows[i] for i in order], B.nrows, rng)
    return A, B


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("ot", [torch.int32, torch.int64])
def test_mixed_tiers_device(oracle_mod, seed, ot):
    A, B = _mixed(seed)
    got = gpu_spgemm(A, B, offset_dtype=ot, timing=True)
    assert_parity(oracle_mod, A, B, got)
    st = got[3]
    used = [b for b, n in enumerate(st["symbolic_bin_rows"]) if n > 0]
    assert len(used) >= 5, st["symbolic_bin_rows"]
    names = " ".join(st["kernels"])
    for k in ("sym_rows_spec", "sym_rows_retry", "sym_tiny", "num_tiny"):
        assert k in names, (k, names)


@pytest.mark.parametrize("blocks", [None, 3, 7])
def test_mixed_tiers_host(oracle_mod, blocks):
    from paper_2103_11991_b200 import CsrMatrix, SpGEMM

    A, B = _mixed(3)

    def host(M):
        return CsrMatrix(M.nrows, M.ncols, M.row_map.to(torch.int64).pin_memory(), M.entries.pin_memory(),
                         M.values.pin_memory())

    h = SpGEMM()
    C = h.multiply_host(host(A), host(B), blocks=blocks)
    got = (C.row_map.numpy().astype(np.int64), C.entries.numpy().copy(), C.values.numpy().copy())
    assert_parity(oracle_mod, A, B, got)
    h.close()
