"""Seeded synthetic CSR generators (input construction only; no SpGEMM arithmetic).

Every generator is a deterministic function of its parameters and seed, written
in integer / elementwise torch ops so it yields bit-identical matrices on CPU
(oracle side) and on CUDA (product side).  Random numbers come from a
counter-based hash (splitmix64) of (seed, row, col, ...), so they are identical
under any device or sharding.

Workload recipes (SURVEY.md §8 size table and readings R12-R15):

* stencil Laplacians ("diagonal value = stencil length - 1,
  off-diagonals = -1"), Dirichlet truncation at the box skin, node numbering
  lexicographic with x fastest;
* 3x3x3 aggregation prolongator P (entries 1) and R = P^T;
* RMAT / Graph500 Kronecker graph, directed, self loops dropped,
  duplicates merged, unit values;
* 27-point block stencil with 3 dof per node, values L27 (x) M;
* small random CSR for brute-force tests, with options for unsorted rows,
  duplicate columns, explicit zeros and empty rows.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

# ---------------------------------------------------------------------------
# counter-based random numbers (splitmix64), identical on CPU and CUDA
# ---------------------------------------------------------------------------


def _s64(x: int) -> int:
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= (1 << 63) else x


_GOLD = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (two's-complement wrap-around)."""
    z = x + _GOLD
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def _key(*parts) -> torch.Tensor:
    h = None
    for p in parts:
        if not torch.is_tensor(p):
            p = torch.tensor(_s64(int(p)), dtype=torch.int64)
        h = splitmix64(p if h is None else (h ^ p))
    return h


def uniform01(*parts) -> torch.Tensor:
    """U[0,1) from the top 53 bits of a splitmix64 chain over `parts`."""
    return _lsr(_key(*parts), 11).to(torch.float64) * (1.0 / 9007199254740992.0)


def random_value(seed: int, rows: torch.Tensor, cols: torch.Tensor) -> torch.Tensor:
    """u(seed,row,col) in [-1,1): the stateless value recipe of SURVEY R12."""
    return 2.0 * uniform01(int(seed) * 0x5851F42D + 7, rows.to(torch.int64), cols.to(torch.int64)) - 1.0


# ---------------------------------------------------------------------------
# container
# ---------------------------------------------------------------------------


@dataclass
class CSR:
    """Compressed row storage (§2): row_map (int64, nrows+1),
    entries (int32 column indices), values (float64 or float32)."""

    nrows: int
    ncols: int
    row_map: torch.Tensor
    entries: torch.Tensor
    values: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.entries.numel())

    @property
    def device(self):
        return self.entries.device

    def to(self, device=None, value_dtype=None, offset_dtype=None, non_blocking=False) -> "CSR":
        rm = self.row_map
        vals = self.values
        if offset_dtype is not None:
            rm = rm.to(offset_dtype)
        if value_dtype is not None:
            vals = vals.to(value_dtype)
        if device is not None:
            rm = rm.to(device, non_blocking=non_blocking)
            vals = vals.to(device, non_blocking=non_blocking)
            ent = self.entries.to(device, non_blocking=non_blocking)
        else:
            ent = self.entries
        return CSR(self.nrows, self.ncols, rm, ent, vals)

    def clone(self) -> "CSR":
        return CSR(self.nrows, self.ncols, self.row_map.clone(), self.entries.clone(), self.values.clone())

    def row_lengths(self) -> torch.Tensor:
        rm = self.row_map.to(torch.int64)
        return rm[1:] - rm[:-1]

    def to_dense(self) -> torch.Tensor:
        """Dense fp64 copy with duplicates summed (tiny matrices only)."""
        d = torch.zeros(self.nrows, self.ncols, dtype=torch.float64)
        rows = torch.repeat_interleave(torch.arange(self.nrows), self.row_lengths().cpu())
        d.index_put_((rows, self.entries.cpu().to(torch.int64)), self.values.cpu().to(torch.float64), accumulate=True)
        return d


def _from_rows(nrows: int, ncols: int, rows: torch.Tensor, counts: torch.Tensor,
               entries: torch.Tensor, values: torch.Tensor) -> CSR:
    """Assemble a CSR of `nrows` rows where only `rows` (sorted) are non-empty."""
    dev = entries.device
    lens = torch.zeros(nrows, dtype=torch.int64, device=dev)
    lens[rows] = counts.to(torch.int64)
    row_map = torch.zeros(nrows + 1, dtype=torch.int64, device=dev)
    row_map[1:] = torch.cumsum(lens, 0)
    return CSR(nrows, ncols, row_map, entries.to(torch.int32).contiguous(), values.contiguous())


# ---------------------------------------------------------------------------
# stencils
# ---------------------------------------------------------------------------


def _sorted_offsets(offsets: Sequence[Sequence[int]], dims: Sequence[int]):
    strides = [1]
    for d in dims[:-1]:
        strides.append(strides[-1] * d)
    lin = [sum(o[a] * strides[a] for a in range(len(dims))) for o in offsets]
    order = sorted(range(len(offsets)), key=lambda t: lin[t])
    return [tuple(offsets[t]) for t in order], strides


def stencil_laplacian(dims: Sequence[int], offsets: Sequence[Sequence[int]], rows: Optional[torch.Tensor] = None,
                      values: str = "int", seed: int = 1, device="cpu") -> CSR:
    """Stencil Laplacian on a box with Dirichlet truncation.

    diag = (#stencil points - 1), off-diagonal = -1; `values="random"`
    replaces every stored value by u(seed,row,col).  `rows` selects a
    sorted subset of rows to materialise (other rows empty) for sampled parity.
    """
    dims = list(dims)
    offs, strides = _sorted_offsets(offsets, dims)
    N = math.prod(dims)
    if rows is None:
        ids = torch.arange(N, dtype=torch.int64, device=device)
    else:
        ids = rows.to(device=device, dtype=torch.int64)
    coord = []
    rem = ids
    for a, d in enumerate(dims):
        coord.append(rem % d)
        rem = rem // d
    S = len(offs)
    cols = torch.empty(ids.numel(), S, dtype=torch.int64, device=device)
    valid = torch.ones(ids.numel(), S, dtype=torch.bool, device=device)
    diag = torch.zeros(ids.numel(), S, dtype=torch.bool, device=device)
    for s, o in enumerate(offs):
        lin = 0
        for a in range(len(dims)):
            c = coord[a] + o[a]
            valid[:, s] &= (c >= 0) & (c < dims[a])
            lin += o[a] * strides[a]
        cols[:, s] = ids + lin
        diag[:, s] = all(v == 0 for v in o)
    counts = valid.sum(1)
    rr = ids.unsqueeze(1).expand(-1, S)[valid]
    cc = cols[valid]
    if values == "int":
        vals = torch.where(diag[valid], torch.tensor(float(S - 1), dtype=torch.float64, device=device),
                           torch.tensor(-1.0, dtype=torch.float64, device=device))
    elif values == "random":
        vals = random_value(seed, rr, cc)
    else:
        raise ValueError(values)
    return _from_rows(N, N, ids, counts, cc, vals)


def _box_offsets(ndim: int, radius: int = 1, kind: str = "box"):
    out = []
    for o in itertools.product(range(-radius, radius + 1), repeat=ndim):
        if kind == "box" or sum(abs(v) for v in o) <= radius:
            out.append(o)
    return out


def laplacian_2d_5pt(n: int, **kw) -> CSR:
    """2D 5-point Laplacian on an n x n grid (BASELINE.json configs[0])."""
    return stencil_laplacian((n, n), _box_offsets(2, 1, "cross"), **kw)


def laplacian_3d_7pt(n: int, **kw) -> CSR:
    """3D 7-point Laplacian on n^3 (BASELINE.json configs[2])."""
    return stencil_laplacian((n, n, n), _box_offsets(3, 1, "cross"), **kw)


def laplacian_3d_27pt(n: int, **kw) -> CSR:
    """3D 27-point Laplacian on n^3 (BASELINE.json configs[1])."""
    return stencil_laplacian((n, n, n), _box_offsets(3, 1, "box"), **kw)


_BLOCK_M = ((2.0, 1.0, 1.0), (1.0, 2.0, 1.0), (1.0, 1.0, 2.0))


def block_stencil_27pt(n: int, dof: int = 3, rows: Optional[torch.Tensor] = None, values: str = "int",
                       seed: int = 1, device="cpu") -> CSR:
    """27-point block stencil with `dof` unknowns per node (BASELINE.json configs[4]).

    Row = dof*node + d (node lexicographic, x fastest); pattern L27 (x) ones(dof,dof);
    integer values L27[node,nb] * M[d,d'] with M = [[2,1,1],[1,2,1],[1,1,2]].
    """
    assert dof == 3 or values == "random", "integer block values defined for dof=3"
    dims = (n, n, n)
    offs, strides = _sorted_offsets(_box_offsets(3, 1, "box"), dims)
    Nn = n ** 3
    if rows is None:
        rid = torch.arange(Nn * dof, dtype=torch.int64, device=device)
    else:
        rid = rows.to(device=device, dtype=torch.int64)
    node = rid // dof
    d = rid % dof
    coord = [node % n, (node // n) % n, node // (n * n)]
    S = len(offs)
    nb = torch.empty(rid.numel(), S, dtype=torch.int64, device=device)
    valid = torch.ones(rid.numel(), S, dtype=torch.bool, device=device)
    lval = torch.empty(rid.numel(), S, dtype=torch.float64, device=device)
    for s, o in enumerate(offs):
        for a in range(3):
            c = coord[a] + o[a]
            valid[:, s] &= (c >= 0) & (c < n)
        nb[:, s] = node + o[0] * strides[0] + o[1] * strides[1] + o[2] * strides[2]
        lval[:, s] = float(S - 1) if o == (0, 0, 0) else -1.0
    dp = torch.arange(dof, dtype=torch.int64, device=device)
    cols = (nb.unsqueeze(2) * dof + dp.view(1, 1, dof))  # [R, S, dof]
    v3 = valid.unsqueeze(2).expand(-1, -1, dof)
    counts = v3.reshape(rid.numel(), -1).sum(1)
    cc = cols[v3]
    if values == "int":
        M = torch.tensor(_BLOCK_M, dtype=torch.float64, device=device)
        mrow = M[d]  # [R, dof]
        vv = lval.unsqueeze(2) * mrow.unsqueeze(1)
        vals = vv[v3]
    else:
        rr = rid.view(-1, 1, 1).expand(-1, S, dof)[v3]
        vals = random_value(seed, rr, cc)
    return _from_rows(Nn * dof, Nn * dof, rid, counts, cc, vals)


# ---------------------------------------------------------------------------
# multigrid aggregation
# ---------------------------------------------------------------------------


def aggregation_prolongator(n: int, agg: int = 3, values: str = "int", seed: int = 1, device="cpu") -> CSR:
    """Unsmoothed aggregation prolongator on an n^3 grid with agg^3 aggregates.

    P[i, agg(i)] = 1 with agg(i) = (x//agg) + nc*((y//agg) + nc*(z//agg)),
    nc = ceil(n/agg) (128 -> 43 aggregates per axis, the last 2 wide).
    """
    N = n ** 3
    nc = -(-n // agg)
    ids = torch.arange(N, dtype=torch.int64, device=device)
    x, y, z = ids % n, (ids // n) % n, ids // (n * n)
    col = (x // agg) + nc * ((y // agg) + nc * (z // agg))
    if values == "int":
        vals = torch.ones(N, dtype=torch.float64, device=device)
    else:
        vals = random_value(seed, ids, col)
    row_map = torch.arange(N + 1, dtype=torch.int64, device=device)
    return CSR(N, nc ** 3, row_map, col.to(torch.int32), vals)


def transpose(A: CSR) -> CSR:
    """Explicit transpose (input construction for R = P^T; rows come out sorted)."""
    dev = A.entries.device
    lens = A.row_lengths()
    rows = torch.repeat_interleave(torch.arange(A.nrows, dtype=torch.int64, device=dev), lens)
    key = A.entries.to(torch.int64) * max(A.nrows, 1) + rows
    order = torch.argsort(key, stable=True)
    cols_t = rows[order]
    rows_t = A.entries.to(torch.int64)[order]
    counts = torch.bincount(rows_t, minlength=A.ncols)
    row_map = torch.zeros(A.ncols + 1, dtype=torch.int64, device=dev)
    row_map[1:] = torch.cumsum(counts, 0)
    return CSR(A.ncols, A.nrows, row_map, cols_t.to(torch.int32), A.values[order].contiguous())


def transpose_pattern_ones(P: CSR) -> CSR:
    """R = P^T."""
    return transpose(P)


# ---------------------------------------------------------------------------
# RMAT (Graph500 Kronecker)
# ---------------------------------------------------------------------------


def rmat(scale: int = 20, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
         d: float = 0.05, seed: int = 1, symmetrize: bool = False, values: str = "int", device="cpu") -> CSR:
    """RMAT graph adjacency: 2^scale vertices, edge_factor*2^scale drawn edges,
    Graph500 bitwise Kronecker levels, random label permutation, self loops dropped,
    duplicates merged, directed unless `symmetrize`, unit values."""
    N = 1 << scale
    E = edge_factor * N
    e = torch.arange(E, dtype=torch.int64, device=device)
    src = torch.zeros(E, dtype=torch.int64, device=device)
    dst = torch.zeros(E, dtype=torch.int64, device=device)
    ab = a + b
    c_norm = c / (c + d)
    a_norm = a / (a + b)
    for lev in range(scale):
        u = uniform01(seed, e, 2 * lev)
        v = uniform01(seed, e, 2 * lev + 1)
        ii = u > ab
        jj = torch.where(ii, v > c_norm, v > a_norm)
        src |= ii.to(torch.int64) << lev
        dst |= jj.to(torch.int64) << lev
    # random vertex relabelling: rank of (hash, vertex) keys
    verts = torch.arange(N, dtype=torch.int64, device=device)
    hk = (_lsr(_key(seed + 0x1234567, verts), 1 + scale) << scale) | verts
    perm = torch.argsort(hk)
    label = torch.empty(N, dtype=torch.int64, device=device)
    label[perm] = verts
    src = label[src]
    dst = label[dst]
    if symmetrize:
        src, dst = torch.cat([src, dst]), torch.cat([dst, src])
    keep = src != dst
    key = torch.unique(src[keep] * N + dst[keep], sorted=True)
    r = key // N
    cidx = key % N
    counts = torch.bincount(r, minlength=N)
    row_map = torch.zeros(N + 1, dtype=torch.int64, device=device)
    row_map[1:] = torch.cumsum(counts, 0)
    if values == "int":
        vals = torch.ones(key.numel(), dtype=torch.float64, device=device)
    else:
        vals = random_value(seed, r, cidx)
    return CSR(N, N, row_map, cidx.to(torch.int32), vals)


# ---------------------------------------------------------------------------
# small random matrices (brute-force tests)
# ---------------------------------------------------------------------------


def random_csr(m: int, n: int, max_row_nnz: int, seed: int = 1, sorted_rows: bool = True,
               duplicates: bool = False, explicit_zeros: bool = False, empty_row_frac: float = 0.1,
               integer_values: bool = False, device="cpu") -> CSR:
    """Random m x n CSR. Row lengths uniform in [0, max_row_nnz]; a fraction of rows forced
    empty; optional unsorted rows, duplicate columns and explicit stored zeros."""
    ri = torch.arange(m, dtype=torch.int64)
    lens = (uniform01(seed, ri, 11) * (max_row_nnz + 1)).floor().to(torch.int64).clamp(max=max_row_nnz)
    lens = torch.where(uniform01(seed, ri, 12) < empty_row_frac, torch.zeros_like(lens), lens)
    if n == 0:
        lens.zero_()
    if not duplicates:
        lens = lens.clamp(max=n)
    nnz = int(lens.sum())
    rows = torch.repeat_interleave(ri, lens)
    pos = torch.arange(nnz, dtype=torch.int64)
    if duplicates:
        cols = (uniform01(seed, pos, 13) * n).floor().to(torch.int64).clamp(max=max(n - 1, 0))
    else:
        # distinct columns per row: rank of hashed keys within each row
        cols = torch.empty(nnz, dtype=torch.int64)
        start = 0
        for i in range(m):
            L = int(lens[i])
            if L:
                sc = torch.argsort(uniform01(seed, torch.full((n,), i, dtype=torch.int64), torch.arange(n), 14))[:L]
                cols[start:start + L] = sc
            start += L
    if sorted_rows:
        order = torch.argsort(rows * max(n, 1) + cols, stable=True)
    else:
        order = torch.argsort(rows * 4294967296 + _lsr(_key(seed, pos, 15), 33), stable=True)
    rows, cols = rows[order], cols[order]
    if integer_values:
        vals = (uniform01(seed, rows, cols, pos, 16) * 9).floor() - 4.0
    else:
        vals = random_value(seed, rows, cols * 7 + pos)
    if explicit_zeros:
        z = uniform01(seed, pos, 17) < 0.15
        vals = torch.where(z, torch.zeros_like(vals), vals)
    row_map = torch.zeros(m + 1, dtype=torch.int64)
    row_map[1:] = torch.cumsum(lens, 0)
    return CSR(m, n, row_map.to(device), cols.to(torch.int32).to(device), vals.to(device))


def random_rows_csr(m: int, k: int, per_row: int, seed: int = 1, device="cpu") -> CSR:
    """m x k CSR with `per_row` uniformly random columns in every row (vectorised; repeated
    columns are kept as unmerged entries, rows sorted), values u in [-1, 1): the paper's
    SpAdd test matrices ("each have 30 randomized entries per row")."""
    nnz = m * per_row
    pos = torch.arange(nnz, dtype=torch.int64)
    rows = pos // max(per_row, 1)
    cols = (uniform01(seed, pos, 31) * k).floor().to(torch.int64).clamp(max=max(k - 1, 0))
    order = torch.argsort(rows * max(k, 1) + cols)
    rows, cols = rows[order], cols[order]
    vals = random_value(seed, rows, cols * 7 + pos)
    row_map = torch.arange(0, nnz + 1, max(per_row, 1), dtype=torch.int64)[: m + 1]
    return CSR(m, k, row_map.to(device), cols.to(torch.int32).to(device), vals.to(device))


# ---------------------------------------------------------------------------
# named workloads (BASELINE.json configs)
# ---------------------------------------------------------------------------

CONFIGS = {
    "C1": "A*A, 2D 5-point Laplacian 32x32 (1,024 rows)",
    "C2": "A*A, 3D 27-point Laplacian 100^3 (1M rows)",
    "C3": "Galerkin R*A*P, 3D 7-point Laplacian 128^3, 3x3x3 aggregation P, R=P^T",
    "C4": "A*A, RMAT scale 20, edge factor 16, directed",
    "C5": "A*A, 3D 27-point block stencil, 3 dof/node, 160^3",
    "C3J": "Jacobi-fused (I - w D^-1 A) P: smoothed-aggregation prolongator, 7-point 128^3, 3x3x3 aggregates",
}


def diagonal_inverse(A: CSR) -> torch.Tensor:
    """D^-1 of a square CSR matrix (input preparation for the Jacobi-fused product,
    PAPER.md:192: "D^-1 represents the inverse of the diagonal matrix of A"): 1 / A(i,i),
    summed over duplicate diagonal entries; rows without a stored diagonal get 0."""
    rm = A.row_map.to(torch.int64).cpu()
    rows = torch.repeat_interleave(torch.arange(A.nrows, dtype=torch.int64), rm[1:] - rm[:-1])
    ent = A.entries.cpu().to(torch.int64)
    d = torch.zeros(A.nrows, dtype=torch.float64)
    on = ent == rows
    d.index_add_(0, rows[on], A.values.cpu().to(torch.float64)[on])
    out = torch.where(d != 0, 1.0 / torch.where(d != 0, d, torch.ones_like(d)), torch.zeros_like(d))
    return out.to(A.values.device)


def config(name: str, size: Optional[int] = None, values: str = "int", seed: int = 1, device="cpu"):
    """Return the operands of a named configuration.

    C1/C2/C4/C5: (A, B) with B a separate copy of A (both operands count).
    C3: (A, P, R) for the two products T = A*P, Ac = R*T.
    `size` overrides the grid edge (or RMAT scale) for scaled-down test instances.
    """
    if name == "C1":
        A = laplacian_2d_5pt(size or 32, values=values, seed=seed, device=device)
    elif name == "C2":
        A = laplacian_3d_27pt(size or 100, values=values, seed=seed, device=device)
    elif name == "C3":
        n = size or 128
        A = laplacian_3d_7pt(n, values=values, seed=seed, device=device)
        P = aggregation_prolongator(n, values=values, seed=seed + 1, device=device)
        R = transpose(P)
        return A, P, R
    elif name == "C3J":
        # smoothed-aggregation prolongator: returns (A, P, dinv, omega)
        n = size or 128
        A = laplacian_3d_7pt(n, values=values, seed=seed, device=device)
        P = aggregation_prolongator(n, values=values, seed=seed + 1, device=device)
        return A, P, diagonal_inverse(A), 2.0 / 3.0
    elif name == "C4":
        A = rmat(scale=size or 20, edge_factor=16, seed=seed, values=values, device=device)
    elif name == "C5":
        A = block_stencil_27pt(size or 160, values=values, seed=seed, device=device)
    else:
        raise KeyError(name)
    return A, A.clone()
