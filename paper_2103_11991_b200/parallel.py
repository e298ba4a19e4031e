"""Row-sharded multi-GPU SpGEMM: one process per GPU, torch.distributed.

C(i,:) depends only on A(i,:) and all of B (Eq. 1), so rows of A
are split into contiguous, flop-balanced blocks; B is replicated with one broadcast
(NCCL over NVLink/NVSwitch); after the local symbolic phase the ranks all-gather their
nnz(C_p) so each knows the global offset O_p of its block of C (the layout of a
row-distributed Tpetra matrix).  The numeric phase is local.

Everything here is plumbing around the single-GPU C ABI (include/kk_spgemm.h): row
ranges, collectives and offsets.  The arithmetic of every step runs in
libkk_spgemm.so.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .spgemm import CsrMatrix, SpGEMM

_DT = [torch.int32, torch.int64, torch.float32, torch.float64]


def flop_balanced_cuts(F: Sequence[int], world: int, align: int = 1) -> List[int]:
    """Split points r_0=0 <= r_1 <= ... <= r_P=m of rows, from the exclusive prefix F
    (length m+1) of per-row multiply-adds: r_p is the first row whose prefix reaches
    p*F[m]/P, rounded to a multiple of `align` (whole 3-dof nodes of the
    block stencil C5: align=3)."""
    import numpy as np

    F = np.asarray(F, dtype=np.int64)
    m = len(F) - 1
    total = int(F[m]) if m >= 0 else 0
    cuts = [0]
    for p in range(1, world):
        c = int(np.searchsorted(F, (total * p) // world, side="left"))
        if align > 1:
            c = int(round(c / align)) * align
        cuts.append(c)
    cuts.append(max(m, 0))
    out = [min(max(c, 0), max(m, 0)) for c in cuts]
    for i in range(1, len(out)):
        out[i] = max(out[i], out[i - 1])
    return out


def global_offsets(nnz_per_rank: Sequence[int]) -> List[int]:
    """Exclusive prefix of the gathered per-rank nnz: O_p = sum_{q<p} nnz_q."""
    out, run = [], 0
    for v in nnz_per_rank:
        out.append(run)
        run += int(v)
    return out


def galerkin_slab_cuts(n: int, agg: int, world: int) -> Tuple[List[int], List[int]]:
    """z-slab partition of the C3 Galerkin product on an n^3 grid with agg^3 aggregates
    (SURVEY §8e "C3 at P > 1"): slab p holds whole aggregate planes, i.e. fine z-planes
    [agg*z_p, agg*z_{p+1}) and coarse z-planes [z_p, z_{p+1}).  With lexicographic
    numbering (z slowest) both are contiguous row ranges: fine rows [n*n*agg*z_p, ...) of A
    and T, coarse rows [nc*nc*z_p, ...) of R and Ac.  R's row block p references only fine
    rows of slab p, so R_p * T_p needs no second exchange.  Returns (fine_cuts, coarse_cuts)."""
    nc = (n + agg - 1) // agg
    zc = [(nc * p) // world for p in range(world + 1)]
    fine = [min(n, agg * z) * n * n for z in zc]
    coarse = [z * nc * nc for z in zc]
    return fine, coarse


def slice_rows(M: CsrMatrix, r0: int, r1: int) -> CsrMatrix:
    """Rows [r0, r1) of M as a CSR matrix of its own (row map rebased to 0; entries and
    values are views, no copy)."""
    rm = M.row_map
    s = int(rm[r0].item())
    e = int(rm[r1].item())
    sub_rm = (rm[r0:r1 + 1] - rm[r0]).contiguous()
    vals = M.values[s:e] if M.values is not None else None
    return CsrMatrix(r1 - r0, M.ncols, sub_rm, M.entries[s:e], vals)


def shift_columns(M: CsrMatrix, c0: int, ncols: int) -> CsrMatrix:
    """The same rows with column indices shifted by -c0 into [0, ncols) (a row block whose
    columns all lie in [c0, c0 + ncols), e.g. R_p of the slab-partitioned Galerkin product)."""
    return CsrMatrix(M.nrows, ncols, M.row_map, (M.entries - c0).to(torch.int32), M.values)


def _bcast(t: torch.Tensor, src: int, group, async_op: bool = False):
    """Broadcast in place.  NCCL takes device tensors; gloo (CPU tests, or several ranks
    sharing one GPU in the single-GPU tests) is staged through host memory."""
    if dist.get_backend(group) == "nccl" or t.device.type == "cpu":
        return dist.broadcast(t, src, group=group, async_op=async_op)
    h = t.cpu()
    dist.broadcast(h, src, group=group)
    t.copy_(h)
    return None


def broadcast_csr(M: Optional[CsrMatrix], src: int = 0, device=None, group=None, async_values: bool = False):
    """Replicate a CSR matrix from rank `src` to every rank: a small header broadcast,
    then row map + entries (the pattern: symbolic can start once they have arrived), then
    the values.  async_values=True returns (M, work) with the values' broadcast still in
    flight (NCCL, its own stream): the caller overlaps it with the symbolic phase, which
    reads only the pattern, and waits on `work` before the numeric phase."""
    rank = dist.get_rank(group)
    dev = torch.device(device) if device is not None else (
        M.row_map.device if M is not None else torch.device("cpu"))
    hdr = torch.zeros(6, dtype=torch.int64, device=dev)
    if rank == src:
        hdr[0], hdr[1], hdr[2] = M.nrows, M.ncols, M.nnz
        hdr[3] = _DT.index(M.row_map.dtype)
        hdr[4] = _DT.index(M.values.dtype) if M.values is not None else -1
    _bcast(hdr, src, group)
    nrows, ncols, nnz, od, vd = (int(x) for x in hdr[:5].tolist())
    if rank == src:
        rm, ent = M.row_map.to(dev).contiguous(), M.entries.to(dev).contiguous()
        val = M.values.to(dev).contiguous() if M.values is not None else None
    else:
        rm = torch.empty(nrows + 1, dtype=_DT[od], device=dev)
        ent = torch.empty(nnz, dtype=torch.int32, device=dev)
        val = torch.empty(nnz, dtype=_DT[vd], device=dev) if vd >= 0 else None
    _bcast(rm, src, group)
    work = None
    if nnz:
        _bcast(ent, src, group)
        if val is not None:
            work = _bcast(val, src, group, async_op=async_values)
    out = CsrMatrix(nrows, ncols, rm, ent, val)
    return (out, work) if async_values else out


def allgather_row_map_total(c_row_map: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather nnz(C_p) = c_row_map[m_p] straight from the device row map the symbolic
    scan kernel wrote (the all-gather's send buffer is that last entry: no host round trip
    and no host-built tensor).  Returns the per-rank counts as an int64 device tensor."""
    world = dist.get_world_size(group)
    mine = c_row_map[-1:].to(torch.int64)
    if dist.get_backend(group) == "nccl":
        allv = torch.empty(world, dtype=torch.int64, device=c_row_map.device)
        dist.all_gather_into_tensor(allv, mine, group=group)
        return allv
    parts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, mine.cpu(), group=group)
    return torch.cat(parts).to(c_row_map.device)


def allgather_nnz(nnz_local: int, device, group=None) -> List[int]:
    """All-gather one int64 nnz(C_p) per rank (host values)."""
    world = dist.get_world_size(group)
    mine = torch.tensor([int(nnz_local)], dtype=torch.int64, device=device)
    if dist.get_backend(group) == "nccl":
        allv = torch.zeros(world, dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(allv, mine, group=group)
        return [int(x) for x in allv.tolist()]
    parts = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    return [int(p.item()) for p in parts]


def _all_to_all_var(send: torch.Tensor, send_counts: List[int], group=None) -> Tuple[torch.Tensor, List[int]]:
    """Variable-size all-to-all of a 1-D tensor: send_counts[q] elements go to rank q.
    NCCL: all_to_all_single; gloo (CPU tests): pairwise isend/irecv."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = send.device
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty(world, dtype=torch.int64, device=dev)
    if dist.get_backend(group) == "nccl":
        dist.all_to_all_single(rc, sc, group=group)
    else:
        allc = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allc, sc.cpu(), group=group)
        rc = torch.stack([allc[q][rank] for q in range(world)]).to(dev)
    recv_counts = [int(x) for x in rc.tolist()]
    recv = torch.empty(sum(recv_counts), dtype=send.dtype, device=dev)
    if dist.get_backend(group) == "nccl":
        dist.all_to_all_single(recv, send, output_split_sizes=recv_counts, input_split_sizes=send_counts, group=group)
    else:
        so = [0]
        for c in send_counts:
            so.append(so[-1] + c)
        ro = [0]
        for c in recv_counts:
            ro.append(ro[-1] + c)
        reqs = []
        for q in range(world):
            if q == rank:
                recv[ro[q]:ro[q + 1]] = send[so[q]:so[q + 1]]
                continue
            if send_counts[q]:
                reqs.append(dist.isend(send[so[q]:so[q + 1]].contiguous(), q, group=group))
            if recv_counts[q]:
                buf = torch.empty(recv_counts[q], dtype=send.dtype, device=dev)
                reqs.append((dist.irecv(buf, q, group=group), buf, ro[q]))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                recv[r[2]:r[2] + len(r[1])] = r[1]
            else:
                r.wait()
    return recv, recv_counts


def halo_exchange_b(A_local: CsrMatrix, B_local: CsrMatrix, b_cuts: Sequence[int], group=None) -> CsrMatrix:
    """Halo-only B exchange: B is row-distributed
    (rank q owns rows [b_cuts[q], b_cuts[q+1]) as B_local, row map rebased to 0); each rank
    fetches only the B rows its A block references (the distinct column indices of A_local)
    instead of a broadcast of all of B.  Returns a B of full shape (n x k) whose row map has
    the fetched rows and empty rows elsewhere, so A_local's column indices need no remap and
    the single-GPU SpGEMM applies unchanged.  Collectives: two variable all-to-alls for the
    requests (row ids) and one each for the replies' row lengths, entries and values."""
    world = dist.get_world_size(group)
    dev = A_local.row_map.device
    n = int(b_cuts[-1])
    need = torch.unique(A_local.entries.to(torch.int64)) if A_local.nnz else torch.zeros(0, dtype=torch.int64,
                                                                                          device=dev)
    cuts_t = torch.tensor(list(b_cuts), dtype=torch.int64, device=dev)
    owner = torch.searchsorted(cuts_t, need, right=True) - 1
    req_counts = [int(x) for x in torch.bincount(owner, minlength=world).tolist()] if need.numel() else [0] * world
    # requests: row ids (sorted, grouped by owner since `need` is sorted and cuts increase)
    got_req, got_counts = _all_to_all_var(need, req_counts, group)
    # serve: rows got_req (global ids in my range) -> lengths, entries, values
    rank = dist.get_rank(group)
    my0 = int(b_cuts[rank])
    loc = got_req - my0
    brm = B_local.row_map.to(torch.int64)
    lens = (brm[loc + 1] - brm[loc]) if loc.numel() else torch.zeros(0, dtype=torch.int64, device=dev)
    starts = brm[loc] if loc.numel() else torch.zeros(0, dtype=torch.int64, device=dev)
    # gather the entries of the requested rows (in request order)
    if lens.numel():
        rows_rep = torch.repeat_interleave(torch.arange(lens.numel(), device=dev), lens)
        offs_in = torch.cumsum(lens, 0) - lens
        idx = starts[rows_rep] + (torch.arange(rows_rep.numel(), device=dev) - offs_in[rows_rep])
        ent_out = B_local.entries[idx]
        val_out = B_local.values[idx]
    else:
        ent_out = torch.zeros(0, dtype=torch.int32, device=dev)
        val_out = torch.zeros(0, dtype=B_local.values.dtype, device=dev)
    # reply sizes per requesting rank
    ro = [0]
    for c in got_counts:
        ro.append(ro[-1] + c)
    ent_counts = [int(lens[ro[q]:ro[q + 1]].sum()) for q in range(world)]
    rlens, _ = _all_to_all_var(lens, got_counts, group)
    rent, _ = _all_to_all_var(ent_out, ent_counts, group)
    rval, _ = _all_to_all_var(val_out, ent_counts, group)
    # assemble: full-shape row map with the fetched rows (need order = reply order)
    rowlen = torch.zeros(n, dtype=torch.int64, device=dev)
    if need.numel():
        rowlen[need] = rlens
    rm = torch.zeros(n + 1, dtype=B_local.row_map.dtype, device=dev)
    rm[1:] = torch.cumsum(rowlen, 0).to(rm.dtype)
    return CsrMatrix(n, B_local.ncols, rm, rent.to(torch.int32), rval)


class ShardedSpGEMM:
    """C = A*B with rows of A block-distributed over the ranks of `group`.

    Each rank passes its local row block A_p (rows [r_p, r_{p+1}) of A) and the full B.
    Returns (C_p, O_p, nnz_total): the local rows of C and their global entry offset."""

    def __init__(self, device=None, group=None, **opts):
        self.group = group
        self.h = SpGEMM(device=device, **opts)

    def __call__(self, A_local: CsrMatrix, B: CsrMatrix, values_work=None) -> Tuple[CsrMatrix, int, int]:
        """values_work: the in-flight broadcast of B's values (broadcast_csr(...,
        async_values=True)); the symbolic phase reads only B's pattern, so the wait is placed
        just before the numeric phase."""
        rm, nnz = self.h.symbolic(A_local, B)
        counts = allgather_row_map_total(rm, self.group).tolist()
        offs = global_offsets(counts)
        if values_work is not None:
            values_work.wait()
        ent, val = self.h.numeric(A_local, B, rm, nnz=nnz)
        rank = dist.get_rank(self.group)
        return CsrMatrix(A_local.nrows, B.ncols, rm, ent, val), offs[rank], sum(counts)

    def close(self):
        self.h.close()
