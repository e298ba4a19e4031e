"""Multi-GPU host logic on CPU: the flop-balanced row split, global offsets,
and the collectives of paper_2103_11991_b200.parallel over gloo with world size 2.

The partition arithmetic is checked without any GPU: the oracle's product of each row
block, stitched with the all-gathered offsets, must equal the oracle's full product."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import generators as g


def test_flop_balanced_cuts_basic():
    from paper_2103_11991_b200.parallel import flop_balanced_cuts

    F = np.concatenate([[0], np.cumsum([5, 5, 5, 5, 100, 5, 5, 5])])
    cuts = flop_balanced_cuts(F, 2)
    assert cuts[0] == 0 and cuts[-1] == 8 and cuts == sorted(cuts)
    for world in (1, 2, 3, 8, 16):
        c = flop_balanced_cuts(F, world)
        assert len(c) == world + 1 and c[0] == 0 and c[-1] == 8 and c == sorted(c)
    assert flop_balanced_cuts(np.zeros(1, dtype=np.int64), 4) == [0, 0, 0, 0, 0]


def test_global_offsets():
    from paper_2103_11991_b200.parallel import global_offsets

    assert global_offsets([3, 0, 5, 2]) == [0, 3, 3, 8]
    assert global_offsets([]) == []


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_split_stitches_to_full_product(oracle_mod, world):
    """Oracle on each flop-balanced row block, stitched by global offsets == full oracle."""
    from paper_2103_11991_b200.parallel import flop_balanced_cuts, global_offsets

    A, B = g.config("C2", size=9, values="random")
    f, tot = oracle_mod.row_flops(A, B)
    F = np.concatenate([[0], np.cumsum(f)])
    cuts = flop_balanced_cuts(F, world)
    rm_full, ent_full, val_full, _ = oracle_mod.spgemm(A, B)
    rms, ents, vals, nnzs = [], [], [], []
    arm = A.row_map.numpy()
    for p in range(world):
        r0, r1 = cuts[p], cuts[p + 1]
        s, e = int(arm[r0]), int(arm[r1])
        Ap = g.CSR(r1 - r0, A.ncols, torch.tensor(arm[r0:r1 + 1] - s), A.entries[s:e], A.values[s:e])
        rm, ent, val, _ = oracle_mod.spgemm(Ap, B)
        rms.append(rm)
        ents.append(ent)
        vals.append(val)
        nnzs.append(int(rm[-1]))
    offs = global_offsets(nnzs)
    stitched = np.concatenate([[0]] + [rms[p][1:] + offs[p] for p in range(world)])
    assert np.array_equal(stitched, rm_full)
    assert np.array_equal(np.concatenate(ents), ent_full)
    assert np.array_equal(np.concatenate(vals), val_full)
    # balance: no block carries more than its share plus one row's work
    blk = [F[cuts[p + 1]] - F[cuts[p]] for p in range(world)]
    assert max(blk) <= tot / world + f.max()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_11991_b200.parallel import allgather_nnz, broadcast_csr, global_offsets
        from paper_2103_11991_b200.spgemm import CsrMatrix

        if rank == 0:
            A, _ = g.config("C1", size=6, values="random")
            M = CsrMatrix(A.nrows, A.ncols, A.row_map, A.entries, A.values)
        else:
            M = None
        R = broadcast_csr(M, src=0, device="cpu")
        counts = allgather_nnz(10 * rank + 7, "cpu")
        q.put((rank, R.nrows, R.ncols, R.row_map.tolist(), R.entries.tolist(), R.values.tolist(), counts,
               global_offsets(counts)))
    finally:
        dist.destroy_process_group()


def test_gloo_broadcast_and_allgather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    A, _ = g.config("C1", size=6, values="random")
    for r in res:
        assert r[1] == A.nrows and r[2] == A.ncols
        assert r[3] == A.row_map.tolist() and r[4] == A.entries.tolist() and r[5] == A.values.tolist()
        assert r[6] == [7, 17] and r[7] == [0, 7]


def _halo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2103_11991_b200.parallel import halo_exchange_b, slice_rows
        from paper_2103_11991_b200.spgemm import CsrMatrix

        A, B = g.config("C2", size=7, values="random")
        n = B.nrows
        cuts = [n * p // world for p in range(world + 1)]
        Bfull = CsrMatrix(B.nrows, B.ncols, B.row_map, B.entries, B.values)
        Af = CsrMatrix(A.nrows, A.ncols, A.row_map, A.entries, A.values)
        B_loc = slice_rows(Bfull, cuts[rank], cuts[rank + 1])
        A_loc = slice_rows(Af, cuts[rank], cuts[rank + 1])
        Bh = halo_exchange_b(A_loc, B_loc, cuts)
        # the product of the local block with the fetched rows equals the rows of A*B
        Ap = g.CSR(A_loc.nrows, A_loc.ncols, A_loc.row_map, A_loc.entries, A_loc.values)
        Bp = g.CSR(Bh.nrows, Bh.ncols, Bh.row_map, Bh.entries, Bh.values)
        rm, ent, val, _ = oracle.spgemm(Ap, Bp)
        need = sorted(set(A_loc.entries.tolist()))
        fetched = int(Bh.row_map[-1])
        q.put((rank, rm.tolist(), ent.tolist(), val.tolist(), len(need), fetched,
               int((B.row_map[1:] - B.row_map[:-1])[need].sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_exchange(oracle_mod, world):
    """NEXT-2: each rank fetches only the B rows its A block references; the local product
    with the fetched rows equals its rows of the full product, and exactly the referenced
    rows' entries travel."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, B = g.config("C2", size=7, values="random")
    rm_full, ent_full, val_full, _ = oracle_mod.spgemm(A, B)
    n = B.nrows
    cuts = [n * p // world for p in range(world + 1)]
    for rank, rm, ent, val, nneed, fetched, want_fetched in res:
        r0, r1 = cuts[rank], cuts[rank + 1]
        s, e = int(rm_full[r0]), int(rm_full[r1])
        assert np.array_equal(np.asarray(rm), rm_full[r0:r1 + 1] - s)
        assert np.array_equal(np.asarray(ent, dtype=np.int32), ent_full[s:e])
        assert np.array_equal(np.asarray(val), val_full[s:e])
        assert fetched == want_fetched and nneed < n


def test_flop_balanced_cuts_align():
    from paper_2103_11991_b200.parallel import flop_balanced_cuts

    A, B = g.config("C5", size=5)
    rm = A.row_map.numpy()
    f = np.array([int(B.row_map[int(j) + 1] - B.row_map[int(j)]) for j in A.entries.numpy()])
    per_row = np.add.reduceat(f, rm[:-1]) if len(f) else np.zeros(A.nrows, dtype=np.int64)
    F = np.concatenate([[0], np.cumsum(per_row)])
    for world in (2, 3, 4, 8):
        c = flop_balanced_cuts(F, world, align=3)
        assert c[0] == 0 and c[-1] == A.nrows and c == sorted(c)
        assert all(x % 3 == 0 for x in c), c


@pytest.mark.parametrize("n,world", [(12, 2), (13, 3), (128, 8), (30, 4)])
def test_galerkin_slab_cuts(n, world):
    """Slab p's coarse rows (R's row block) reference only fine rows of slab p, so R_p * T_p
    needs no exchange."""
    from paper_2103_11991_b200.parallel import galerkin_slab_cuts

    fc, cc = galerkin_slab_cuts(n, 3, world)
    nc = (n + 2) // 3
    assert fc[0] == 0 and fc[-1] == n ** 3 and cc[0] == 0 and cc[-1] == nc ** 3
    if n <= 30:
        _, _, R = g.config("C3", size=n)
        rrm, rent = R.row_map.numpy(), R.entries.numpy()
        for p in range(world):
            s, e = int(rrm[cc[p]]), int(rrm[cc[p + 1]])
            cols = rent[s:e]
            assert cols.size == 0 or (cols.min() >= fc[p] and cols.max() < fc[p + 1])
