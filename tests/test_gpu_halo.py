"""The halo-only B exchange over NCCL (world size 1 on the one GPU of a test box: the
all_to_all_single calls with split sizes run for real) feeding the CUDA SpGEMM."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from workloads import generators as g

from .helpers import assert_parity

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2103_11991_b200 import CsrMatrix, SpGEMM
        from paper_2103_11991_b200.parallel import halo_exchange_b, slice_rows

        A, B = g.config("C2", size=10, values="random")
        Bd = CsrMatrix(B.nrows, B.ncols, B.row_map.cuda(), B.entries.cuda(), B.values.cuda())
        Ad = CsrMatrix(A.nrows, A.ncols, A.row_map.cuda(), A.entries.cuda(), A.values.cuda())
        r0, r1 = 200, 700  # a row block of A; B whole on the single rank
        Ablk = slice_rows(Ad, r0, r1)
        Ablk = CsrMatrix(Ablk.nrows, Ablk.ncols, Ablk.row_map, Ablk.entries.contiguous(), Ablk.values.contiguous())
        Bh = halo_exchange_b(Ablk, Bd, [0, B.nrows])
        h = SpGEMM()
        C = h(Ablk, Bh)
        torch.cuda.synchronize()
        q.put((int(Bh.row_map[-1]), C.row_map.cpu().numpy(), C.entries.cpu().numpy(), C.values.cpu().numpy()))
        h.close()
    finally:
        dist.destroy_process_group()


def test_halo_exchange_nccl_world1(oracle_mod):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_port(), q))
    p.start()
    fetched, rm, ent, val = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    A, B = g.config("C2", size=10, values="random")
    rmA = A.row_map.numpy()
    s, e = int(rmA[200]), int(rmA[700])
    Ablk = g.CSR(500, A.ncols, torch.tensor(rmA[200:701] - s), A.entries[s:e], A.values[s:e])
    need = np.unique(Ablk.entries.numpy())
    assert fetched == int(np.diff(B.row_map.numpy())[need].sum()) and len(need) < B.nrows
    assert_parity(oracle_mod, Ablk, B, (rm.astype(np.int64), ent, val))
