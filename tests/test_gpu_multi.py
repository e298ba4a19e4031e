"""The N>1 data path exercised on ONE GPU: two ranks over gloo, both on cuda:0,
running the real kernels.  This run has a single GPU, so these tests check correctness of
the sharded path by construction -- flop-balanced (and node-aligned) row splits, the B
broadcast with its values overlapped with the symbolic phase, nnz(C_p) all-gathered from the
device row map, the z-slab Galerkin partition -- and compare the stitched C with the oracle.
They say nothing about multi-GPU performance (the ranks share one device)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, out_path):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    from paper_2103_11991_b200 import CsrMatrix, SpGEMM
    from paper_2103_11991_b200.parallel import (ShardedSpGEMM, broadcast_csr, flop_balanced_cuts,
                                                galerkin_slab_cuts, shift_columns, slice_rows)
    from workloads import generators as g

    def dv(M):
        return CsrMatrix(M.nrows, M.ncols, M.row_map.to(dev), M.entries.to(dev), M.values.to(dev))

    if case in ("C2", "C5"):
        size = 10 if case == "C2" else 6
        A0, _ = g.config(case, size=size, values="random")
        B, work = broadcast_csr(dv(A0) if rank == 0 else None, src=0, device=dev, async_values=True)
        h = SpGEMM(device=dev)
        _, F, _ = h.row_flops(B, B, scan=True, total=False)
        h.close()
        cuts = flop_balanced_cuts(F.cpu().numpy(), world, 3 if case == "C5" else 1)
        A_p = slice_rows(B, cuts[rank], cuts[rank + 1])
        sh = ShardedSpGEMM(device=dev)
        C_p, off, tot = sh(A_p, B, values_work=work)
        torch.cuda.synchronize()
        sh.close()
    else:  # C3: slab-partitioned R*(A*P)
        n = 12
        A_f, P_f, R_f = g.config("C3", size=n, values="int")
        fc, cc = galerkin_slab_cuts(n, 3, world)
        cuts = fc
        P = broadcast_csr(dv(P_f) if rank == 0 else None, src=0, device=dev)
        A_p = dv(slice_rows(A_f, fc[rank], fc[rank + 1]))
        R_p = dv(shift_columns(slice_rows(R_f, cc[rank], cc[rank + 1]), fc[rank], fc[rank + 1] - fc[rank]))
        T_p, _, _ = ShardedSpGEMM(device=dev)(A_p, P)
        C_p, off, tot = ShardedSpGEMM(device=dev)(R_p, T_p)
        torch.cuda.synchronize()
    pieces = [C_p.row_map.cpu().to(torch.int64), C_p.entries.cpu(), C_p.values.cpu().double(),
              torch.tensor([off, tot, cuts[rank], cuts[rank + 1]])]
    gathered = [None] * world
    dist.all_gather_object(gathered, [p.numpy().tolist() for p in pieces])
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(gathered, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["C2", "C5", "C3"])
def test_sharded_world2_on_one_gpu(oracle_mod, tmp_path, case):
    import torch.multiprocessing as mp

    from workloads import generators as g

    out = str(tmp_path / "c.json")
    mp.spawn(_worker, args=(2, _free_port(), case, out), nprocs=2, join=True)
    got = json.load(open(out))
    if case == "C3":
        A, P, R = g.config("C3", size=12, values="int")
        orm, oent, oval, _ = oracle_mod.spgemm(A, P)
        T = g.CSR(A.nrows, P.ncols, torch.tensor(orm), torch.tensor(oent), torch.tensor(oval))
        orm, oent, oval, _ = oracle_mod.spgemm(R, T)
    else:
        A, _ = g.config(case, size=10 if case == "C2" else 6, values="random")
        orm, oent, oval, obnd = oracle_mod.spgemm(A, A)
    # stitch: row maps shifted by the all-gathered offsets, blocks in rank order
    rm = [0]
    ent, val = [], []
    for p, (prm, pent, pval, meta) in enumerate(got):
        off, tot = meta[0], meta[1]
        assert off == rm[-1], "global offset O_p = sum of the earlier ranks' nnz"
        rm.extend(int(x) + off for x in prm[1:])
        ent.extend(pent)
        val.extend(pval)
        if case == "C5":
            assert meta[2] % 3 == 0 and meta[3] % 3 == 0, "split points on whole 3-dof nodes"
    assert got[-1][3][1] == rm[-1] == len(ent)
    assert np.array_equal(np.array(rm), orm)
    assert np.array_equal(np.array(ent, dtype=np.int32), oent)
    if case == "C3":
        assert np.array_equal(np.array(val), oval)
    else:
        assert np.all(np.abs(np.array(val) - oval) <= 1e-12 * obnd)


def test_bench_world2_on_one_gpu():
    """bench.py's N>1 step (B broadcast with overlapped values, per-step nnz all-gather from
    the device row map, max-over-ranks timing) through torchrun, both ranks on cuda:0 over
    gloo: the JSON line reports the whole product (closed forms of C2 at n = 20)."""
    n = 20
    env = dict(os.environ, BENCH_BACKEND="gloo", BENCH_SHARE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2", "--steps", "2",
           "--warmup", "1", "--size", str(n), "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2
    assert d["config"]["multiply_adds"] == (9 * n - 10) ** 3 and d["config"]["nnz_C"] == (5 * n - 6) ** 3
    # C3 on the slab partition
    cmd[cmd.index("--size") + 1] = "24"
    r = subprocess.run(cmd + ["--config", "C3"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 2 and "z-slabs" in d["config"]["parallelism"]
