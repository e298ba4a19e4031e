"""Small products through every tier, for compute-sanitizer:

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_driver.py

C1 (2D 5-point 32x32), C2 at 20^3 (pattern / rank tier), a short-B-row product (warp
tables), long rows over k = 200K (CTA bit-vector tier) and k = 20K (windowed dense tier),
the Jacobi-fused product and SpAdd; each checked against the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2103_11991_b200 import SpGEMM  # noqa: E402
from workloads import generators as g  # noqa: E402


def run(name, A, B, **opts):
    Ad = A.to(device="cuda", offset_dtype=torch.int32)
    Bd = B.to(device="cuda", offset_dtype=torch.int32)
    h = SpGEMM(**opts)
    rm, nnz = h.symbolic(Ad, Bd)
    ent, val = h.numeric(Ad, Bd, rm, nnz=nnz)
    torch.cuda.synchronize()
    orm, oent, oval, obnd = oracle.spgemm(A, B)
    ok = np.array_equal(rm.cpu().numpy().astype(np.int64), orm) and np.array_equal(ent.cpu().numpy(), oent) and \
        bool(np.all(np.abs(val.cpu().numpy() - oval) <= 1e-12 * obnd))
    h.close()
    print(f"{name}: nnz={nnz} parity={'ok' if ok else 'FAIL'}", flush=True)
    return ok


def main():
    oracle.build()
    ok = True
    A, B = g.config("C1", values="random")
    ok &= run("C1", A, B)
    A, B = g.config("C2", size=20, values="random")
    ok &= run("C2 n=20", A, B)
    ok &= run("C2 n=20 deterministic", A, B, deterministic=True)
    A = g.random_csr(200, 150, 20, seed=3)
    B = g.random_csr(150, 300, 2, seed=4)
    ok &= run("short B rows", A, B)
    A = g.random_csr(12, 300, 60, seed=5, empty_row_frac=0.0)
    B = g.random_csr(300, 200000, 200, seed=6, empty_row_frac=0.0)
    ok &= run("long rows k=200K", A, B)
    B = g.random_csr(300, 20000, 200, seed=7, empty_row_frac=0.0)
    ok &= run("long rows k=20K", A, B)
    A, B = g.config("C2", size=10, values="random")
    Ad = A.to(device="cuda", offset_dtype=torch.int32)
    Bd = B.to(device="cuda", offset_dtype=torch.int32)
    h = SpGEMM()
    dinv = g.diagonal_inverse(A)
    J = h.jacobi(2.0 / 3.0, dinv.to("cuda"), Ad, Bd)
    S = h.spadd(0.5, Ad, -1.0, Bd)
    torch.cuda.synchronize()
    jrm, jent, jval, jbnd = oracle.jacobi(2.0 / 3.0, dinv.numpy(), A, B)
    srm, sent, sval, sbnd = oracle.spadd(0.5, A, -1.0, B)
    okj = np.array_equal(J.entries.cpu().numpy(), jent) and bool(np.all(np.abs(J.values.cpu().numpy() - jval) <= 1e-12 * jbnd))
    oks = np.array_equal(S.entries.cpu().numpy(), sent) and bool(np.all(np.abs(S.values.cpu().numpy() - sval) <= 1e-12 * sbnd))
    print(f"jacobi parity={'ok' if okj else 'FAIL'} spadd parity={'ok' if oks else 'FAIL'}", flush=True)
    h.close()
    ok &= okj and oks
    print("ALL OK" if ok else "PARITY FAILURES")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
