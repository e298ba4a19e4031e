"""GPU parity of the fallback kernels that the default launch configuration does not pick.

k_num_pattern (pattern bins) and k_sym_window / k_sym_hash (window and hash symbolic bins)
are what the library runs when B.nnz >= 2^31 (their element offsets are 64-bit); with
KK_NUM_RANK=0 / KK_SYM_ROWS=0 they also take the bins of smaller products.  The cluster
tier of the dense bin (k_num_cluster, KK_HUB_CLUSTER=1) is measured slower than the CTA
tier with L2 reductions on C4 and is off by default; its parity is checked here too.  The selection
is read once per process, so each case runs in a subprocess with those variables set; the
subprocess checks, through the per-kernel timing records of the C ABI, that the fallback
kernels actually ran, and compares C with the oracle.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = ["C2", "C5", "banded", "wide", "unsorted", "cluster"]


def _run_case(name):
    import numpy as np
    import torch

    sys.path.insert(0, ROOT)
    import oracle
    from paper_2103_11991_b200 import SpGEMM
    from tests.helpers import assert_parity, to_device
    from tests.test_gpu_parity import _banded, _diag_first
    from workloads import generators as g

    oracle.build()
    if name == "C2":
        A, B = g.config("C2", size=14, values="random")
    elif name == "C5":
        A, B = g.config("C5", size=8, values="random")
    elif name == "banded":
        A, B = _banded(1500, 3000, 12, 1500, seed=6000), _banded(3000, 3000, 60, 6000, seed=6001)
    elif name == "wide":
        A, B = _banded(1200, 4000, 4, 40, seed=21), _banded(4000, 400000, 14, 60000, seed=22)
    elif name == "cluster":
        # rows far above one CTA's value array over k = 1M: the cluster tier (KK_HUB_CLUSTER=1)
        rng = np.random.default_rng(29)
        k, nb = 1_000_000, 160
        b_rows = [np.sort(rng.choice(k, 12000 - 7 * j, replace=False)) for j in range(nb)]
        brm = np.cumsum([0] + [len(r) for r in b_rows])
        B = g.CSR(nb, k, torch.tensor(brm), torch.tensor(np.concatenate(b_rows), dtype=torch.int32),
                  torch.tensor(rng.uniform(-1, 1, brm[-1])))
        a_rows = [np.arange(nb), np.sort(rng.choice(nb, 30, replace=False)), np.array([5, 77]), np.array([9])]
        arm = np.cumsum([0] + [len(r) for r in a_rows])
        A = g.CSR(len(a_rows), nb, torch.tensor(arm), torch.tensor(np.concatenate(a_rows), dtype=torch.int32),
                  torch.tensor(rng.uniform(-1, 1, arm[-1])))
    else:
        A, B = g.config("C2", size=12, values="random")
        A, B = _diag_first(A), _diag_first(B)
    names = set()
    for ot in (torch.int32, torch.int64):
        for vt in (torch.float64, torch.float32):
            h = SpGEMM(timing=True)
            Ad, Bd = to_device(A, "cuda", vt, ot), to_device(B, "cuda", vt, ot)
            rm, nnz = h.symbolic(Ad, Bd)
            ent, val = h.numeric(Ad, Bd, rm, nnz=nnz)
            torch.cuda.synchronize()
            names |= {k[0] for k in h.kernel_times()}
            got = (rm.cpu().numpy().astype(np.int64), ent.cpu().numpy(), val.cpu().double().numpy())
            assert_parity(oracle, A, B, got, value_dtype=vt)
            h.close()
    print(json.dumps(sorted(names)))


@pytest.mark.parametrize("case", CASES)
def test_fallback_kernels(case):
    env = dict(os.environ, KK_NUM_RANK="0", KK_SYM_ROWS="0", KK_HUB_CLUSTER="1")
    r = subprocess.run([sys.executable, os.path.abspath(__file__), case], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    names = set(json.loads(r.stdout.strip().splitlines()[-1]))
    assert not any(n.startswith("num_rank") or n.startswith("sym_rows") for n in names), names
    if case in ("C2", "C5", "wide"):
        assert any(n.startswith("num_pattern") for n in names), names
    if case in ("C2", "banded"):
        assert any(n.startswith("sym_window") for n in names), names
    if case in ("C5", "wide", "unsorted"):
        assert any(n.startswith("sym_hash") for n in names), names
    if case == "cluster":
        assert any(n.startswith("num_cluster") for n in names), names


if __name__ == "__main__":
    _run_case(sys.argv[1])
