"""Per-kernel device time inside one kk_spgemm_multiply_host call (diagnostic for the host
path's per-block cost): python tools/e2e_kernels.py [C2|C3] [blocks]."""
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_2103_11991_b200 import CsrMatrix, SpGEMM  # noqa: E402
from workloads import generators as g  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 0
mats = g.config(cfg)


def host(M):
    return CsrMatrix(M.nrows, M.ncols, M.row_map.to(torch.int32).pin_memory(), M.entries.pin_memory(),
                     M.values.pin_memory())


A = host(mats[0])
B = A if cfg in ("C2", "C4", "C5") else host(mats[1])
h = SpGEMM(timing=True)
for it in range(3):
    h.timing_reset()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    h.multiply_host(A, B, blocks=blocks or None)
    t1.record()
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for r in h.kernel_times():
    agg[r[0]][0] += r[1]
    agg[r[0]][1] += r[2]
tot = sum(v[1] for v in agg.values())
print(f"{cfg} blocks={blocks or 'default'}: call {t0.elapsed_time(t1):.3f} ms, kernels {tot:.3f} ms")
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:<28s} launches={n:4d} total={ms:8.3f} ms per={ms / max(n, 1):.4f}")
