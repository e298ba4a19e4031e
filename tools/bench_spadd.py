"""SpAdd benchmark (NEXT-3): C = A + B on the paper's SpAdd matrices (PAPER.md:318-321:
square, 30 random entries per row), device-resident, fp64, int32 offsets.  Prints one JSON
line: symbolic and numeric ms (CUDA events, median of K), the numeric phase's algorithmic
GB/s against the measured HBM peak, and nnz.

    python tools/bench_spadd.py [--rows 2000000] [--per-row 30] [--steps 20] [--warmup 3]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=2_000_000)
    ap.add_argument("--per-row", type=int, default=30)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    from paper_2103_11991_b200 import CsrMatrix, SpGEMM
    from workloads import generators as g

    m = args.rows
    mats = []
    for seed in (1, 2):
        M = g.random_rows_csr(m, m, args.per_row, seed=seed, device="cuda")
        mats.append(CsrMatrix(m, m, M.row_map.to(torch.int32), M.entries, M.values))
    A, B = mats
    h = SpGEMM()
    rm = torch.empty(m + 1, dtype=torch.int32, device="cuda")
    _, nnz = h.spadd_symbolic(A, B, c_row_map=rm)
    ent = torch.empty(nnz, dtype=torch.int32, device="cuda")
    val = torch.empty(nnz, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(args.warmup):
        h.spadd_symbolic(A, B, c_row_map=rm)
        h.spadd_numeric(1.0, A, 1.0, B, rm, nnz, c_entries=ent, c_values=val)
    torch.cuda.synchronize()
    ts, tn = [], []
    for _ in range(args.steps):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(st)
        h.spadd_symbolic(A, B, c_row_map=rm)
        e1.record(st)
        h.spadd_numeric(1.0, A, 1.0, B, rm, nnz, c_entries=ent, c_values=val)
        e2.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        tn.append(e1.elapsed_time(e2))
    sym, num = statistics.median(ts), statistics.median(tn)
    # numeric algorithmic bytes: A, B (row maps, entries, values), Apos/Bpos, C row map read,
    # C entries + values written
    nz = A.nnz + B.nnz
    num_bytes = 2 * (m + 1) * 4 + nz * (4 + 8 + 4) + (m + 1) * 4 + nnz * 12
    peak = None
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except Exception:
        pass
    gbs = num_bytes / (num * 1e-3) / 1e9
    print(json.dumps({"workload": f"SpAdd A+B, {m} x {m}, {args.per_row} random entries per row, fp64, int32",
                      "symbolic_ms": round(sym, 4), "numeric_ms": round(num, 4), "nnz_C": int(nnz),
                      "numeric_alg_bytes": int(num_bytes), "numeric_gbs": round(gbs, 1),
                      "numeric_frac_of_hbm": round(gbs / peak, 4) if peak else None, "hbm_peak_gbs": peak}))
    h.close()


if __name__ == "__main__":
    main()
