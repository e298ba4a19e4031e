"""Benchmark: two-phase hash SpGEMM (symbolic + numeric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--dtype f64]
    python bench.py --impl reference ...      # the CPU oracle arm

One step = one pass of the whole hot path over the
resident synthetic workload: kk_spgemm_symbolic (flop count, scans, binning, B
compression, symbolic counts, row map, the nnz device->host read) followed by
kk_spgemm_numeric (hash accumulation + fused row sort) into caller-allocated C
arrays.  Metric (BASELINE.json): GFLOP/s = 2 * multiply-adds / time,
with the algorithmic HBM GB/s beside it.

At N=1 the workload is BASELINE.json configs[1] (C2: A*A, 3D 27-point Laplacian
100^3, fp64, int32 offsets).  Inputs (A 322 MB, B 322 MB) and C (1.45 GB) exceed
the 126 MB L2, so no flush is needed between steps.  For N>1 (torchrun, one rank
per GPU, NCCL) the rows of A are split in flop-balanced contiguous blocks, B is
replicated by an NCCL broadcast (setup, outside the timed region), and every step
all-gathers the per-rank nnz(C) to form global row offsets -- strong
scaling of the same product.

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import torch  # noqa: E402

METRIC = "SpGEMM (symbolic+numeric) GFLOP/s and HBM GB/s at 1/2/4/8 B200"
UNIT = "GFLOP/s"

WORKLOADS = {
    "C1": "A*A 2D 5-point Laplacian 32x32 (1,024 rows)",
    "C2": "A*A 3D 27-point Laplacian 100^3 (1,000,000 rows)",
    "C3": "Galerkin R*(A*P): 3D 7-point Laplacian 128^3, 3x3x3 aggregation P, R = P^T (two products)",
    "C4": "A*A RMAT scale 20, edge factor 16, directed (1,048,576 rows)",
    "C5": "A*A 3D 27-point block stencil, 3 dof/node, 160^3 (12,288,000 rows)",
    "C3J": "Jacobi-fused (I - w D^-1 A) P: 3D 7-point Laplacian 128^3, 3x3x3 aggregation P, w = 2/3 (NEXT-1)",
    "C3F": "fused Galerkin R*A*P in one pass (NEXT-4): 3D 7-point Laplacian 128^3, 3x3x3 aggregation P, R = P^T",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--size", type=int, default=None, help="override grid edge / RMAT scale")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--values", default="int", choices=["int", "random"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU oracle time budget (cpu_baseline)")
    ap.add_argument("--cpu-rows", type=int, default=None, help="rows of A in the oracle sample")
    ap.add_argument("--kernel-table", action="store_true", help="print the per-kernel timing table to stderr")
    ap.add_argument("--streams", type=int, default=2, help="library internal streams (1 = serialise the bins)")
    ap.add_argument("--no-patterns", action="store_true",
                    help="opts.patterns = 0 (numeric re-derives every row: the A/B of the kept patterns)")
    ap.add_argument("--halo", action="store_true",
                    help="N>1: B row-distributed, each rank fetches only the B rows its A block references "
                         "(NEXT-2) instead of a broadcast of B")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------------------


def offset_dtype_for(cfg):
    return torch.int64 if cfg in ("C4", "C5") else torch.int32


def make_workload(cfg, size, values, device):
    """(A, B) for the A*B configs; (A, P, R) for C3."""
    from workloads import generators as g

    return g.config("C3" if cfg == "C3F" else cfg, size=size, values=values, device=device)


def nbytes(t):
    return t.numel() * t.element_size()


def alg_bytes(A, B, crm, nnz, val_size):
    """SURVEY.md §8d algorithmic bytes: each input array once, each output array once."""
    off = crm.element_size()
    a_pat = (A.nrows + 1) * off + A.nnz * 4
    b_pat = (B.nrows + 1) * off + B.nnz * 4
    sym = a_pat + b_pat + (A.nrows + 1) * off
    num = a_pat + A.nnz * val_size + b_pat + B.nnz * val_size + (A.nrows + 1) * off + nnz * (4 + val_size)
    return sym, num


def _clock_proc(idx, period, conn):
    """Child process: poll NVML (SM clock, clock-event reasons) until told to stop."""
    out = []
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        conn.send(("ready", mx))
        while not conn.poll():
            out.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), int(get_r(h))))
            time.sleep(period)
    except Exception as e:  # noqa: BLE001
        conn.send(("error", str(e)))
        return
    conn.recv()
    conn.send(("samples", out))


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons polled through NVML every few ms by a
    separate process (no GIL contention with the timed loop); only samples taken inside
    the timed region [mark_start, mark_end] are kept (the B200_PROFILING.md clocks line)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu_index, period_s=0.002):
        import multiprocessing as mp

        self.ctx = mp.get_context("spawn")
        self.idx = gpu_index
        self.period = period_s
        self.proc = None
        self.conn = None
        self.max_mhz = None
        self.err = None
        self.t0 = self.t1 = None

    def start(self):
        a, b = self.ctx.Pipe()
        self.conn = a
        self.proc = self.ctx.Process(target=_clock_proc, args=(self.idx, self.period, b), daemon=True)
        self.proc.start()
        if a.poll(60):
            kind, v = a.recv()
            if kind == "ready":
                self.max_mhz = v
            else:
                self.err = v

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        samples = []
        if self.proc is not None and self.err is None:
            self.conn.send("stop")
            if self.conn.poll(30):
                kind, v = self.conn.recv()
                if kind == "samples":
                    samples = v
                else:
                    self.err = v
            self.proc.join(timeout=10)
        t0 = self.t0 if self.t0 is not None else 0.0
        t1 = self.t1 if self.t1 is not None else float("inf")
        win = [(c, r) for t, c, r in samples if t0 <= t <= t1]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [self.err or "no samples"], "samples": 0}
        mask = 0
        for _, r in win:
            mask |= r
        return {"sm_mhz": statistics.median(c for c, _ in win), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(n for n, bit in self.REASONS.items() if mask & bit), "samples": len(win)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "dominant_kernel_traffic.json")
    try:
        return json.load(open(p))
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------------------


def oracle_sample(A, rows):
    """A's contiguous row block [r0, r0+rows) from the middle of the matrix (other rows
    dropped): the bounded sample of the workload the oracle is timed on."""
    from workloads import generators as g

    m = A.nrows
    rows = max(1, min(rows, m))
    r0 = (m - rows) // 2
    rm = A.row_map.to(torch.int64).cpu()
    s, e = int(rm[r0]), int(rm[r0 + rows])
    sub = g.CSR(rows, A.ncols, (rm[r0:r0 + rows + 1] - s).contiguous(), A.entries.cpu()[s:e].contiguous(),
                A.values.cpu()[s:e].to(torch.float64).contiguous())
    return sub, r0


def time_oracle_once(oracle, As, Bh):
    t0 = time.perf_counter()
    rm = oracle.symbolic(As, Bh)
    oracle.numeric(As, Bh, rm)
    return time.perf_counter() - t0


def host_info():
    """CPU model (lscpu), logical CPUs usable by this process, host RAM."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal:"):
                    ram = round(int(line.split()[1]) / 1024 ** 2, 1)
                    break
    except Exception:
        pass
    return {"cpu_model": model, "cpus_usable": len(os.sched_getaffinity(0)), "host_ram_gib": ram}


def cpu_baseline(A, B, seconds, rows):
    """The oracle as it stands on the host: all usable cores (the reported value) and one
    thread (OMP=1, the plain oracle; a fifth of the time budget), SURVEY §8d."""
    import oracle

    oracle.build()
    cores = len(os.sched_getaffinity(0))
    from workloads import generators as g

    def host(M):
        return g.CSR(M.nrows, M.ncols, M.row_map.to(torch.int64).cpu(), M.entries.cpu(),
                     M.values.to(torch.float64).cpu())

    Bh = host(B)
    As, r0 = oracle_sample(host(A), rows)
    f, muladds = oracle.row_flops(As, Bh)

    def timed(threads, budget):
        oracle.set_num_threads(threads)
        tot, reps = 0.0, 0
        while reps < 1 or (tot < budget and reps < 50):
            tot += time_oracle_once(oracle, As, Bh)
            reps += 1
        return 2.0 * muladds * reps / tot / 1e9, reps, tot

    value, reps, tot = timed(cores, seconds)
    used = oracle.num_threads()
    v1, reps1, tot1 = timed(1, seconds / 5)
    oracle.set_num_threads(cores)
    return {"value": round(value, 3), "unit": UNIT, "cores": used, "kind": "oracle",
            "sample": f"rows [{r0}, {r0 + As.nrows}) of A ({As.nrows} of {A.nrows} rows, {muladds} multiply-adds) "
                      f"x full B, symbolic+numeric, {reps} reps in {tot:.2f} s, OpenMP threads={used}",
            "one_thread": {"value": round(v1, 3), "reps": reps1, "seconds": round(tot1, 2)},
            "host": host_info()}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, one bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    oracle.build()
    cores = len(os.sched_getaffinity(0))
    oracle.set_num_threads(cores)
    mats = make_workload(args.config, args.size, args.values, "cpu")
    A, B = mats[0], mats[1]  # C3: the first product T = A*P
    rows = args.cpu_rows or max(1, A.nrows // 8)
    As, r0 = oracle_sample(A, rows)
    Bh = B.to(value_dtype=torch.float64)
    _, muladds = oracle.row_flops(As, Bh)
    for _ in range(args.warmup):
        time_oracle_once(oracle, As, Bh)
    ts = [time_oracle_once(oracle, As, Bh) for _ in range(args.steps)]
    tot = sum(ts)
    value = 2.0 * muladds * args.steps / tot / 1e9
    sample = (f"rows [{r0}, {r0 + As.nrows}) of A ({As.nrows} of {A.nrows} rows, {muladds} multiply-adds) x full B "
              f"per step, symbolic+numeric, OpenMP threads={oracle.num_threads()}")
    out = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 3), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{args.config}: {WORKLOADS[args.config]}", "values": args.values,
                      "offsets": "int32" if offset_dtype_for(args.config) == torch.int32 else "int64"},
           "impl": "reference",
           "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                            "sample": sample, "host": host_info()},
           "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------


def run_ours(args):
    from paper_2103_11991_b200 import CsrMatrix, SpGEMM

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N>1 must be launched with torchrun (one rank per GPU)")
    # BENCH_SHARE_DEVICE=1 / BENCH_BACKEND=gloo: every rank on cuda:0 over gloo -- only for
    # the single-GPU test of the N>1 path (tests/test_gpu_multi.py); never a measurement
    if os.environ.get("BENCH_SHARE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    vdt = torch.float64 if args.dtype == "f64" else torch.float32
    odt = offset_dtype_for(args.config)
    vwork = None

    # ---- workload (generated on the device: inputs resident in HBM) ----
    t_bcast = None
    def conv(M):
        return CsrMatrix(M.nrows, M.ncols, M.row_map.to(odt), M.entries, M.values.to(vdt))

    jac = None
    if world == 1:
        wl = make_workload(args.config, args.size, args.values, dev)
        if args.config == "C3J":  # (A, P, dinv, omega)
            jac = (wl[3], wl[2].to(vdt))
            wl = wl[:2]
        mats = [conv(M) for M in wl]
        A, B = mats[0], mats[1]
        r0, r1 = 0, A.nrows
    else:
        if args.config in ("C3J", "C3F"):
            raise SystemExit(f"{args.config} is benchmarked on one GPU")
        from paper_2103_11991_b200.parallel import (broadcast_csr, flop_balanced_cuts, galerkin_slab_cuts,
                                                    halo_exchange_b, shift_columns, slice_rows)

        align = 3 if args.config == "C5" else 1  # whole 3-dof nodes
        vwork = None
        if args.config == "C3":
            # z-slab partition: P broadcast from rank 0; A and R row blocks of
            # whole aggregate planes, so R_p * T_p needs no second exchange
            A_f, P_f, R_f = make_workload(args.config, args.size, args.values, dev)
            n = round(A_f.nrows ** (1.0 / 3.0))
            fc, cc = galerkin_slab_cuts(n, 3, world)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            P = broadcast_csr(conv(P_f) if rank == 0 else None, src=0, device=dev)
            e1.record()
            torch.cuda.synchronize()
            t_bcast = e0.elapsed_time(e1)
            r0, r1 = fc[rank], fc[rank + 1]
            A = conv(slice_rows(A_f, r0, r1))
            R_p = conv(shift_columns(slice_rows(R_f, cc[rank], cc[rank + 1]), r0, r1 - r0))
            mats = [A, P, R_p]
            B = P
            del A_f, R_f
        elif args.halo:
            # every rank holds its row block of B (here: generated whole, then sliced -- the
            # input of a row-distributed solver) and fetches the rows its A block needs
            full = conv(make_workload(args.config, args.size, args.values, dev)[1])
            hf = SpGEMM(device=dev)
            _, F, _ = hf.row_flops(full, full, scan=True, total=False)
            hf.close()
            cuts = flop_balanced_cuts(F.cpu().numpy(), world, align)
            r0, r1 = cuts[rank], cuts[rank + 1]
            A = slice_rows(full, r0, r1)
            B_loc = slice_rows(full, r0, r1)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            B = halo_exchange_b(A, B_loc, cuts)
            e1.record()
            torch.cuda.synchronize()
            t_bcast = e0.elapsed_time(e1)
            A = CsrMatrix(A.nrows, A.ncols, A.row_map.contiguous(), A.entries.contiguous(), A.values.contiguous())
            del full
            mats = [A, B]
        else:
            if rank == 0:
                B0 = conv(make_workload(args.config, args.size, args.values, dev)[1])
            else:
                B0 = None
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            # the values' broadcast stays in flight while the row split and the first symbolic
            # phase (pattern only) run; the first numeric phase waits for it
            B, vwork = broadcast_csr(B0, src=0, device=dev, async_values=True)
            e1.record()
            # A*A: A is B (a separate copy on every rank would only double memory; row block
            # of the broadcast matrix, SURVEY §8e "A needs no extra traffic")
            hf = SpGEMM(device=dev)
            _, F, _ = hf.row_flops(B, B, scan=True, total=False)
            hf.close()
            cuts = flop_balanced_cuts(F.cpu().numpy(), world, align)
            r0, r1 = cuts[rank], cuts[rank + 1]
            A = slice_rows(B, r0, r1)
            mats = [A, B]

    stream = torch.cuda.current_stream(dev)

    class Product:
        """One C = X*Y of the step: its handle, row map and preallocated C arrays."""

        def __init__(self, X, Y, jacobi=None):
            self.X, self.Y, self.jacobi = X, Y, jacobi
            self.h = SpGEMM(device=dev, timing=True, num_streams=args.streams, patterns=not args.no_patterns)
            self.crm = torch.empty(X.nrows + 1, dtype=odt, device=dev)
            _, n = self.h.symbolic(X, Y, c_row_map=self.crm)
            self.cent = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            self.cval = torch.empty(max(n, 1), dtype=vdt, device=dev)
            self.nnz = n

        def C(self):
            return CsrMatrix(self.X.nrows, self.Y.ncols, self.crm, self.cent[:self.nnz], self.cval[:self.nnz])

    class RapProduct:
        """The fused triple product Ac = R*A*P of C3F (one symbolic + one numeric call)."""

        def __init__(self, R, A_, P):
            self.R, self.A, self.P = R, A_, P
            self.X, self.Y, self.jacobi, self.rap = R, P, None, True
            self.h = SpGEMM(device=dev, timing=True, num_streams=args.streams)
            self.crm = torch.empty(R.nrows + 1, dtype=odt, device=dev)
            _, n = self.h.rap_symbolic(R, A_, P, c_row_map=self.crm)
            self.cent = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            self.cval = torch.empty(max(n, 1), dtype=vdt, device=dev)
            self.nnz = n
            # the work of the product it replaces (T = A*P, Ac = R*T), for a comparable GFLOP/s
            h2 = SpGEMM(device=dev)
            T = h2(A_, P)
            self.muladds = h2.stats()["muladds"]
            h3 = SpGEMM(device=dev)
            h3.symbolic(R, T)
            self.muladds += h3.stats()["muladds"]
            h2.close()
            h3.close()

    # the step's products: A*B, or for C3 T = A*P then Ac = R*T (T stays in HBM)
    if args.config == "C3F":
        prods = [RapProduct(mats[2], A, B)]
    else:
        prods = [Product(A, B, jac)]
    if world > 1 and vwork is not None:
        vwork.wait()  # B's values (in flight during the row split and the first symbolic phase)
        torch.cuda.synchronize()
        t_bcast = e0.elapsed_time(e1)  # the blocking part: header, row map, entries
    if args.config == "C3":
        prods.append(Product(mats[2], prods[0].C()))
    if world > 1:
        from paper_2103_11991_b200.parallel import allgather_row_map_total

    def step(ev=None):
        for k, pr in enumerate(prods):
            if ev is not None:
                ev[2 * k].record(stream)
            if getattr(pr, "rap", False):
                _, n = pr.h.rap_symbolic(pr.R, pr.A, pr.P, c_row_map=pr.crm)
                if ev is not None:
                    ev[2 * k + 1].record(stream)
                pr.h.rap_numeric(pr.R, pr.A, pr.P, pr.crm, n, c_entries=pr.cent[:n], c_values=pr.cval[:n])
                continue
            _, n = pr.h.symbolic(pr.X, pr.Y, c_row_map=pr.crm)
            if world > 1:
                # nnz(C_p) straight from the row map the scan kernel wrote (no host tensor)
                allgather_row_map_total(pr.crm)
            if ev is not None:
                ev[2 * k + 1].record(stream)
            if pr.jacobi is not None:
                pr.h.jacobi_numeric(pr.jacobi[0], pr.jacobi[1], pr.X, pr.Y, pr.crm, nnz=n, c_entries=pr.cent[:n],
                                    c_values=pr.cval[:n])
            else:
                pr.h.numeric(pr.X, pr.Y, pr.crm, nnz=n, c_entries=pr.cent[:n], c_values=pr.cval[:n])
        if ev is not None:
            ev[2 * len(prods)].record(stream)

    clk = ClockSampler(local)
    clk.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sts = [pr.h.stats() for pr in prods]
    for pr, st in zip(prods, sts):
        if getattr(pr, "rap", False):  # the fused product reports the work of R*(A*P)
            st["muladds"], st["nnz_c"] = pr.muladds, pr.nnz
    muladds = sum(st["muladds"] for st in sts)
    nnz = sts[-1]["nnz_c"]
    for pr in prods:
        pr.h.timing_reset()
    launches0 = sum(st["kernel_launches"] for st in sts)
    ne = 2 * len(prods) + 1
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(ne)] for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark_start()
    t_start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    clk.mark_end()
    if dist is not None:
        dist.barrier()
    clocks = clk.stop()
    launches = sum(pr.h.stats()["kernel_launches"] for pr in prods) - launches0
    ktimes = {}
    for pr in prods:
        for name, n_, tot, mx in pr.h.kernel_times():
            a_ = ktimes.setdefault(name, [name, 0, 0.0, 0.0])
            a_[1] += n_
            a_[2] += tot
            a_[3] = max(a_[3], mx)
    ktimes = [tuple(v) for v in ktimes.values()]
    ms_total = t_start.elapsed_time(t_end)
    sym_ms = statistics.median(sum(e[2 * k].elapsed_time(e[2 * k + 1]) for k in range(len(prods))) for e in evs)
    num_ms = statistics.median(sum(e[2 * k + 1].elapsed_time(e[2 * k + 2]) for k in range(len(prods)))
                               for e in evs)

    # max over ranks (device-timed); aggregate work = sum over ranks
    if dist is not None:
        t = torch.tensor([ms_total, sym_ms, num_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total, sym_ms_max, num_ms_max = t.tolist()
        w = torch.tensor([muladds, nnz, A.nnz], dtype=torch.int64, device=dev)
        dist.all_reduce(w)
        muladds_all, nnz_all_c, nnzA_all = w.tolist()
    else:
        sym_ms_max, num_ms_max = sym_ms, num_ms
        muladds_all, nnz_all_c = muladds, nnz
    ms_step = ms_total / args.steps
    gflops = 2.0 * muladds_all / (ms_step * 1e-3) / 1e9

    val_size = 8 if vdt == torch.float64 else 4
    sym_b = num_b = 0
    for pr, st in zip(prods, sts):
        sb, nb = alg_bytes(pr.X, pr.Y, pr.crm, st["nnz_c"], val_size)
        if getattr(pr, "rap", False):  # + A, read by both phases
            off = pr.crm.element_size()
            a_pat = (pr.A.nrows + 1) * off + pr.A.nnz * 4
            sb += a_pat
            nb += a_pat + pr.A.nnz * val_size
        sym_b += sb
        num_b += nb
    if dist is not None:
        w = torch.tensor([sym_b, num_b], dtype=torch.int64, device=dev)
        dist.all_reduce(w)
        sym_b_all, num_b_all = w.tolist()
    else:
        sym_b_all, num_b_all = sym_b, num_b
    hbm_gbs = (sym_b_all + num_b_all) / (ms_step * 1e-3) / 1e9
    peak, peak_src = load_peaks()

    # dominant kernel (most device time in the timed region)
    kt = sorted(ktimes, key=lambda r: -r[2])
    dom = kt[0] if kt else ("none", 1, float("nan"), 0.0)
    num_kernels = [r for r in ktimes if r[0].startswith("num_")]
    num_launch_ms = sum(r[2] for r in num_kernels) / args.steps
    # numeric phase = the dominant unit on every config here (~85% of bytes);
    # its algorithmic bytes per step are the numeric bytes.
    roof_achieved = num_b / (num_launch_ms * 1e-3) / 1e9 if num_launch_ms > 0 else None
    traffic = ncu_traffic() if args.config == "C2" and args.size is None else None
    roofline = {"bound": "hbm", "achieved": round(roof_achieved, 1) if roof_achieved else None,
                "peak": peak, "unit": "GB/s", "frac": round(roof_achieved / peak, 4) if roof_achieved else None,
                "traffic": (traffic or {}).get("dram_bytes_per_step"),
                "kernel": "+".join(r[0] for r in num_kernels),
                "alg_bytes_per_launch": num_b,
                "launch_ms": round(num_launch_ms, 4),
                "peak_source": peak_src,
                "dominant_single_kernel": {"name": dom[0], "ms_per_launch": round(dom[2] / max(dom[1], 1), 4),
                                           "share_of_step": round(dom[2] / ms_total, 4) if ms_total else None}}
    if args.kernel_table and rank == 0:
        for r in kt:
            sys.stderr.write(f"  {r[0]:<24s} launches={r[1]:>4d} total={r[2]:9.3f} ms  "
                             f"per={r[2] / max(r[1], 1):8.4f} ms  share={r[2] / ms_total:6.3f}\n")

    # ---- e2e through the public API from pinned host buffers (N=1; per rank for N>1) ----
    e2e = None
    host_bytes = sum(nbytes(x) for M in mats for x in (M.row_map, M.entries, M.values)) + \
        nnz * (4 + val_size) + (prods[-1].X.nrows + 1) * 8
    if args.no_e2e:
        e2e = None
    elif jac is not None or args.config == "C3F":
        e2e = {"value": None, "unit": UNIT,
               "skipped": f"{args.config}: the host-buffer path covers the plain product only"}
    elif host_bytes > 48e9:
        e2e = {"value": None, "unit": UNIT, "skipped": f"inputs + C = {host_bytes / 1e9:.0f} GB of pinned host memory"}
    else:
        def host(M):
            return CsrMatrix(M.nrows, M.ncols, M.row_map.cpu().pin_memory(), M.entries.cpu().pin_memory(),
                             M.values.cpu().pin_memory())

        # A*A workloads square ONE host matrix (the library copies it to the device once and
        # takes A's row blocks from that copy); the device-timed leg keeps two copies
        square = world == 1 and args.config in ("C2", "C4", "C5")
        hmats = [host(M) for M in (mats[:1] if square else mats)]
        if square:
            hmats = [hmats[0], hmats[0]] + [host(M) for M in mats[2:]]
        hes = [SpGEMM(device=dev) for _ in prods]

        def e2e_step():
            # the user-level host path: C = A*B, or T = A*P then Ac = R*T, each call copying
            # its operands in and its result out
            nb = int(os.environ["KK_E2E_BLOCKS"]) if os.environ.get("KK_E2E_BLOCKS") else None
            C = hes[0].multiply_host(hmats[0], hmats[1], blocks=nb)
            ins = [hmats[0]] if square else [hmats[0], hmats[1]]
            if len(prods) > 1:
                ins += [hmats[2], C]
                C = hes[1].multiply_host(hmats[2], C, blocks=nb)
            return ins, C

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        reps = max(2, min(args.steps, 5))
        e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_s.record(stream)
        for _ in range(reps):
            ins, Ch = e2e_step()
        e_e.record(stream)
        torch.cuda.synchronize()
        e_ms = e_s.elapsed_time(e_e) / reps
        if dist is not None:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = t.item()
        h2d = sum(nbytes(x) for M in ins for x in (M.row_map, M.entries, M.values))
        if square:  # A's row maps, rebased per row block, cross PCIe in addition to the matrix
            h2d += nbytes(ins[0].row_map)
        d2h = sum(nbytes(x) for x in (Ch.row_map, Ch.entries, Ch.values))
        if len(prods) > 1:
            d2h += sum(nbytes(x) for x in (ins[3].row_map, ins[3].entries, ins[3].values))
        if dist is not None:
            w = torch.tensor([h2d, d2h], dtype=torch.int64, device=dev)
            dist.all_reduce(w)
            h2d, d2h = w.tolist()
        e2e = {"value": round(2.0 * muladds_all / (e_ms * 1e-3) / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e_ms, 3)}
        for he in hes:
            he.close()
        del hmats

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # a quarter of the rows, fewer when the product is big (bounded oracle memory/time)
        frac = min(0.25, 2e8 / max(sts[0]["muladds"], 1))
        rows = args.cpu_rows or max(1, int(A.nrows * frac))
        cpu = cpu_baseline(A, B, args.cpu_seconds, rows)
        if args.config == "C3":
            cpu["sample"] = "first product T = A*P only: " + cpu["sample"]
        if args.config == "C3J":
            cpu["sample"] = "plain E = A*P (the oracle's usual product): " + cpu["sample"]
        if args.config == "C3F":
            cpu["sample"] = "first product T = A*P only: " + cpu["sample"]

    if rank == 0:
        out = {"metric": METRIC, "value": round(gflops, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
               "config": {"workload": f"{args.config}: {WORKLOADS[args.config]}", "values": args.values,
                          "offsets": "int32" if odt == torch.int32 else "int64",
                          "l2": "inputs (A, B) and output C each exceed the 126 MB L2; no flush",
                          "parallelism": f"row-sharded x{world}" + (
                              (", z-slabs, P broadcast (NCCL), nnz all-gather" if args.config == "C3" else
                               ", B halo exchange (NCCL), nnz all-gather" if args.halo else
                               ", B broadcast (NCCL, values overlapped with symbolic), nnz all-gather")
                              if world > 1 else ""),
                          "nnz_A": int(A.nnz) if world == 1 else int(nnzA_all), "nnz_C": int(nnz_all_c),
                          "multiply_adds": int(muladds_all)},
               "hbm_gbs": round(hbm_gbs, 1), "hbm_frac": round(hbm_gbs / peak, 4),
               "phases_ms": {"symbolic": round(sym_ms_max, 4), "numeric": round(num_ms_max, 4),
                             "broadcast_B": round(t_bcast, 3) if t_bcast is not None else None,
                             "B_exchange": (("halo" if args.halo else "broadcast") if world > 1 else None)},
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
               "clocks": clocks}
        print(json.dumps(out), flush=True)
    for pr in prods:
        pr.h.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
