"""Summarise a gpurun measurement set into profiles/ (tracked).

    python tools/summarize_profiles.py TAG [--steps 2]

Reads gpurun_out/launches_TAG.csv (ncu launch list of `bench.py --steps S --warmup 1`),
gpurun_out/prof_top_TAG.ncu-rep (ncu --set full of the dominant kernels) and
gpurun_out/bench_TAG.json, and writes
  profiles/TAG_launches.md     per-kernel device time and share of the step (ncu, cold, serialised)
  profiles/TAG_ncu_top.md      key counters of the full captures (+ hottest SASS lines)
  profiles/TAG_launches.csv    the raw launch list (kernel, duration, dram bytes if captured)
  profiles/dominant_kernel_traffic.json   dram bytes per step of the numeric-phase kernels
"""
from __future__ import annotations

import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def short(name: str) -> str:
    m = re.match(r"(?:void )?(?:kk::)?(\w+)(<[^(]*>)?", name.strip())
    if not m:
        return name[:60]
    tmpl = (m.group(2) or "").replace("(int)", "").replace("(bool)", "").replace(" ", "")
    return m.group(1) + tmpl


def read_launches(tag):
    path = os.path.join(OUT, f"launches_{tag}.csv")
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    hdr = rows[0]
    ci = {h: k for k, h in enumerate(hdr)}
    data = []
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        data.append(r)
    # one row per (launch, metric)
    launches = OrderedDict()
    for r in data:
        key = (r[ci["ID"]], r[ci["Kernel Name"]])
        d = launches.setdefault(key, {"name": short(r[ci["Kernel Name"]])})
        unit = r[ci["Metric Unit"]]
        val = float(r[ci["Metric Value"]].replace(",", ""))
        mname = r[ci["Metric Name"]]
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "second": 1e3, "s": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                 "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1.0)
        d[mname] = val * scale
    return list(launches.values())


def summarize_launches(tag, steps):
    L = read_launches(tag)
    # the bench runs warmup(1) + steps; keep the last `steps` steps: every kernel name that
    # appears per step appears (warmup + steps) times -> take the trailing share
    per = OrderedDict()
    other = {"n": 0, "ms": 0.0}
    for d in L:
        if not d["name"].startswith("k_"):  # PyTorch kernels of the workload generator / plumbing
            other["n"] += 1
            other["ms"] += d.get("gpu__time_duration.sum", 0.0)
            continue
        p = per.setdefault(d["name"], {"n": 0, "ms": 0.0, "dram": 0.0})
        p["n"] += 1
        p["ms"] += d.get("gpu__time_duration.sum", 0.0)
        p["dram"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(p["ms"] for p in per.values())
    lines = [f"# ncu launch list, tag {tag}", "",
             "Source: `ncu --metrics gpu__time_duration.sum[,dram__bytes_*] --clock-control none` over "
             "`python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline` (C2). Per-launch times are "
             "cold-cache and serialised: compare shares, not absolutes.", "",
             "| kernel | launches | total ms | ms/launch | share | dram MB/launch |", "|---|---|---|---|---|---|"]
    for name, p in sorted(per.items(), key=lambda kv: -kv[1]["ms"]):
        dram = f"{p['dram'] / p['n'] / 1e6:.1f}" if p["dram"] else "-"
        lines.append(f"| `{name}` | {p['n']} | {p['ms']:.3f} | {p['ms'] / p['n']:.4f} | {p['ms'] / tot:.3f} | {dram} |")
    lines.append(f"| **total (libkk_spgemm)** | {sum(p['n'] for p in per.values())} | {tot:.3f} | | 1.000 | |")
    lines.append("")
    lines.append(f"Not counted: {other['n']} PyTorch launches ({other['ms']:.3f} ms) that generate the synthetic "
                 "workload and allocate buffers outside the timed region.")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "ms", "dram_read_bytes", "dram_write_bytes"])
        for d in L:
            w.writerow([d["name"], d.get("gpu__time_duration.sum", ""), d.get("dram__bytes_read.sum", ""),
                        d.get("dram__bytes_write.sum", "")])
    num = {k: v for k, v in per.items() if k.startswith("k_num_")}
    dram_num = sum(v["dram"] / v["n"] for v in num.values())  # per launch of each numeric kernel
    if dram_num:
        json.dump({"tag": tag, "kernels": sorted(num), "dram_bytes_per_step": dram_num,
                   "source": f"profiles/{tag}_launches.csv (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                             f"numeric-phase kernels, per step)"},
                  open(os.path.join(PROF, "dominant_kernel_traffic.json"), "w"), indent=1)
    return per


RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
       "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
       "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def summarize_ncu(tag):
    rep = os.path.join(OUT, f"prof_top_{tag}.ncu-rep")
    if not os.path.exists(rep) and os.path.exists(rep + ".gz"):
        import gzip
        import shutil
        with gzip.open(rep + ".gz", "rb") as fi, open(rep, "wb") as fo:
            shutil.copyfileobj(fi, fo)
    if not os.path.exists(rep):
        return None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ci = {h: k for k, h in enumerate(hdr)}
    lines = [f"# ncu --set full, tag {tag}", "",
             "Source: `ncu --set full --clock-control none --import-source on` on the dominant kernels of the C2 "
             "step (one launch each after warm-up).", ""]
    res = {}
    for r in rows[2:]:
        name = short(r[ci["Kernel Name"]])
        if name in res:
            continue
        res[name] = {m: (r[ci[m]], units[ci[m]]) for m in RAW if m in ci}
        lines.append(f"## `{name}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for m, (v, u) in res[name].items():
            lines.append(f"| {m} | {v} | {u} |")
        lines.append("")
    # stall summary + hottest SASS via tools/ncu_sass_hot.py
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_sass_hot.py"), rep, ".", "12"],
                         capture_output=True, text=True).stdout
    lines += ["## Stall reasons and hottest SASS (warp-stall samples)", "", "```", hot.strip(), "```", ""]
    open(os.path.join(PROF, f"{tag}_ncu_top.md"), "w").write("\n".join(lines))
    return res


def main():
    tag = sys.argv[1]
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 2
    os.makedirs(PROF, exist_ok=True)
    per = summarize_launches(tag, steps)
    res = summarize_ncu(tag)
    b = os.path.join(OUT, f"bench_{tag}.json")
    if os.path.exists(b) and os.path.getsize(b):
        open(os.path.join(PROF, f"{tag}_bench.json"), "w").write(open(b).read())
    print("kernels:", len(per), "ncu:", list(res) if res else None)


if __name__ == "__main__":
    main()
