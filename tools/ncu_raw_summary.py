"""Summarise one `ncu --set full` capture (exported with `ncu -i X.ncu-rep --page raw --csv`)
into a tracked markdown table under profiles/.

    python tools/ncu_raw_summary.py gpurun_out/raw_hub_r2c.csv profiles/r2c_ncu_hub_C4.md "title" "source line"

Key counters of every captured launch (time, DRAM bytes, throughputs, occupancy, issue
activity, LSU wavefronts) and the warp-stall shares from the PC sampler.
"""
from __future__ import annotations

import csv
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def main():
    src, dst, title, how = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else ""
    rows = list(csv.reader(open(src)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {n: i for i, n in enumerate(head)}
    out = [f"# {title}", ""]
    if how:
        out += [how, ""]
    for r in data:
        out += [f"Kernel: `{r[col['Kernel Name']][:160]}`", "", "| metric | value | unit |", "|---|---|---|"]
        for k in KEYS:
            if k in col and r[col[k]] != "":
                v = r[col[k]].replace(",", "")
                u = units[col[k]]
                try:
                    x = float(v)
                    if k == "gpu__time_duration.sum" and u == "ns":
                        x, u = x / 1e6, "ms"
                    elif k == "gpu__time_duration.sum" and u == "us":
                        x, u = x / 1e3, "ms"
                    v = f"{x:.6g}"
                except ValueError:
                    pass
                out.append(f"| {k} | {v} | {u} |")
        st = {}
        for n, i in col.items():
            if n.startswith(STALL) and not n.endswith("_not_issued") and r[i] not in ("", "n/a"):
                try:
                    st[n[len(STALL):]] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values())
        if tot > 0:
            top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
            out += ["", "Stall reasons (share of warp-stall samples): " +
                    ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top)]
        out.append("")
    open(dst, "w").write("\n".join(out) + "\n")
    print(f"wrote {dst} ({len(data)} launch(es))")


if __name__ == "__main__":
    main()
