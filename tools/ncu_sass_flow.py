"""Per-instruction execution counts of one kernel in an ncu report, normalised by a unit
count (e.g. warp steps), to read the instruction budget of a loop.

    python tools/ncu_sass_flow.py REPORT KERNEL_REGEX UNITS [min_per_unit]
"""
import csv
import io
import re
import subprocess
import sys

rep, kre, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
mn = float(sys.argv[4]) if len(sys.argv) > 4 else 0.05
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for b in re.split(r'(?m)^"Kernel Name",', out)[1:]:
    name = b.split("\n", 1)[0]
    if not re.search(kre, name):
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    hdr = rows[0]
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    ci = {h: i for i, h in enumerate(hdr)}
    IE, S = ci["Instructions Executed"], ci["Warp Stall Sampling (All Samples)"]
    tot = sum(float(r[IE] or 0) for r in data)
    ts = sum(float(r[S] or 0) for r in data)
    print(name[:120])
    for k, r in enumerate(data):
        ie = float(r[IE] or 0)
        if ie / units >= mn:
            print(f"{k:4d} {ie / units:6.2f} thr={r[ci['Avg. Threads Executed']]:>3} samp={100 * float(r[S] or 0) / ts:5.2f}% "
                  f"{r[ci['Source']].strip()[:80]}")
    print("per-unit total", tot / units)
    break
