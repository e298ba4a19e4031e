"""Summarise an ncu report's SASS source page: hottest instructions by stall samples and
by executed instructions, plus the stall-reason totals.

    python tools/ncu_sass_hot.py gpurun_out/prof.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import re
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else None
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', out)
    for b in blocks[1:]:
        name = b.split("\n", 1)[0]
        if kre and not re.search(kre, name):
            continue
        rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
        hdr = rows[0]
        data = [r for r in rows[1:] if len(r) == len(hdr)]
        ci = {h: i for i, h in enumerate(hdr)}
        S, IE = ci["Warp Stall Sampling (All Samples)"], ci["Instructions Executed"]
        tot_s = sum(float(r[S] or 0) for r in data)
        tot_i = sum(float(r[IE] or 0) for r in data)
        print(f"=== {name[:150]}\n samples={tot_s:.0f} warp-instructions={tot_i:.3e} sass={len(data)}")
        stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        tots = {h: sum(float(r[ci[h]] or 0) for r in data) for h in stalls}
        print(" stalls:", ", ".join(f"{h[6:]}={100 * v / max(tot_s, 1):.1f}%" for h, v in
                                    sorted(tots.items(), key=lambda x: -x[1]) if v > 0.005 * tot_s))
        print(f" {'addr':>6} {'samp%':>6} {'inst%':>6} {'thr':>5} {'shWF':>9} {'shIdeal':>9}  sass")
        order = sorted(range(len(data)), key=lambda i: -float(data[i][S] or 0))[:top]
        for i in sorted(order):
            r = data[i]
            print(f" {i:6d} {100 * float(r[S] or 0) / max(tot_s, 1):6.2f} {100 * float(r[IE] or 0) / max(tot_i, 1):6.2f} "
                  f"{r[ci['Avg. Threads Executed']]:>5} {r[ci['L1 Wavefronts Shared']]:>9} "
                  f"{r[ci['L1 Wavefronts Shared Ideal']]:>9}  {r[ci['Source']].strip()[:90]}")


if __name__ == "__main__":
    main()
