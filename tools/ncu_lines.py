"""Per-source-line instruction and stall summary from an exported ncu source page
(--page source --csv --print-source cuda,sass), one block per kernel.

    python tools/ncu_lines.py gpurun_out/src_TAG.csv [kernel-regex] [top] [rows-divisor]
"""
import csv
import re
import sys


def main():
    path = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else None
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    div = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if len(r) >= 2 and r[0] == "Function Name":
            cur = [r[1], None, []]
            blocks.append(cur)
        elif len(r) > 2 and r[0] == "Line No" and cur is not None:
            cur[1] = {h: i for i, h in enumerate(r)}
        elif cur is not None and cur[1] is not None and len(r) > 8 and r[0] not in ("",):
            cur[2].append(r)
    merged = {}
    for name, hdr, data in blocks:
        if kre and not re.search(kre, name):
            continue
        m = merged.setdefault(name, {})
        ie, ws = hdr["Instructions Executed"], hdr["Warp Stall Sampling (All Samples)"]
        for r in data:
            try:
                a, b = float(r[ie] or 0), float(r[ws] or 0)
            except ValueError:
                continue
            k = (r[0], r[1].strip()[:110])
            x = m.setdefault(k, [0.0, 0.0])
            x[0] += a
            x[1] += b
    for name, m in merged.items():
        ti = sum(v[0] for v in m.values())
        ts = sum(v[1] for v in m.values())
        print(f"=== {name[:140]}\n inst={ti:.4g} (/{div:g} = {ti / div:.1f}) samples={ts:.0f}")
        for (ln, src), (a, b) in sorted(m.items(), key=lambda kv: -kv[1][1])[:top]:
            print(f" {a / div:8.1f} {100 * b / max(ts, 1):5.1f}%  L{ln:>5} {src}")


if __name__ == "__main__":
    main()
