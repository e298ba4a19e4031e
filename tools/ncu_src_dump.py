"""Dump an exported ncu source page (--page source --csv --print-source sass or cuda,sass)
as executed-instruction counts and shared wavefronts per SASS line.

    python tools/ncu_src_dump.py gpurun_out/src_TAG.csv [kernel-regex] [min_exec_fraction]
"""
import csv
import io
import re
import sys


def main():
    path = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else None
    minf = float(sys.argv[3]) if len(sys.argv) > 3 else 0.002
    out = open(path).read()
    blocks = re.split(r'(?m)^"Kernel Name",', out)
    for b in blocks[1:]:
        name = b.split("\n", 1)[0]
        if kre and not re.search(kre, name):
            continue
        body = b.split("\n", 1)[1]
        # with cuda,sass the sass table follows the cuda table; take the one with "Address"
        tables = re.split(r'\n(?=")', body)
        rows = list(csv.reader(io.StringIO(body)))
        hdr_i = [i for i, r in enumerate(rows) if r and r[0] in ("Address", "# Address")]
        if not hdr_i:
            hdr_i = [0]
        hdr = rows[hdr_i[-1]]
        data = [r for r in rows[hdr_i[-1] + 1:] if len(r) == len(hdr)]
        ci = {h: i for i, h in enumerate(hdr)}
        IE = ci["Instructions Executed"]
        tot = sum(float(r[IE] or 0) for r in data)
        wf = ci.get("L1 Wavefronts Shared")
        wfi = ci.get("L1 Wavefronts Shared Ideal")
        print(f"=== {name[:120]}  warp-instructions={tot:.4e}")
        tw = sum(float(r[wf] or 0) for r in data) if wf is not None else 0
        print(f"shared wavefronts={tw:.4e}")
        for i, r in enumerate(data):
            ie = float(r[IE] or 0)
            if ie < minf * tot / 100:
                continue
            w = r[wf] if wf is not None else ""
            wi = r[wfi] if wfi is not None else ""
            print(f"{i:5d} {ie / 1e6:9.3f}M {w:>10} {wi:>10}  {r[ci['Source']].strip()[:90]}")


if __name__ == "__main__":
    main()
