"""Aggregate ncu warp-stall samples per CUDA source line.

usage: ncu -i R.ncu-rep --page source --csv --print-source cuda,sass > S.csv
       python tools/ncu_lines.py S.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    f = None
    hdr = None
    cur = None
    agg = defaultdict(lambda: [0, 0, ""])
    stall_cols = {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            stall_cols = {i: n for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n}
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0]:
            cur = (f, int(r[0]), r[1][:110])
        if r[2] and cur:
            try:
                s = int(r[4] or 0)
            except ValueError:
                continue
            a = agg[(cur[0], cur[1])]
            a[0] += s
            a[2] = cur[2]
            best = max(stall_cols, key=lambda i: float(r[i] or 0)) if stall_cols else None
            if best is not None and float(r[best] or 0) > 0:
                a.append((stall_cols[best], float(r[best])))
    tot = sum(v[0] for v in agg.values()) or 1
    print("total samples", tot)
    for (fn, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        st = defaultdict(float)
        for x in v[3:]:
            st[x[0]] += x[1]
        s2 = ", ".join(f"{k[6:]}:{int(c)}" for k, c in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print(f"{100 * v[0] / tot:5.1f}% {fn}:{ln}  [{s2}]  {v[2].strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
