"""Warp-stall samples of one kernel per call site in gemm_tc.cu (inlined helpers
attributed to the line that calls them), from an ncu SASS source page and the
exact library that was profiled.

usage: ncu -i R.ncu-rep --page source --csv --print-source sass > S.csv
       python tools/ncu_callsites.py S.csv lib.so '<mangled kernel>' [top]
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_map(so, kernel):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True, check=True)
    out = {}
    for f in os.listdir(tmp):
        txt = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, f)], capture_output=True, text=True).stdout
        at = txt.find(f".text.{kernel}:")
        if at < 0:
            continue
        cur = None
        for ln in txt[at:].splitlines()[1:]:
            if ln.startswith(".text."):
                break
            m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
            if m:
                fn, l, ifn, il = m.groups()
                if fn.endswith("gemm_tc.cu"):
                    cur = int(l)
                elif ifn and ifn.endswith("gemm_tc.cu"):
                    cur = int(il)
                else:
                    cur = None if not cur else cur
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
            if m:
                out[int(m.group(1), 16)] = (cur, m.group(2).strip()[:60])
        return out
    raise SystemExit(f"kernel {kernel} not found in {so}")


def main(path, so, kernel, top=40):
    lm = line_map(so, kernel)
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    ia, isamp = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    stall = {i: n for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n}
    data = [r for r in rows if len(r) == len(hdr) and r[ia].startswith("0x")]
    base = int(data[0][ia], 16)
    agg = collections.defaultdict(lambda: [0, collections.Counter()])
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2601_05296_b200", "csrc", "gemm_tc.cu")).read().splitlines()
    for r in data:
        off = int(r[ia], 16) - base
        n = int(float(r[isamp] or 0))
        if not n:
            continue
        line = lm.get(off, (None, ""))[0]
        a = agg[line]
        a[0] += n
        for i, nm in stall.items():
            v = float(r[i] or 0)
            if v:
                a[1][nm[6:]] += v
    tot = sum(v[0] for v in agg.values()) or 1
    print("total samples", tot)
    for line, (n, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        txt = src[line - 1].strip()[:90] if line else "?"
        s3 = ", ".join(f"{k}:{int(v)}" for k, v in st.most_common(3))
        print(f"{100 * n / tot:5.1f}% gemm_tc.cu:{line}  [{s3}]  {txt}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
