"""Regenerate profiles/ncu_traffic.json (bench.py's roofline `traffic`) from ncu launch lists.

Per expert-GEMM kind: mean over its launches of dram__bytes_read.sum +
dram__bytes_write.sum (bytes per launch).  Kind ids follow TcKind in
csrc/gemm_tc.cu (BWD_DH_LK = 7 is the BWD_DH kind's long-K engine).
usage: python tools/ncu_traffic.py TAG   (reads profiles/launches_TAG_{mixtral,deepseek}.csv)"""
import csv
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {0: "FWD_UP", 1: "FWD_DOWN", 2: "BWD_DH", 7: "BWD_DH", 9: "BWD_DH", 3: "BWD_DX", 4: "DW3", 5: "DW12"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def traffic(path):
    per = defaultdict(float)  # (launch id) -> bytes
    kind = {}
    for r in csv.DictReader(l for l in open(path) if not l.startswith("==")):
        m = re.search(r"tc_gemm_kernel<(\d+),", r["Kernel Name"])
        if not m or int(m.group(1)) not in NAMES:
            continue
        if r["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v = float(r["Metric Value"].replace(",", ""))
            per[r["ID"]] += v * UNIT[r["Metric Unit"]]
            kind[r["ID"]] = NAMES[int(m.group(1))]
    acc = defaultdict(list)
    for i, b in per.items():
        acc[kind[i]].append(b)
    return {k: int(sum(v) / len(v)) for k, v in acc.items()}


if __name__ == "__main__":
    tag = sys.argv[1]
    out = {w: traffic(os.path.join(ROOT, "profiles", f"launches_{tag}_{w}.csv")) for w in ("mixtral", "deepseek")}
    out["source"] = f"profiles/launches_{tag}_{{mixtral,deepseek}}.csv (tools/ncu_traffic.py)"
    json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))
