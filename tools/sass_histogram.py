"""Per-kernel SASS instruction histogram of libmoeblaze.so (cuobjdump -sass).

Counts the mnemonics that prove the sm_100a data path: UTCHMMA / UTCBAR
(tcgen05.mma / commit), LDTM (tcgen05.ld), UTMALDG / UTMASTG / UTMAPF (TMA
load / store / L2 prefetch), LDGSTS (cp.async), REDG (red.global), HMMA (legacy
mma.sync: must be 0 on the expert GEMMs), MUFU (SFU: exp / rcp), SYNCS (mbarrier).

usage: python tools/sass_histogram.py [lib.so] > profiles/sass_histogram_rNN.txt
"""
import collections
import re
import subprocess
import sys

KEYS = ("UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UTMAPF", "UTMAREDG", "LDGSTS", "REDG", "HMMA", "MUFU",
        "SYNCS", "FFMA", "LDS", "STS", "LDG", "STG")


def main(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    kern, hist = None, collections.OrderedDict()
    for ln in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            kern = m.group(1)
            hist[kern] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", ln)
        if m and kern:
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k):
                    hist[kern][k] += 1
                    break
    demangle = subprocess.run(["c++filt"], input="\n".join(hist), capture_output=True, text=True).stdout.split("\n")
    print("kernel\t" + "\t".join(KEYS))
    for (k, h), name in zip(hist.items(), demangle):
        name = re.sub(r"\(.*", "", name).replace("moeb::", "")
        print(name[:70] + "\t" + "\t".join(str(h[x]) for x in KEYS))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2601_05296_b200/libmoeblaze.so")
