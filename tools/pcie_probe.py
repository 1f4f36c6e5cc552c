"""Host<->device copy bandwidth on this box, for reading bench.py's e2e number.

Times (CUDA events) the per-step copies of the e2e leg at the DeepSeek-like
size (X and dY in, Y and dX out: 2 x 67 MB each way, pinned): H2D alone, D2H
alone, both directions at once on two streams.  No library code is used.
usage: python tools/pcie_probe.py [T] [d]"""
import json
import sys

import torch

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
d = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
dev = torch.device("cuda", 0)
nbytes = 2 * T * d * 2
hin = [torch.empty(T, d, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
hout = [torch.empty(T, d, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
din = [torch.empty(T, d, dtype=torch.bfloat16, device=dev) for _ in range(2)]
dout = [torch.ones(T, d, dtype=torch.bfloat16, device=dev) for _ in range(2)]
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        s1.wait_stream(torch.cuda.current_stream())
        for a, b in zip(din, hin):
            a.copy_(b, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        s2.wait_stream(torch.cuda.current_stream())
        for a, b in zip(hout, dout):
            a.copy_(b, non_blocking=True)


def both():
    h2d()
    d2h()


out = {"bytes_each_way": nbytes}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    out[name] = {"ms": round(ms, 3), "GB/s_each_way": round(nbytes / ms / 1e6, 1)}
print(json.dumps(out))
