"""Where does the host-fed (e2e) DeepSeek-like step lose time?  Per-step CUDA-event
times of the autograd layer (a) device-resident, (b) with the H2D copies only, (c) with
the D2H copies only, (d) both (HostPipeline, as bench.py's e2e leg), (e) the functional
API device-resident."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2601_05296_b200 as M  # noqa: E402
from moe_inputs import CONFIGS, make_inputs  # noqa: E402
from paper_2601_05296_b200.pipeline import HostPipeline  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "deepseek"]
dev = torch.device("cuda", 0)
inp = make_inputs(cfg.T, cfg.d, cfg.h, cfg.E, cfg.k, dtype="bf16", seed=0, device=dev)
x, wg, w1, w2, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
params = [torch.nn.Parameter(t) for t in (wg, w1, w2, w3)]
k = cfg.k


def layer_step(xd, dyd):
    xl = xd.detach().requires_grad_(True)
    for p in params:
        p.grad = None
    y = M.moe_layer(xl, *params, k)
    y.backward(dyd)
    return y, xl.grad


def timed(fn, n=30, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


x_h = x.cpu().pin_memory()
dy_h = dy.cpu().pin_memory()
outs = [torch.empty_like(x_h).pin_memory() for _ in range(2)]
res = {}
res["a_device_autograd"] = timed(lambda: layer_step(x, dy))


def func_step():
    logits, ids, w = M.route(x, wg, k)
    disp = M.dispatch_build(ids, cfg.E)
    y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp)
    M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits)


res["e_device_functional"] = timed(func_step)
xs = [torch.empty_like(x) for _ in range(2)]
dys = [torch.empty_like(dy) for _ in range(2)]
h2d = torch.cuda.Stream()
d2h = torch.cuda.Stream()
cnt = [0]


def h2d_only():
    i = cnt[0] % 2
    cnt[0] += 1
    with torch.cuda.stream(h2d):
        xs[i].copy_(x_h, non_blocking=True)
        dys[i].copy_(dy_h, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(h2d)
    torch.cuda.current_stream().wait_event(ev)
    layer_step(xs[i], dys[i])


res["b_h2d_only"] = timed(h2d_only)


def d2h_only():
    i = cnt[0] % 2
    cnt[0] += 1
    y, gx = layer_step(x, dy)
    ev = torch.cuda.Event()
    ev.record()
    with torch.cuda.stream(d2h):
        d2h.wait_event(ev)
        outs[i].copy_(y, non_blocking=True)
        outs[1 - i].copy_(gx, non_blocking=True)
    y.record_stream(d2h)
    gx.record_stream(d2h)


res["c_d2h_only"] = timed(d2h_only)
pipe = HostPipeline(layer_step, x.shape, x.dtype, dev)
ys = [torch.empty_like(x_h).pin_memory() for _ in range(2)]
dxs = [torch.empty_like(x_h).pin_memory() for _ in range(2)]
for _ in range(2):
    pipe.run([x_h] * 5, [dy_h] * 5, [ys[i % 2] for i in range(5)], [dxs[i % 2] for i in range(5)])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
pipe.run([x_h] * 30, [dy_h] * 30, [ys[i % 2] for i in range(30)], [dxs[i % 2] for i in range(30)])
e1.record()
torch.cuda.synchronize()
res["d_pipeline_both"] = e0.elapsed_time(e1) / 30
res["host_time_per_step_ms"] = None
t0 = time.time()
for _ in range(10):
    layer_step(x, dy)
res["host_enqueue_ms_per_step"] = round((time.time() - t0) * 100, 3)
torch.cuda.synchronize()
print(json.dumps({n: (round(v, 4) if isinstance(v, float) else v) for n, v in res.items()}))
