"""Host issue time per step vs device time per step (is the bench step host-bound?)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2601_05296_b200 as M
from moe_inputs import CONFIGS, make_inputs

wl = sys.argv[1] if len(sys.argv) > 1 else "deepseek"
cfg = CONFIGS[wl]
inp = make_inputs(cfg.T, cfg.d, cfg.h, cfg.E, cfg.k, dtype=cfg.dtype, seed=0, device="cuda")
x, wg, w1, w2, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))


def step():
    logits, ids, w = M.route(x, wg, cfg.k)
    disp = M.dispatch_build(ids, cfg.E, dtype=x.dtype)
    y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp)
    return M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits)


for _ in range(5):
    step()
torch.cuda.synchronize()
n = 30
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for _ in range(n):
    step()
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"{wl}: host issue {1e3 * (t1 - t0) / n:.3f} ms/step, device {e0.elapsed_time(e1) / n:.3f} ms/step, "
      f"wall {1e3 * (t2 - t0) / n:.3f} ms/step")
