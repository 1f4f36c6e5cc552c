"""Staged vs single-call backward on the device: step times and per-kernel event times."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2601_05296_b200 as M  # noqa: E402
from paper_2601_05296_b200 import _lib as L  # noqa: E402
from moe_inputs import CONFIGS, make_inputs  # noqa: E402

res = {}
for W in sys.argv[1:] or ("deepseek",):
    cfg = CONFIGS[W]
    inp = make_inputs(cfg.T, cfg.d, cfg.h, cfg.E, cfg.k, dtype="bf16", seed=0, device="cuda")
    x, wg, w1, w2, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))

    def func(mode):
        logits, ids, w = M.route(x, wg, cfg.k)
        disp = M.dispatch_build(ids, cfg.E)
        y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp)
        if mode == "single":
            M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits)
        elif mode == "staged":
            M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits, staged=True, release_ab=True)
        else:  # staged calls in the single call's order (DW3 before DW12), nothing released
            p = M.layer._problem(cfg.T, cfg.d, cfg.h, cfg.E, cfg.k, x.dtype)
            ws = L.workspace(p, L.MOE_OP_FFN_BWD, x.device)
            dx = torch.empty_like(x)
            dg = torch.empty(cfg.T, cfg.k, dtype=torch.float32, device=x.device)
            dwg = torch.empty_like(wg)
            router = L.MoeRouterBwd(wg.data_ptr(), logits.data_ptr(), disp.ids.data_ptr(), dwg.data_ptr())
            args = (p, dy, x, w1, w2, w3, w, disp.c(), a, b, None)
            L.moe_ffn_bwd(*args, dx, None, None, None, dg, router, ws, stages=L.MOE_BWD_DATA)
            dw3 = torch.empty_like(w3)
            L.moe_ffn_bwd(*args, dx, None, None, dw3, dg, None, ws, stages=L.MOE_BWD_DW3)
            dw1, dw2 = torch.empty_like(w1), torch.empty_like(w2)
            L.moe_ffn_bwd(*args, dx, dw1, dw2, None, dg, None, ws, stages=L.MOE_BWD_DW12)

    def timed(mode, n=20):
        for _ in range(4):
            func(mode)
        torch.cuda.synchronize()
        L.profile_reset()
        L.profile_enable(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            func(mode)
        e1.record()
        torch.cuda.synchronize()
        L.profile_enable(False)
        prof = {k: round(v[0] / max(v[1], 1), 4) for k, v in L.profile_read().items()}
        return {"ms": round(e0.elapsed_time(e1) / n, 4), "kernels": prof}

    for rep in range(2):
        for mode in ("single", "staged", "staged_dw3_first"):
            res[f"{W}_{mode}_{rep}"] = timed(mode)
    del inp, x, wg, w1, w2, w3, dy
    torch.cuda.empty_cache()
print(json.dumps(res, indent=0))
