"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (same functional API, same kernels), on outputs the fp64 oracle can
compute exactly from a sample:

* y and dX of sampled tokens: the layer is per-token given the routing, so
  the oracle run on the token subset (full weights, forced routing on the
  GPU's fp32 logits) gives those rows exactly;
* dW1[e][S,:], dW2[e][S,:], dW3[e][:,S] for sampled experts e and hidden
  units S: the SwiGLU FFN is separable across hidden units, so the oracle's
  backward on the h-sliced weights (all routed rows of e) gives them exactly;
* dg of sampled tokens; dW_g from the oracle's router backward on the GPU's
  (sampled-checked) dg.
Indices (ids, offsets, eti, tim) are compared in full, bit-exact."""
import numpy as np
import pytest
import torch

import oracle as O
from moe_inputs import CONFIGS, make_inputs
from tests._util import BF16_TOL, f64, i64, normwise

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _sample(n, m, seed):
    return np.sort(np.random.default_rng(seed).choice(n, size=min(m, n), replace=False))


@pytest.mark.parametrize("name", ["mixtral", "deepseek", "sweep_4k", "ep"])
def test_fullsize_sampled_parity(name):
    import paper_2601_05296_b200 as M
    cfg = CONFIGS[name]
    T, d, h, E, k = cfg.T, cfg.d, cfg.h, cfg.E, cfg.k
    inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=0, device=DEV)
    x, wg, w1, w2, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
    experts = _sample(E, 2, 2)
    hid = {int(e): _sample(h, 64, 3 + int(e)) for e in experts}
    logits, ids, w = M.route(x, wg, k)
    disp = M.dispatch_build(ids, E)
    y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp)
    offs = i64(disp.offs)
    ckpt = {e: (f64(a[offs[e]:offs[e + 1], torch.from_numpy(S).to(DEV)]),
                f64(b[offs[e]:offs[e + 1], torch.from_numpy(S).to(DEV)])) for e, S in hid.items()}
    g = M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits)
    torch.cuda.synchronize()

    # routing + dispatch: full, bit-exact
    L = f64(logits)
    _, rids, rw = O.topk_from_logits(L, k)
    assert np.array_equal(i64(ids), rids)
    assert np.abs(f64(w) - rw).max() < 1e-5
    rd = O.dispatch_argsort(rids, E)
    for key in ("counts", "offs", "eti", "tim", "row_slot"):
        assert np.array_equal(i64(getattr(disp, key)), rd[key]), key

    # sampled tokens: y, dx, dg (full weights, forced routing)
    toks = _sample(T, 48, 1)
    X, DY = f64(x), f64(dy)
    WG, W1, W2, W3 = f64(wg), f64(w1), f64(w2), f64(w3)
    fs = O.layer_forward(X[toks], WG, W1, W2, W3, k, logits=L[toks])
    bs = O.layer_backward(fs, DY[toks], X[toks], WG, W1, W2, W3)
    errs = {"y": normwise(y[toks], fs["y"]), "dx": normwise(g["dx"][toks], bs["dx"]),
            "dg": normwise(g["dg"][toks], bs["dg"])}

    # sampled (expert, hidden-unit) slices of the weight gradients, all routed rows
    for e, S in hid.items():
        sl = O.ffn_forward(X, W1[:, S, :], W2[:, S, :], W3[:, :, S], rids, rw, rd)
        sb = O.ffn_backward(DY, X, W1[:, S, :], W2[:, S, :], W3[:, :, S], rids, rw, rd, sl["A"], sl["B"])
        lo, hi = rd["offs"][e], rd["offs"][e + 1]
        errs[f"A[{e}]"] = normwise(ckpt[e][0], sl["A"][lo:hi])
        errs[f"B[{e}]"] = normwise(ckpt[e][1], sl["B"][lo:hi])
        errs[f"dw1[{e}]"] = normwise(g["dw1"][e][torch.from_numpy(S).to(DEV)], sb["dw1"][e])
        errs[f"dw2[{e}]"] = normwise(g["dw2"][e][torch.from_numpy(S).to(DEV)], sb["dw2"][e])
        errs[f"dw3[{e}]"] = normwise(g["dw3"][e][:, torch.from_numpy(S).to(DEV)], sb["dw3"][e])
    # router backward at full size from the GPU's dg
    rb = O.router_backward(f64(g["dg"]), X, WG, L, rids)
    errs["dw_gate"] = normwise(g["dw_gate"], rb["dw_gate"])
    bad = {n: v for n, v in errs.items() if not v <= BF16_TOL}
    assert not bad, (name, errs)
    print(name, {n: round(v, 5) for n, v in errs.items()})
