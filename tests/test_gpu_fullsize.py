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
from tests._util import BF16_TOL, ROW_TOL_BF16, f64, i64, normwise, rowwise

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _sample(n, m, seed):
    return np.sort(np.random.default_rng(seed).choice(n, size=min(m, n), replace=False))


FULL_CASES = [
    # workload, renormalize, activation, deterministic, checkpoint
    ("mixtral", False, "swiglu", False, "ab"), ("deepseek", False, "swiglu", False, "ab"),
    ("sweep_4k", False, "swiglu", False, "ab"), ("ep", False, "swiglu", False, "ab"),
    # the non-default modes at full size
    ("mixtral", True, "swiglu", False, "ab"),          # Mixtral-style renormalised gates
    ("deepseek", False, "silu", False, "ab"),          # non-gated SiLU experts
    ("deepseek", False, "swiglu", True, "ab"),         # ordered combine, k = 6
    ("mixtral", False, "swiglu", False, "abu"),        # Alg. 1 literal checkpoint
]


@pytest.mark.parametrize("name,renorm,act,det,ckpt", FULL_CASES,
                         ids=["-".join(map(str, c)) for c in FULL_CASES])
def test_fullsize_sampled_parity(name, renorm, act, det, ckpt):
    import paper_2601_05296_b200 as M
    cfg = CONFIGS[name]
    T, d, h, E, k = cfg.T, cfg.d, cfg.h, cfg.E, cfg.k
    gated = act == "swiglu"
    inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=0, device=DEV)
    x, wg, w1, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w3", "dy"))
    w2 = inp["w2"] if gated else None
    experts = _sample(E, 2, 2)
    hid = {int(e): _sample(h, 64, 3 + int(e)) for e in experts}
    logits, ids, w = M.route(x, wg, k, renorm)
    disp = M.dispatch_build(ids, E)
    out = M.ffn_fwd(x, w1, w2, w3, w, disp, renorm, checkpoint=ckpt, activation=act, deterministic=det)
    y, a, b = out[:3]
    offs = i64(disp.offs)
    sel = {e: torch.from_numpy(S).to(DEV) for e, S in hid.items()}
    ckpt_a = {e: f64(a[offs[e]:offs[e + 1], sel[e]]) for e in hid}
    ckpt_b = {e: f64(b[offs[e]:offs[e + 1], sel[e]]) for e in hid} if gated else {}
    g = M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits, renormalize=renorm,
                  checkpoint=ckpt, activation=act, deterministic=det, u_save=out[3] if ckpt == "abu" else None)
    torch.cuda.synchronize()

    # routing + dispatch: full, bit-exact
    L = f64(logits)
    _, rids, rw = O.topk_from_logits(L, k, renorm)
    assert np.array_equal(i64(ids), rids)
    assert np.abs(f64(w) - rw).max() < 1e-5
    rd = O.dispatch_argsort(rids, E)
    for key in ("counts", "offs", "eti", "tim", "row_slot"):
        assert np.array_equal(i64(getattr(disp, key)), rd[key]), key

    # sampled tokens: y, dx, dg (full weights, forced routing)
    toks = _sample(T, 48, 1)
    X, DY = f64(x), f64(dy)
    WG, W1, W3 = f64(wg), f64(w1), f64(w3)
    W2 = f64(w2) if gated else None
    fs = O.layer_forward(X[toks], WG, W1, W2, W3, k, renorm, logits=L[toks], activation=act)
    bs = O.layer_backward(fs, DY[toks], X[toks], WG, W1, W2, W3, renorm)
    errs = {"y": normwise(y[toks], fs["y"]), "dx": normwise(g["dx"][toks], bs["dx"]),
            "dg": normwise(g["dg"][toks], bs["dg"])}
    rows = {"y": rowwise(y[toks], fs["y"]), "dx": rowwise(g["dx"][toks], bs["dx"])}

    # sampled (expert, hidden-unit) slices of the weight gradients, all routed rows
    for e, S in hid.items():
        W2s = W2[:, S, :] if gated else None
        sl = O.ffn_forward(X, W1[:, S, :], W2s, W3[:, :, S], rids, rw, rd, act)
        sb = O.ffn_backward(DY, X, W1[:, S, :], W2s, W3[:, :, S], rids, rw, rd, sl["A"], sl["B"], act)
        lo, hi = rd["offs"][e], rd["offs"][e + 1]
        errs[f"A[{e}]"] = normwise(ckpt_a[e], sl["A"][lo:hi])
        errs[f"dw1[{e}]"] = normwise(g["dw1"][e][sel[e]], sb["dw1"][e])
        errs[f"dw3[{e}]"] = normwise(g["dw3"][e][:, sel[e]], sb["dw3"][e])
        rows[f"dw1[{e}]"] = rowwise(g["dw1"][e][sel[e]], sb["dw1"][e])
        if gated:
            errs[f"B[{e}]"] = normwise(ckpt_b[e], sl["B"][lo:hi])
            errs[f"dw2[{e}]"] = normwise(g["dw2"][e][sel[e]], sb["dw2"][e])
    # router backward at full size from the GPU's dg
    rb = O.router_backward(f64(g["dg"]), X, WG, L, rids, renorm)
    errs["dw_gate"] = normwise(g["dw_gate"], rb["dw_gate"])
    bad = {n: v for n, v in errs.items() if not v <= BF16_TOL}
    bad.update({"row:" + n: v for n, v in rows.items() if not v <= ROW_TOL_BF16})
    assert not bad, (name, errs, rows)
    print(name, renorm, act, det, ckpt, {n: round(v, 5) for n, v in errs.items()})


def test_fullsize_deepseek_full_tensors():
    """The DeepSeek-like layer (BASELINE configs[2]) compared on EVERY element of
    every output -- not a sample: the fp64 oracle runs the whole layer (forced
    routing on the GPU's fp32 logits, ~5 TFLOP in fp64 on the host), so dW_g
    here comes from the oracle's own dg, independent of the GPU's."""
    import paper_2601_05296_b200 as M
    cfg = CONFIGS["deepseek"]
    T, d, h, E, k = cfg.T, cfg.d, cfg.h, cfg.E, cfg.k
    inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=0, device=DEV)
    x, wg, w1, w2, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
    logits, ids, w = M.route(x, wg, k)
    disp = M.dispatch_build(ids, E)
    y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp)
    A0, B0 = f64(a), f64(b)
    g = M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits)
    torch.cuda.synchronize()
    X, WG, W1, W2, W3, DY = (f64(t) for t in (x, wg, w1, w2, w3, dy))
    fwd = O.layer_forward(X, WG, W1, W2, W3, k, logits=f64(logits))
    assert np.array_equal(i64(ids), fwd["ids"])
    bwd = O.layer_backward(fwd, DY, X, WG, W1, W2, W3)
    errs = {"A": normwise(A0, fwd["A"]), "B": normwise(B0, fwd["B"]), "y": normwise(y, fwd["y"]),
            "dA": normwise(a, bwd["dA"]), "dB": normwise(b, bwd["dB"]), "dg": normwise(g["dg"], bwd["dg"]),
            "dx": normwise(g["dx"], bwd["dx"]), "dw1": normwise(g["dw1"], bwd["dw1"]),
            "dw2": normwise(g["dw2"], bwd["dw2"]), "dw3": normwise(g["dw3"], bwd["dw3"]),
            "dw_gate": normwise(g["dw_gate"], bwd["dw_gate"])}
    rows = {n: rowwise(g[n] if n in g else y, bwd[n] if n in bwd else fwd["y"]) for n in ("dx", "dw1", "dw3")}
    rows["y"] = rowwise(y, fwd["y"])
    bad = {n: v for n, v in errs.items() if not v <= BF16_TOL}
    bad.update({"row:" + n: v for n, v in rows.items() if not v <= ROW_TOL_BF16})
    print("deepseek full tensors", {n: round(v, 5) for n, v in errs.items()},
          "rowwise", {n: round(v, 5) for n, v in rows.items()})
    assert not bad, (errs, rows)
