"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same
seeded inputs.  Index structures bit-exact; bf16 within 2e-2 and fp32 within
1e-4 normwise max-relative error (BASELINE.json north_star, reading #18)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
from moe_inputs import make_inputs, make_ids
from tests._util import BF16_TOL, FP32_TOL, f64, i64, normwise

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def M():
    from paper_2601_05296_b200 import build as B
    B.build()
    import paper_2601_05296_b200 as M
    M._lib.load()
    return M


# ------------------------------------------------------------------ K2 dispatch
def _check_dispatch(M, ids_np, E):
    ids = torch.from_numpy(ids_np.astype(np.int32)).to(DEV)
    d = M.dispatch_build(ids, E)
    torch.cuda.synchronize()
    ref = O.dispatch_argsort(ids_np, E)
    assert np.array_equal(i64(d.counts), ref["counts"])
    assert np.array_equal(i64(d.offs), ref["offs"])
    assert np.array_equal(i64(d.eti), ref["eti"])
    assert np.array_equal(i64(d.tim), ref["tim"])
    assert np.array_equal(i64(d.row_slot), ref["row_slot"])


def test_dispatch_fig2(M):
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig2_dispatch.json")))
    ids = np.array(g["ids"], dtype=np.int32)
    _check_dispatch(M, ids, g["E"])
    d = M.dispatch_build(torch.from_numpy(ids).to(DEV), g["E"])
    assert d.eti.tolist() == g["expected"]["expert_token_indices"]
    assert d.tim.tolist() == g["expected"]["token_index_map"]


@pytest.mark.parametrize("T,E,k,kind", [
    (1, 1, 1, "random"), (1, 8, 8, "random"), (5, 4, 2, "random"), (257, 4, 2, "random"),
    (4097, 8, 2, "random"), (3000, 64, 6, "random"), (9000, 16, 2, "skewed"), (777, 8, 8, "random"),
    (4100, 4, 1, "random"), (2048, 256, 16, "random"), (70001, 8, 2, "random"), (20000, 64, 8, "skewed"),
    (1000, 16, 3, "degenerate"),
])
def test_dispatch_random(M, T, E, k, kind):
    _check_dispatch(M, make_ids(T, E, k, seed=T + E, kind=kind).numpy(), E)


def test_dispatch_large_multi_tile(M):
    # R = 1.05M entries -> 256 tiles of 4096 entries (tile size doubling path)
    _check_dispatch(M, make_ids(131072, 16, 8, seed=1, kind="skewed").numpy(), 16)


def test_dispatch_check_routing(M):
    ids = torch.tensor([[0, 1], [2, 2], [3, 0]], dtype=torch.int32, device=DEV)
    d = M.dispatch_build(ids, 4, check_routing=True)
    torch.cuda.synchronize()
    assert int(d.status.item()) == 5
    ok = M.dispatch_build(torch.tensor([[0, 1], [2, 3]], dtype=torch.int32, device=DEV), 4, check_routing=True)
    torch.cuda.synchronize()
    assert int(ok.status.item()) == 0


# ------------------------------------------------------------------ K1 routing
@pytest.mark.parametrize("T,d,E,k,dtype,renorm", [
    (256, 64, 4, 2, "fp32", False), (1000, 256, 8, 2, "bf16", False), (777, 512, 64, 6, "bf16", True),
    (300, 128, 256, 16, "bf16", False), (33, 128, 16, 1, "bf16", False),
])
def test_route(M, T, d, E, k, dtype, renorm):
    inp = make_inputs(T, d, 128, E, k, dtype=dtype, seed=T, device=DEV, with_dy=False)
    logits, ids, w = M.route(inp["x"], inp["w_gate"], k, renorm)
    torch.cuda.synchronize()
    ref = O.route(f64(inp["x"]), f64(inp["w_gate"]), k, renorm)
    assert normwise(logits, ref["logits"]) < (FP32_TOL if dtype == "fp32" else 1e-5)
    # ids bit-exact vs the oracle's top-k on the GPU's own fp32 logits (reading #4)
    p, rids, rw = O.topk_from_logits(f64(logits), k, renorm)
    assert np.array_equal(i64(ids), rids)
    assert np.abs(f64(w) - rw).max() < 1e-5


# ------------------------------------------------------------------ whole layer
LAYER_CASES = [
    # name, T, d, h, E, k, dtype, renorm, routing
    ("tiny_fp32", 256, 64, 128, 4, 2, "fp32", False, "balanced"),
    ("tiny_fp32_renorm", 200, 64, 96, 6, 3, "fp32", True, "skewed"),
    ("small_bf16", 512, 256, 384, 8, 2, "bf16", False, "balanced"),
    ("ragged_bf16", 1000, 128, 256, 16, 6, "bf16", True, "skewed"),
    ("degenerate_bf16", 300, 128, 128, 8, 2, "bf16", False, "degenerate"),
    ("k1_bf16", 333, 256, 256, 4, 1, "bf16", False, "balanced"),
    # h % 256 == 128: BWD_DH / DW3 run their last n-tile as an N = 128 MMA
    ("h_tail_bf16", 700, 256, 640, 8, 2, "bf16", False, "balanced"),
    # d >= 3072: BWD_DH runs its long-K variant (5 stages, 16-column epilogue chunks)
    ("long_k_bf16", 300, 3072, 384, 4, 2, "bf16", False, "skewed"),
]


def _run_layer(M, T, d, h, E, k, dtype, renorm, routing, seed=0, det=False):
    inp = make_inputs(T, d, h, E, k, dtype=dtype, seed=seed, routing=routing, device=DEV)
    x, wg, w1, w2, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
    logits, ids, w = M.route(x, wg, k, renorm)
    disp = M.dispatch_build(ids, E, dtype=x.dtype)
    y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp, renorm, deterministic=det)
    a0, b0 = a.clone(), b.clone()
    g = M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits, renormalize=renorm,
                  deterministic=det)
    torch.cuda.synchronize()
    out = dict(logits=logits, ids=ids, w=w, y=y, A=a0, B=b0, dA=a, dB=b, disp=disp, **g)
    return inp, out


@pytest.mark.parametrize("case", LAYER_CASES, ids=[c[0] for c in LAYER_CASES])
def test_layer_fwd_bwd_parity(M, case):
    name, T, d, h, E, k, dtype, renorm, routing = case
    inp, out = _run_layer(M, T, d, h, E, k, dtype, renorm, routing)
    tol = FP32_TOL if dtype == "fp32" else BF16_TOL
    X, WG, W1, W2, W3, DY = (f64(inp[n]) for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
    fwd = O.layer_forward(X, WG, W1, W2, W3, k, renorm, logits=f64(out["logits"]))
    assert np.array_equal(i64(out["ids"]), fwd["ids"])
    bwd = O.layer_backward(fwd, DY, X, WG, W1, W2, W3, renorm)
    for key in ("offs", "eti"):
        assert np.array_equal(i64(getattr(out["disp"], key)), fwd["disp"][key])
    errs = {
        "A": normwise(out["A"], fwd["A"]), "B": normwise(out["B"], fwd["B"]), "y": normwise(out["y"], fwd["y"]),
        "dA": normwise(out["dA"], bwd["dA"]), "dB": normwise(out["dB"], bwd["dB"]),
        "dg": normwise(out["dg"], bwd["dg"]), "dx": normwise(out["dx"], bwd["dx"]),
        "dw1": normwise(out["dw1"], bwd["dw1"]), "dw2": normwise(out["dw2"], bwd["dw2"]),
        "dw3": normwise(out["dw3"], bwd["dw3"]), "dw_gate": normwise(out["dw_gate"], bwd["dw_gate"]),
    }
    bad = {kk: v for kk, v in errs.items() if not v <= tol}
    assert not bad, (name, errs)
    if routing == "degenerate":
        # experts k..E-1 got no rows: their weight grads are exact zeros
        assert torch.count_nonzero(out["dw1"][k:]).item() == 0
        assert torch.count_nonzero(out["dw3"][k:]).item() == 0


def test_zero_tokens(M):
    x = torch.empty(0, 128, dtype=torch.bfloat16, device=DEV)
    inp = make_inputs(4, 128, 128, 4, 2, dtype="bf16", device=DEV)
    logits, ids, w = M.route(x, inp["w_gate"], 2)
    disp = M.dispatch_build(ids, 4)
    y, a, b = M.ffn_fwd(x, inp["w1"], inp["w2"], inp["w3"], w, disp)
    g = M.ffn_bwd(torch.empty_like(x), x, inp["w1"], inp["w2"], inp["w3"], w, disp, a, b, w_gate=inp["w_gate"],
                  logits=logits)
    torch.cuda.synchronize()
    assert disp.offs.tolist() == [0, 0, 0, 0, 0]
    assert y.shape == (0, 128)
    for n in ("dw1", "dw2", "dw3", "dw_gate"):
        assert torch.count_nonzero(g[n]).item() == 0


def test_autograd_layer_matches_functional(M):
    inp = make_inputs(256, 128, 256, 8, 2, dtype="bf16", seed=3, device=DEV)
    x = inp["x"].clone().requires_grad_(True)
    params = [inp[n].clone().requires_grad_(True) for n in ("w_gate", "w1", "w2", "w3")]
    y = M.moe_layer(x, *params, 2)
    y.backward(inp["dy"])
    _, out = _run_layer(M, 256, 128, 256, 8, 2, "bf16", False, "balanced", seed=3)
    assert torch.equal(y, out["y"])
    assert torch.equal(x.grad, out["dx"])
    assert torch.equal(params[1].grad, out["dw1"])


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_checkpoint_none_recompute_is_bit_identical(M, dtype):
    """checkpoint="none" (NEXT-3): A, B are not saved; backward recomputes them
    with the same kernel, so every gradient is bit-identical to the paper's
    A,B-checkpoint policy, and the autograd saved set loses the 2*T*k*h
    pre-activations."""
    T, d, h, E, k = (512, 256, 384, 8, 2) if dtype == "bf16" else (256, 64, 128, 4, 2)
    inp = make_inputs(T, d, h, E, k, dtype=dtype, seed=11, device=DEV)
    outs = {}
    for ck in ("ab", "none"):
        x = inp["x"].clone().requires_grad_(True)
        params = [inp[n].clone().requires_grad_(True) for n in ("w_gate", "w1", "w2", "w3")]
        saved = {}

        def pack(t):
            saved[t.untyped_storage().data_ptr()] = t.untyped_storage().nbytes()
            return t

        with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
            y = M.moe_layer(x, *params, k, False, ck)
        y.backward(inp["dy"])
        torch.cuda.synchronize()
        outs[ck] = (y, x.grad, [p.grad for p in params], sum(saved.values()))
    for a_, b_ in zip([outs["ab"][0], outs["ab"][1]] + outs["ab"][2], [outs["none"][0], outs["none"][1]] + outs["none"][2]):
        assert torch.equal(a_, b_)
    esz = 2 if dtype == "bf16" else 4
    assert outs["ab"][3] - outs["none"][3] == 2 * T * k * h * esz


EDGE_CASES = [
    # T, d, h, E, k, routing
    (1, 128, 128, 1, 1, "balanced"),        # one token, one expert
    (3, 128, 128, 256, 16, "balanced"),     # max E and k, nearly all experts empty
    (130, 128, 128, 256, 16, "skewed"),     # max E and k, ragged
    (257, 256, 128, 2, 2, "balanced"),      # k = E: every token to every expert
    (129, 128, 256, 16, 1, "degenerate"),   # all rows to expert 0
    (1023, 384, 640, 12, 5, "skewed"),      # odd sizes (d, h multiples of 128 only)
]


@pytest.mark.parametrize("T,d,h,E,k,routing", EDGE_CASES)
def test_layer_edge_shapes(M, T, d, h, E, k, routing):
    inp, out = _run_layer(M, T, d, h, E, k, "bf16", False, routing, seed=T + E)
    X, WG, W1, W2, W3, DY = (f64(inp[n]) for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
    fwd = O.layer_forward(X, WG, W1, W2, W3, k, False, logits=f64(out["logits"]))
    assert np.array_equal(i64(out["ids"]), fwd["ids"])
    bwd = O.layer_backward(fwd, DY, X, WG, W1, W2, W3, False)
    errs = {n: normwise(out[n], fwd[n] if n in ("A", "B", "y") else bwd[n])
            for n in ("A", "B", "y", "dA", "dB", "dg", "dx", "dw1", "dw2", "dw3", "dw_gate")}
    bad = {n: v for n, v in errs.items() if not v <= BF16_TOL}
    assert not bad, errs
    counts = i64(out["disp"].counts)
    empty = np.nonzero(counts == 0)[0]
    if len(empty):  # experts with no rows: exact zero gradients
        sel = torch.from_numpy(empty).to(DEV)
        assert torch.count_nonzero(out["dw1"][sel]).item() == 0
        assert torch.count_nonzero(out["dw3"][sel]).item() == 0


NONGATED_CASES = [
    # name, T, d, h, E, k, dtype, act
    ("silu_fp32", 256, 64, 128, 4, 2, "fp32", "silu"),
    ("relu_fp32", 200, 64, 96, 6, 3, "fp32", "relu"),
    ("silu_bf16", 512, 256, 384, 8, 2, "bf16", "silu"),      # h % 256 == 128 (half n-tile)
    ("relu_bf16", 1000, 128, 512, 16, 4, "bf16", "relu"),
    ("silu_bf16_k1", 333, 256, 256, 4, 1, "bf16", "silu"),
]


@pytest.mark.parametrize("case", NONGATED_CASES, ids=[c[0] for c in NONGATED_CASES])
@pytest.mark.parametrize("ckpt", ["ab", "none"])
def test_nongated_fwd_bwd_parity(M, case, ckpt):
    """Non-gated experts W2 sigma(W1 x) (NEXT-2): y, dX, dW1, dW3, dW_g, dg
    vs the oracle (w2 is not used: passed as None)."""
    name, T, d, h, E, k, dtype, act = case
    inp = make_inputs(T, d, h, E, k, dtype=dtype, seed=T, device=DEV)
    x, wg, w1, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w3", "dy"))
    logits, ids, w = M.route(x, wg, k)
    disp = M.dispatch_build(ids, E, dtype=x.dtype)
    y, a, b = M.ffn_fwd(x, w1, None, w3, w, disp, checkpoint=ckpt, activation=act)
    assert b is None
    a0 = a.clone() if a is not None else None
    g = M.ffn_bwd(dy, x, w1, None, w3, w, disp, a, b, w_gate=wg, logits=logits, checkpoint=ckpt, activation=act)
    torch.cuda.synchronize()
    assert g["dw2"] is None
    tol = FP32_TOL if dtype == "fp32" else BF16_TOL
    X, WG, W1, W3, DY = (f64(inp[n]) for n in ("x", "w_gate", "w1", "w3", "dy"))
    fwd = O.layer_forward(X, WG, W1, None, W3, k, logits=f64(logits), activation=act)
    bwd = O.layer_backward(fwd, DY, X, WG, W1, None, W3)
    errs = {"y": normwise(y, fwd["y"]), "dx": normwise(g["dx"], bwd["dx"]), "dw1": normwise(g["dw1"], bwd["dw1"]),
            "dw3": normwise(g["dw3"], bwd["dw3"]), "dw_gate": normwise(g["dw_gate"], bwd["dw_gate"]),
            "dg": normwise(g["dg"], bwd["dg"])}
    if a0 is not None:
        errs["A"] = normwise(a0, fwd["A"])
        errs["dA"] = normwise(a, bwd["dA"])
    bad = {n: v for n, v in errs.items() if not v <= tol}
    assert not bad, (name, ckpt, errs)


DET_CASES = [
    # T, d, h, E, k, dtype, routing
    (1000, 128, 256, 16, 6, "bf16", "skewed"),
    (130, 128, 128, 256, 16, "bf16", "skewed"),
    (200, 64, 96, 6, 3, "fp32", "skewed"),
    (257, 256, 128, 2, 2, "bf16", "balanced"),   # k = 2: red.add of two terms is already exact
    (256, 64, 128, 4, 2, "fp32", "balanced"),
    (333, 256, 256, 4, 1, "bf16", "balanced"),   # k = 1: flag ignored (direct store)
    (100, 64, 64, 4, 1, "fp32", "skewed"),
]
_DET_KEYS = ("y", "dx", "dA", "dB", "dg", "dw1", "dw2", "dw3", "dw_gate")


@pytest.mark.parametrize("T,d,h,E,k,dtype,routing", DET_CASES)
def test_deterministic_combine(M, T, d, h, E, k, dtype, routing):
    """deterministic=True (NEXT-4): fp32 row results are summed per token
    in slot order, so repeated runs are bitwise identical for every k; the
    result is within tolerance of the oracle, and for k <= 2 bit-identical to
    the fused red.add combine (a + b == b + a exactly)."""
    inp, o1 = _run_layer(M, T, d, h, E, k, dtype, False, routing, seed=7 * T + k, det=True)
    _, o2 = _run_layer(M, T, d, h, E, k, dtype, False, routing, seed=7 * T + k, det=True)
    _, o0 = _run_layer(M, T, d, h, E, k, dtype, False, routing, seed=7 * T + k, det=False)
    for n in _DET_KEYS:
        assert torch.equal(o1[n], o2[n]), n
        if k <= 2:
            assert torch.equal(o1[n], o0[n]), n
    X, WG, W1, W2, W3, DY = (f64(inp[n]) for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
    fwd = O.layer_forward(X, WG, W1, W2, W3, k, False, logits=f64(o1["logits"]))
    bwd = O.layer_backward(fwd, DY, X, WG, W1, W2, W3, False)
    tol = FP32_TOL if dtype == "fp32" else BF16_TOL
    errs = {n: normwise(o1[n], fwd[n] if n == "y" else bwd[n]) for n in _DET_KEYS}
    bad = {n: v for n, v in errs.items() if not v <= tol}
    assert not bad, errs
