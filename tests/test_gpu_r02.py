"""GPU tests of the round-2 additions, through the C ABI, against the fp64
oracle and against the existing paths:

* MOE_CKPT_ABU (Alg. 1 literally, "Store A, B, Y_swi"; P:240 dW3 from
  the saved Y_swi): parity with the oracle, saved set = AB + T*k*h elements;
* the staged backward (MOE_BWD_DATA / DW12 / DW3 as separate calls on one
  workspace, weight gradients allocated per stage, A/B released after DW12):
  bit-identical to the single call for every checkpoint policy;
* the activation-memory audits of SURVEY §8(c): the exact saved set and no
  allocation of the routed-token class (T*k x d) anywhere in fwd+bwd;
* a second backward through one forward raises (A, B were overwritten in place);
* per-row error gates next to the normwise one (localised bugs)."""
import numpy as np
import pytest
import torch

import oracle as O
from moe_inputs import make_inputs
from tests._util import BF16_TOL, FP32_TOL, ROW_TOL_BF16, ROW_TOL_FP32, elementwise, f64, i64, normwise, rowwise

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def M():
    from paper_2601_05296_b200 import build as B
    B.build()
    import paper_2601_05296_b200 as M
    M._lib.load()
    return M


ABU_CASES = [
    # T, d, h, E, k, dtype, act, renorm
    (512, 256, 384, 8, 2, "bf16", "swiglu", False),
    (1000, 128, 256, 16, 6, "bf16", "swiglu", True),
    (300, 3072, 384, 4, 2, "bf16", "swiglu", False),   # long-K dH variant
    (256, 64, 128, 4, 2, "fp32", "swiglu", False),
    (512, 256, 384, 8, 2, "bf16", "silu", False),
    (333, 256, 256, 4, 1, "bf16", "swiglu", False),    # k = 1 direct store
]


@pytest.mark.parametrize("T,d,h,E,k,dtype,act,renorm", ABU_CASES)
def test_abu_parity(M, T, d, h, E, k, dtype, act, renorm):
    inp = make_inputs(T, d, h, E, k, dtype=dtype, seed=T + k, device=DEV)
    gated = act == "swiglu"
    x, wg, w1, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w3", "dy"))
    w2 = inp["w2"] if gated else None
    logits, ids, w = M.route(x, wg, k, renorm)
    disp = M.dispatch_build(ids, E, dtype=x.dtype)
    y, a, b, u = M.ffn_fwd(x, w1, w2, w3, w, disp, renorm, checkpoint="abu", activation=act)
    a0, u0 = a.clone(), u.clone()
    g = M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits, renormalize=renorm,
                  checkpoint="abu", activation=act, u_save=u)
    torch.cuda.synchronize()
    assert torch.equal(u, u0), "the dH GEMM must not write the saved wU under MOE_CKPT_ABU"
    X, WG, W1, W3, DY = (f64(inp[n]) for n in ("x", "w_gate", "w1", "w3", "dy"))
    W2 = f64(inp["w2"]) if gated else None
    fwd = O.layer_forward(X, WG, W1, W2, W3, k, renorm, logits=f64(logits), activation=act)
    bwd = O.layer_backward(fwd, DY, X, WG, W1, W2, W3, renorm)
    # the saved wU against the oracle's w_r * U_r in expert-sorted row order
    rs = i64(disp.row_slot)
    wU = fwd["U"] * np.asarray(fwd["w"]).reshape(-1)[rs][:, None]
    tol = FP32_TOL if dtype == "fp32" else BF16_TOL
    errs = {"y": normwise(y, fwd["y"]), "A": normwise(a0, fwd["A"]), "wU": normwise(u0, wU),
            "dx": normwise(g["dx"], bwd["dx"]), "dw1": normwise(g["dw1"], bwd["dw1"]),
            "dw3": normwise(g["dw3"], bwd["dw3"]), "dg": normwise(g["dg"], bwd["dg"]),
            "dw_gate": normwise(g["dw_gate"], bwd["dw_gate"]), "dA": normwise(a, bwd["dA"])}
    if gated:
        errs["dw2"] = normwise(g["dw2"], bwd["dw2"])
        errs["dB"] = normwise(b, bwd["dB"])
    bad = {n: v for n, v in errs.items() if not v <= tol}
    assert not bad, errs


@pytest.mark.parametrize("ckpt", ["ab", "abu", "none"])
@pytest.mark.parametrize("dtype,act,det", [("bf16", "swiglu", False), ("fp32", "swiglu", False),
                                           ("bf16", "silu", False), ("bf16", "swiglu", True)])
def test_staged_backward_bit_identical(M, ckpt, dtype, act, det):
    """moe_ffn_bwd issued as three stage calls on one workspace == one call (also
    for non-gated experts and the ordered combine)."""
    # k <= 2: the fused red.add combine is then order-independent, so two runs are bitwise
    # equal; the ordered combine (det) is bitwise reproducible at any k
    T, d, h, E, k = (700, 256, 640, 8, 6 if det else 2) if dtype == "bf16" else (200, 64, 96, 6, 2)
    gated = act == "swiglu"
    inp = make_inputs(T, d, h, E, k, dtype=dtype, seed=21, device=DEV)
    x, wg, w1, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w3", "dy"))
    w2 = inp["w2"] if gated else None
    logits, ids, w = M.route(x, wg, k)
    disp = M.dispatch_build(ids, E, dtype=x.dtype)
    out = M.ffn_fwd(x, w1, w2, w3, w, disp, checkpoint=ckpt, activation=act, deterministic=det)
    a, b = out[1], out[2]
    u = out[3] if ckpt == "abu" else None
    res = []
    for staged in (False, True):
        aa = a.clone() if a is not None else None
        bb = b.clone() if b is not None else None
        res.append(M.ffn_bwd(dy, x, w1, w2, w3, w, disp, aa, bb, w_gate=wg, logits=logits, checkpoint=ckpt,
                             activation=act, deterministic=det, u_save=u, staged=staged))
    torch.cuda.synchronize()
    for n in ("dx", "dw1", "dw2", "dw3", "dg", "dw_gate"):
        if res[0][n] is None:
            assert res[1][n] is None
            continue
        assert torch.equal(res[0][n], res[1][n]), n


def test_policies_autograd_bit_identical(M):
    """ab / none / abu through the autograd layer: y identical for ab and none;
    every gradient of the three policies within bf16 noise of each other and
    ab == none bit for bit."""
    inp = make_inputs(512, 256, 384, 8, 2, dtype="bf16", seed=4, device=DEV)
    outs = {}
    for ck in ("ab", "none", "abu"):
        x = inp["x"].clone().requires_grad_(True)
        ps = [inp[n].clone().requires_grad_(True) for n in ("w_gate", "w1", "w2", "w3")]
        y = M.moe_layer(x, *ps, 2, False, ck)
        y.backward(inp["dy"])
        outs[ck] = [y, x.grad] + [p.grad for p in ps]
    torch.cuda.synchronize()
    for a_, b_ in zip(outs["ab"], outs["none"]):
        assert torch.equal(a_, b_)
    for a_, b_ in zip(outs["ab"], outs["abu"]):
        assert normwise(b_, f64(a_)) < 1e-2


def test_second_backward_raises(M):
    inp = make_inputs(128, 128, 128, 4, 2, dtype="bf16", seed=1, device=DEV)
    x = inp["x"].clone().requires_grad_(True)
    ps = [inp[n].clone().requires_grad_(True) for n in ("w_gate", "w1", "w2", "w3")]
    y = M.moe_layer(x, *ps, 2)
    y.backward(inp["dy"], retain_graph=True)
    with pytest.raises(RuntimeError, match="backward ran twice"):
        y.backward(inp["dy"])


def test_saved_set_is_exact(M):
    """SURVEY §8(c) audit 3: the autograd saved set (unique storages, parameters
    excluded) is exactly {X, logits, ids, w, counts, offs, eti, tim, row_slot,
    A, B} (+ wU under abu) -- no routed-token copy of X, no U, no S."""
    T, d, h, E, k = 384, 256, 384, 8, 2
    R = T * k
    inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=2, device=DEV)
    for ck, extra in (("ab", [R * h * 2, R * h * 2]), ("abu", [R * h * 2] * 3), ("none", [])):
        x = inp["x"].clone().requires_grad_(True)
        ps = [inp[n].clone().requires_grad_(True) for n in ("w_gate", "w1", "w2", "w3")]
        pids = {p.untyped_storage().data_ptr() for p in ps}
        seen = {}

        def pack(t):
            s = t.untyped_storage()
            if s.data_ptr() not in pids:
                seen[s.data_ptr()] = s.nbytes()
            return t

        with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
            y = M.moe_layer(x, *ps, k, False, ck)
        y.backward(inp["dy"])
        torch.cuda.synchronize()
        # X, logits [T,E] f32, ids [T,k] i32, w [T,k] f32, counts [E], offs [E+1], eti [R], tim [T,k], row_slot [R]
        expect = sorted([T * d * 2, T * E * 4, R * 4, R * 4, E * 4, (E + 1) * 4, R * 4, R * 4, R * 4] + extra)
        assert sorted(seen.values()) == expect, (ck, sorted(seen.values()), expect)


def test_no_routed_token_allocation(M):
    """SURVEY §8(c) audit 2 (runtime): the CUDA caching allocator's trace over a
    full fwd+bwd contains no allocation of the routed-token class R x d (bf16 or
    fp32), i.e. no permuted or padded copy of X, dY, or of the expert outputs."""
    T, d, h, E, k = 1024, 384, 640, 8, 4
    R = T * k
    inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=6, device=DEV)
    x = inp["x"].clone().requires_grad_(True)
    ps = [inp[n].clone().requires_grad_(True) for n in ("w_gate", "w1", "w2", "w3")]
    torch.cuda.synchronize()
    torch.cuda.memory._record_memory_history(max_entries=100000)
    try:
        y = M.moe_layer(x, *ps, k)
        y.backward(inp["dy"])
        torch.cuda.synchronize()
        snap = torch.cuda.memory._snapshot()
    finally:
        torch.cuda.memory._record_memory_history(enabled=None)
    sizes = [e["size"] for tr in snap["device_traces"] for e in tr if e["action"] == "alloc"]
    assert sizes, "no allocation recorded"
    # the caching allocator rounds requests up to 512 B blocks: compare by class
    routed = {R * d * 2, R * d * 4}
    assert not [s for s in sizes if any(abs(s - r) < 4096 for r in routed)], sorted(set(sizes))
    # nothing larger than the named buffers: weights' grads (E*h*d), A/B/U (R*h), the workspaces
    L = M._lib
    cap = max(E * h * d * 2, R * h * 2,
              L.workspace_size(L.problem(T, d, h, E, k, torch.bfloat16), L.MOE_OP_FFN_FWD),
              L.workspace_size(L.problem(T, d, h, E, k, torch.bfloat16), L.MOE_OP_FFN_BWD))
    assert max(sizes) <= cap + 4096


ROW_CASES = [
    ("small_bf16", 512, 256, 384, 8, 2, "bf16"),
    ("ragged_bf16", 1000, 128, 256, 16, 6, "bf16"),
    ("long_k_bf16", 300, 3072, 384, 4, 2, "bf16"),
    ("tiny_fp32", 256, 64, 128, 4, 2, "fp32"),
]


@pytest.mark.parametrize("case", ROW_CASES, ids=[c[0] for c in ROW_CASES])
def test_rowwise_error_gates(M, case):
    """Per-row max-relative error (each token / routed row / weight row against
    its own max, floored at 1e-3 of the tensor max) next to the normwise gate:
    a dropped K block or a wrong gather index in one segment moves a row by
    O(10 %), far above bf16 noise (<= 2e-2 per row)."""
    from tests.test_gpu_parity import _run_layer
    name, T, d, h, E, k, dtype = case
    inp, out = _run_layer(M, T, d, h, E, k, dtype, False, "skewed", seed=9)
    X, WG, W1, W2, W3, DY = (f64(inp[n]) for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
    fwd = O.layer_forward(X, WG, W1, W2, W3, k, False, logits=f64(out["logits"]))
    bwd = O.layer_backward(fwd, DY, X, WG, W1, W2, W3, False)
    rtol = ROW_TOL_FP32 if dtype == "fp32" else ROW_TOL_BF16
    errs, elem = {}, {}
    for n in ("A", "B", "y", "dA", "dB", "dx", "dw1", "dw2", "dw3"):
        ref = fwd[n] if n in ("A", "B", "y") else bwd[n]
        got = out[n]
        if n.startswith("dw"):  # rows of every expert's matrix
            got, ref = got.reshape(-1, got.shape[-1]), ref.reshape(-1, ref.shape[-1])
        errs[n] = rowwise(got, ref)
        elem[n] = elementwise(got, ref, 1e-3)
    bad = {n: v for n, v in errs.items() if not v <= rtol}
    print(name, "rowwise", {n: round(v, 5) for n, v in errs.items()},
          "elementwise(floor 1e-3)", {n: round(v, 4) for n, v in elem.items()})
    assert not bad, (name, errs)


def test_kernel_copy_into_pinned_host_memory(M):
    """moe_gather_rows with index = NULL copies rows with a kernel, also into pinned
    host memory (UVA): the EP split-size read (ep.CudaOps.read_host) uses it so the
    read never queues behind the host pipeline's bulk copy-engine transfers."""
    from paper_2601_05296_b200.ep import CudaOps
    src = torch.arange(3000, dtype=torch.int32, device=DEV) * 7 - 11
    pinned = torch.zeros(3000, dtype=torch.int32, pin_memory=True)
    M._lib.moe_gather_rows(src.view(-1, 1), None, pinned.view(-1, 1))
    torch.cuda.synchronize()
    assert torch.equal(pinned, src.cpu())
    assert torch.equal(CudaOps().read_host(src[:17]), src[:17].cpu())
    # device rows, identity copy of the first n rows (bf16, 16-byte rows path)
    a = torch.randn(64, 256, device=DEV).to(torch.bfloat16)
    b = torch.empty(40, 256, dtype=torch.bfloat16, device=DEV)
    M._lib.moe_gather_rows(a, None, b)
    torch.cuda.synchronize()
    assert torch.equal(b, a[:40])


def test_cuda_graph_capture_and_replay(M):
    """The whole fwd+bwd (route, dispatch, both FFN calls, router backward) captures
    into one CUDA graph and replays with fresh inputs, bit-identical to eager: no
    host sync inside any call, all scratch (incl. the tile-scheduler counters,
    ADVICE r01) in stream-ordered workspaces."""
    T, d, h, E, k = 640, 256, 384, 8, 2
    inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=31, device=DEV)
    wg, w1, w2, w3 = (inp[n] for n in ("w_gate", "w1", "w2", "w3"))
    x = inp["x"].clone()
    dy = inp["dy"].clone()

    def step():
        logits, ids, w = M.route(x, wg, k)
        disp = M.dispatch_build(ids, E, dtype=x.dtype)
        y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp)
        g = M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits)
        return [y, ids, g["dx"], g["dw1"], g["dw2"], g["dw3"], g["dw_gate"]]

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        static_out = step()
    for seed in (32, 33):
        new = make_inputs(T, d, h, E, k, dtype="bf16", seed=seed, device=DEV)
        x.copy_(new["x"])
        dy.copy_(new["dy"])
        graph.replay()
        torch.cuda.synchronize()
        ref = step()
        torch.cuda.synchronize()
        for a_, b_ in zip(static_out, ref):
            assert torch.equal(a_, b_)
