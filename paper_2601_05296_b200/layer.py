"""Functional API and autograd layer over the C ABI.

Each function allocates its outputs with torch (device memory only) and calls
the library entry point of the same name; nothing is computed in Python.
Citations: P:n = line of the paper text.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib as L


def _problem(T, d, h, E, k, dtype, renormalize=False, check_routing=False, checkpoint="ab", activation="swiglu",
             deterministic=False):
    return L.problem(T, d, h, E, k, dtype, renormalize, check_routing, checkpoint, activation, deterministic)


@dataclass
class Dispatch:
    """The index structures of §4.1; int32 device tensors."""
    counts: torch.Tensor      # [E]      expert_lengths
    offs: torch.Tensor        # [E+1]    expert_token_offsets
    eti: torch.Tensor         # [T*k]    expert_token_indices
    tim: torch.Tensor         # [T, k]   token_index_map
    row_slot: torch.Tensor    # [T*k]    inverse of tim
    ids: torch.Tensor         # [T, k]   token_expert_indices

    token_rows = None         # optional device int32 [1]: token rows >= it carry no slot

    def c(self):
        return L.make_dispatch(self.counts, self.offs, self.eti, self.tim, self.row_slot, self.ids, self.token_rows)


def route(x, w_gate, k, renormalize=False, stream=None):
    """moe_route: logits [T,E] fp32, ids [T,k] int32, w [T,k] fp32."""
    T, d = x.shape
    E = w_gate.shape[0]
    p = _problem(T, d, 128, E, k, x.dtype, renormalize)  # h is not used by routing
    logits = torch.empty(T, E, dtype=torch.float32, device=x.device)
    ids = torch.empty(T, k, dtype=torch.int32, device=x.device)
    w = torch.empty(T, k, dtype=torch.float32, device=x.device)
    L.moe_route(p, x, w_gate, logits, ids, w, stream)
    return logits, ids, w


def dispatch_build(ids, E, check_routing=False, stream=None, dtype=torch.bfloat16):
    """moe_dispatch_build (§4.2)."""
    T, k = ids.shape
    dev = ids.device
    p = _problem(T, 128, 128, E, k, dtype, False, check_routing)
    R = T * k
    disp = Dispatch(torch.empty(E, dtype=torch.int32, device=dev), torch.empty(E + 1, dtype=torch.int32, device=dev),
                    torch.empty(max(R, 1), dtype=torch.int32, device=dev)[:R],
                    torch.empty(T, k, dtype=torch.int32, device=dev),
                    torch.empty(max(R, 1), dtype=torch.int32, device=dev)[:R], ids)
    ws = L.workspace(p, L.MOE_OP_DISPATCH, dev)
    L.moe_dispatch_build(p, ids, disp.c(), ws, stream)
    if check_routing:
        disp.status = ws[:4].view(torch.int32)
    return disp


def ffn_fwd(x, w1, w2, w3, topk_w, disp: Dispatch, renormalize=False, stream=None, checkpoint="ab",
            activation="swiglu", deterministic=False):
    """moe_ffn_fwd (§3.1, Alg. 1 FusedForward): returns y, A, B (A, B checkpointed;
    None, None under checkpoint="none", where backward recomputes them), and under
    checkpoint="abu" (Alg. 1 literally) a fourth element, the saved wU.
    activation "silu" | "relu": the non-gated expert W2 sigma(W1 x); w2
    may be None and B is None.  deterministic: ordered token-side combine
    (bitwise reproducible for every k; NEXT-4)."""
    T, d = x.shape
    E, h, _ = w1.shape
    k = topk_w.shape[1]
    p = _problem(T, d, h, E, k, x.dtype, renormalize, checkpoint=checkpoint, activation=activation,
                 deterministic=deterministic)
    R = T * k
    save = checkpoint in ("ab", "abu")
    gated = activation == "swiglu"
    a = torch.empty(R, h, dtype=x.dtype, device=x.device) if save else None
    b = torch.empty(R, h, dtype=x.dtype, device=x.device) if (save and gated) else None
    u = torch.empty(R, h, dtype=x.dtype, device=x.device) if checkpoint == "abu" else None
    y = torch.empty(T, d, dtype=x.dtype, device=x.device)
    ws = L.workspace(p, L.MOE_OP_FFN_FWD, x.device)
    L.moe_ffn_fwd(p, x, w1, w2, w3, topk_w, disp.c(), a, b, u, y, ws, stream)
    return (y, a, b, u) if checkpoint == "abu" else (y, a, b)


def ffn_bwd(dy, x, w1, w2, w3, topk_w, disp: Dispatch, a_save, b_save, w_gate=None, logits=None,
            renormalize=False, stream=None, checkpoint="ab", activation="swiglu", deterministic=False, u_save=None,
            staged=False, release_ab=False):
    """moe_ffn_bwd (§3.2, Alg. 1 FusedBackward).  a_save/b_save are overwritten
    with dA/dB (checkpoint="none": pass None, A and B are recomputed into
    scratch buffers); u_save = the saved wU under checkpoint="abu".  With
    w_gate/logits: router backward too (dx includes it).

    staged=True issues the three MOE_BWD_* stages as separate calls on the same
    workspace and allocates each weight gradient only when its GEMM runs:
    data grads -> dW1/dW2 (the last reader of A/B: with release_ab their
    storage is released here) -> dW3 (reads wU).  Same results, lower peak."""
    T, d = x.shape
    E, h, _ = w1.shape
    k = topk_w.shape[1]
    p = _problem(T, d, h, E, k, x.dtype, renormalize, checkpoint=checkpoint, activation=activation,
                 deterministic=deterministic)
    gated = activation == "swiglu"
    R = T * k
    if checkpoint == "none":  # scratch for the recomputed A, B (then dA, dB)
        a_save = torch.empty(R, h, dtype=x.dtype, device=x.device)
        b_save = torch.empty(R, h, dtype=x.dtype, device=x.device) if gated else None
        release_ab = True
    dx = torch.empty_like(x)
    dg = torch.empty(T, k, dtype=torch.float32, device=x.device)
    router = None
    dwg = None
    if w_gate is not None:
        dwg = torch.empty_like(w_gate)
        router = L.MoeRouterBwd(w_gate.data_ptr(), logits.data_ptr(), disp.ids.data_ptr(), dwg.data_ptr())
    ws = L.workspace(p, L.MOE_OP_FFN_BWD, x.device)
    args = (p, dy, x, w1, w2, w3, topk_w, disp.c(), a_save, b_save, u_save)
    if not staged:
        dw1 = torch.empty_like(w1)
        dw2 = torch.empty_like(w2) if gated else None
        dw3 = torch.empty_like(w3)
        L.moe_ffn_bwd(*args, dx, dw1, dw2, dw3, dg, router, ws, stream)
    else:
        L.moe_ffn_bwd(*args, dx, None, None, None, dg, router, ws, stream, stages=L.MOE_BWD_DATA)
        dw1 = torch.empty_like(w1)
        dw2 = torch.empty_like(w2) if gated else None
        L.moe_ffn_bwd(*args, dx, dw1, dw2, None, dg, None, ws, stream, stages=L.MOE_BWD_DW12)
        if release_ab:  # dA/dB are dead: give their memory back (stream-ordered reuse)
            for t in (a_save, b_save):
                if t is not None:
                    t.untyped_storage().resize_(0)
        dw3 = torch.empty_like(w3)
        L.moe_ffn_bwd(*args, dx, None, None, dw3, dg, None, ws, stream, stages=L.MOE_BWD_DW3)
    return dict(dx=dx, dw1=dw1, dw2=dw2, dw3=dw3, dg=dg, dw_gate=dwg)


class MoEBlazeFunction(torch.autograd.Function):
    """y = MoE(x): route -> dispatch -> fused expert forward; backward recomputes
    SiLU from the checkpointed A, B.  Saved for backward: x, logits,
    ids, w, the index structures, A, B (+ wU under checkpoint="abu") -- no
    routed-token buffer.  With checkpoint="none" A, B are not saved either
    (recomputed in backward).  Backward runs staged (ffn_bwd(staged=True)) and
    releases A/B as soon as dW1/dW2 are done, so it can run only once per
    forward: the saved A, B are overwritten in place by dA, dB."""

    @staticmethod
    def forward(ctx, x, w_gate, w1, w2, w3, k, renormalize, checkpoint="ab", activation="swiglu",
                deterministic=False):
        logits, ids, w = route(x, w_gate, k, renormalize)
        disp = dispatch_build(ids, w_gate.shape[0], dtype=x.dtype)
        out = ffn_fwd(x, w1, w2, w3, w, disp, renormalize, checkpoint=checkpoint, activation=activation,
                      deterministic=deterministic)
        y, a, b = out[:3]
        gated = activation == "swiglu"
        saved = [x, w_gate, w1, w2 if gated else w1, w3, logits, ids, w, disp.counts, disp.offs, disp.eti, disp.tim,
                 disp.row_slot]
        if checkpoint in ("ab", "abu"):
            saved += [a, b if gated else a]
        if checkpoint == "abu":
            saved += [out[3]]
        ctx.save_for_backward(*saved)
        ctx.renormalize = renormalize
        ctx.checkpoint = checkpoint
        ctx.activation = activation
        ctx.deterministic = deterministic
        ctx.consumed = False
        return y

    @staticmethod
    def backward(ctx, dy):
        if ctx.consumed:
            raise RuntimeError("MoEBlazeFunction: backward ran twice on one forward; the checkpointed A, B were "
                               "overwritten in place by dA, dB (and released) by the first backward")
        ctx.consumed = True
        t = ctx.saved_tensors
        (x, w_gate, w1, w2, w3, logits, ids, w, counts, offs, eti, tim, row_slot) = t[:13]
        gated = ctx.activation == "swiglu"
        a, b = (t[13], t[14] if gated else None) if ctx.checkpoint in ("ab", "abu") else (None, None)
        u = t[15] if ctx.checkpoint == "abu" else None
        disp = Dispatch(counts, offs, eti, tim, row_slot, ids)
        g = ffn_bwd(dy.contiguous(), x, w1, w2 if gated else None, w3, w, disp, a, b, w_gate=w_gate, logits=logits,
                    renormalize=ctx.renormalize, checkpoint=ctx.checkpoint, activation=ctx.activation,
                    deterministic=ctx.deterministic, u_save=u, staged=True, release_ab=True)
        return g["dx"], g["dw_gate"], g["dw1"], g["dw2"], g["dw3"], None, None, None, None, None


def moe_layer(x, w_gate, w1, w2, w3, k, renormalize=False, checkpoint="ab", activation="swiglu",
              deterministic=False):
    """checkpoint: "ab" (paper: save A (,B), recompute the activation) | "none" (recompute A, B)
    | "abu" (Alg. 1 literally: save A, B and wU; no recompute of U for dW3).
    activation: "swiglu" | "silu" | "relu" (non-gated W2 sigma(W1 x); w2 unused).
    deterministic: ordered combine of a token's k expert outputs (bitwise reproducible for k >= 3)."""
    return MoEBlazeFunction.apply(x, w_gate, w1, w2, w3, k, renormalize, checkpoint, activation, deterministic)


class MoEBlazeLayer(torch.nn.Module):
    """Dropless top-k MoE layer on the MoEBlaze path: SwiGLU
    experts or non-gated SiLU/ReLU experts (no w2)."""

    def __init__(self, d, h, E, k, renormalize=False, dtype=torch.bfloat16, device="cuda", checkpoint="ab",
                 activation="swiglu", deterministic=False):
        super().__init__()
        self.k, self.renormalize, self.checkpoint = k, renormalize, checkpoint
        self.activation, self.deterministic = activation, deterministic
        kw = dict(dtype=dtype, device=device)
        self.w_gate = torch.nn.Parameter(torch.randn(E, d, **kw) / d ** 0.5)
        self.w1 = torch.nn.Parameter(torch.randn(E, h, d, **kw) / d ** 0.5)
        self.w2 = torch.nn.Parameter(torch.randn(E, h, d, **kw) / d ** 0.5) if activation == "swiglu" else None
        self.w3 = torch.nn.Parameter(torch.randn(E, d, h, **kw) / h ** 0.5)

    def forward(self, x):
        return moe_layer(x, self.w_gate, self.w1, self.w2, self.w3, self.k, self.renormalize, self.checkpoint,
                         self.activation, self.deterministic)
