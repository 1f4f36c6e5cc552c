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

    def c(self):
        return L.make_dispatch(self.counts, self.offs, self.eti, self.tim, self.row_slot, self.ids)


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
    None, None under checkpoint="none", where backward recomputes them).
    activation "silu" | "relu": the non-gated expert W2 sigma(W1 x); w2
    may be None and B is None.  deterministic: ordered token-side combine
    (bitwise reproducible for every k; NEXT-4)."""
    T, d = x.shape
    E, h, _ = w1.shape
    k = topk_w.shape[1]
    p = _problem(T, d, h, E, k, x.dtype, renormalize, checkpoint=checkpoint, activation=activation,
                 deterministic=deterministic)
    R = T * k
    save = checkpoint == "ab"
    gated = activation == "swiglu"
    a = torch.empty(R, h, dtype=x.dtype, device=x.device) if save else None
    b = torch.empty(R, h, dtype=x.dtype, device=x.device) if (save and gated) else None
    y = torch.empty(T, d, dtype=x.dtype, device=x.device)
    ws = L.workspace(p, L.MOE_OP_FFN_FWD, x.device)
    L.moe_ffn_fwd(p, x, w1, w2, w3, topk_w, disp.c(), a, b, y, ws, stream)
    return y, a, b


def ffn_bwd(dy, x, w1, w2, w3, topk_w, disp: Dispatch, a_save, b_save, w_gate=None, logits=None,
            renormalize=False, stream=None, checkpoint="ab", activation="swiglu", deterministic=False):
    """moe_ffn_bwd (§3.2, Alg. 1 FusedBackward).  a_save/b_save are overwritten
    with dA/dB (checkpoint="none": pass None, A and B are recomputed).  With
    w_gate/logits: router backward too (dx includes it)."""
    T, d = x.shape
    E, h, _ = w1.shape
    k = topk_w.shape[1]
    p = _problem(T, d, h, E, k, x.dtype, renormalize, checkpoint=checkpoint, activation=activation,
                 deterministic=deterministic)
    dx = torch.empty_like(x)
    dw1 = torch.empty_like(w1)
    dw2 = torch.empty_like(w2) if activation == "swiglu" else None
    dw3 = torch.empty_like(w3)
    dg = torch.empty(T, k, dtype=torch.float32, device=x.device)
    router = None
    dwg = None
    if w_gate is not None:
        dwg = torch.empty_like(w_gate)
        router = L.MoeRouterBwd(w_gate.data_ptr(), logits.data_ptr(), disp.ids.data_ptr(), dwg.data_ptr())
    ws = L.workspace(p, L.MOE_OP_FFN_BWD, x.device)
    L.moe_ffn_bwd(p, dy, x, w1, w2, w3, topk_w, disp.c(), a_save, b_save, dx, dw1, dw2, dw3, dg, router, ws, stream)
    return dict(dx=dx, dw1=dw1, dw2=dw2, dw3=dw3, dg=dg, dw_gate=dwg)


class MoEBlazeFunction(torch.autograd.Function):
    """y = MoE(x): route -> dispatch -> fused expert forward; backward recomputes
    SiLU from the checkpointed A, B.  Saved for backward: x, logits,
    ids, w, the index structures, A, B — no routed-token buffer.  With
    checkpoint="none" A, B are not saved either (recomputed in backward)."""

    @staticmethod
    def forward(ctx, x, w_gate, w1, w2, w3, k, renormalize, checkpoint="ab", activation="swiglu",
                deterministic=False):
        logits, ids, w = route(x, w_gate, k, renormalize)
        disp = dispatch_build(ids, w_gate.shape[0], dtype=x.dtype)
        y, a, b = ffn_fwd(x, w1, w2, w3, w, disp, renormalize, checkpoint=checkpoint, activation=activation,
                          deterministic=deterministic)
        gated = activation == "swiglu"
        saved = [x, w_gate, w1, w2 if gated else w1, w3, logits, ids, w, disp.counts, disp.offs, disp.eti, disp.tim,
                 disp.row_slot]
        if checkpoint == "ab":
            saved += [a, b if gated else a]
        ctx.save_for_backward(*saved)
        ctx.renormalize = renormalize
        ctx.checkpoint = checkpoint
        ctx.activation = activation
        ctx.deterministic = deterministic
        return y

    @staticmethod
    def backward(ctx, dy):
        t = ctx.saved_tensors
        (x, w_gate, w1, w2, w3, logits, ids, w, counts, offs, eti, tim, row_slot) = t[:13]
        gated = ctx.activation == "swiglu"
        a, b = (t[13], t[14] if gated else None) if ctx.checkpoint == "ab" else (None, None)
        disp = Dispatch(counts, offs, eti, tim, row_slot, ids)
        g = ffn_bwd(dy.contiguous(), x, w1, w2 if gated else None, w3, w, disp, a, b, w_gate=w_gate, logits=logits,
                    renormalize=ctx.renormalize, checkpoint=ctx.checkpoint, activation=ctx.activation,
                    deterministic=ctx.deterministic)
        return g["dx"], g["dw_gate"], g["dw1"], g["dw2"], g["dw3"], None, None, None, None, None


def moe_layer(x, w_gate, w1, w2, w3, k, renormalize=False, checkpoint="ab", activation="swiglu",
              deterministic=False):
    """checkpoint: "ab" (paper: save A (,B), recompute the activation) | "none" (recompute A, B).
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
