"""Materialise-everything MoE layer in PyTorch eager (memory / speed comparator).

This is the conventional implementation the paper contrasts MoEBlaze with
(Fig. 1-left): an argsort dispatch, a routed-token buffer
X[eti] of shape [T*k, d], per-expert grouped GEMMs on that buffer, and
eager SwiGLU / combine whose intermediates autograd saves.  It is NOT the
product and never runs on the product path; bench.py uses it only to measure
saved-activation bytes (P:289's saved-tensor-hook method) next to ours.
"""
import torch
import torch.nn.functional as F


def materialized_moe(x, w_gate, w1, w2, w3, k, renormalize=False, activation="swiglu"):
    T, d = x.shape
    E = w_gate.shape[0]
    logits = x.float() @ w_gate.float().t()
    p = torch.softmax(logits, dim=1)
    topv, ids = torch.topk(logits, k, dim=1)
    w = torch.gather(p, 1, ids)
    if renormalize:
        w = w / w.sum(1, keepdim=True)
    flat = ids.reshape(-1)
    order = torch.argsort(flat, stable=True)
    eti = order // k
    counts = torch.bincount(flat, minlength=E)
    offs = torch.cumsum(counts, 0).to(torch.int32)
    xr = x[eti]                                            # routed-token buffer [T*k, d]
    a = F.grouped_mm(xr, w1.transpose(1, 2), offs=offs)    # [R, h]
    if activation == "swiglu":
        b = F.grouped_mm(xr, w2.transpose(1, 2), offs=offs)
        u = F.silu(a) * b
    else:                                                  # non-gated expert
        u = F.silu(a) if activation == "silu" else F.relu(a)
    o = F.grouped_mm(u, w3.transpose(1, 2), offs=offs)     # expert outputs [R, d] before combine
    wr = w.reshape(-1)[order].to(o.dtype)
    y = torch.zeros(T, d, dtype=o.dtype, device=x.device).index_add_(0, eti, o * wr[:, None])
    return y
