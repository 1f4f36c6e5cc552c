"""Expert-parallel MoEBlaze layer over torch.distributed.

The paper is single-GPU and names distribution as future work.  The
layer shards naturally by expert: rank r owns experts [r*E/P, (r+1)*E/P);
tokens stay data-parallel (T per rank); the router W_g is replicated.

Forward, per rank:
  1. route + dispatch build over the GLOBAL experts (moe_route,
     moe_dispatch_build): expert_token_indices is then grouped by owner rank.
  2. split sizes per destination from expert_token_offsets (one D2H) and the
     per-expert counts all-to-all (C1) -> receive sizes.
  3. send buffer = X rows in expert_token_indices order (moe_gather_rows) +
     each row's gate weight and local expert id (moe_ep_row_meta): exactly the
     routed rows, no padding, freed after the exchange (C2, NCCL all-to-all).
  4. the receiver runs the SAME kernels on its received rows as a k = 1
     problem (moe_dispatch_build over local expert ids, moe_ffn_fwd): each
     received row's output w*O comes back (C3) in the sender's order, and
     moe_combine_rows sums the k returned rows per token through
     token_index_map.
Backward mirrors it: dY rows and X rows travel again (C4; keeping the received
X would be a saved permuted activation), moe_ffn_bwd on the receiver, dX rows
and gate-grads return (C5), moe_combine_rows + moe_router_backward on the
source, and all_reduce of dW_g (C6).  Expert weight grads stay local.

`ops` (the compute) and `a2a` (the exchange) are injectable so the host-side
bookkeeping is testable with gloo on CPU; the product binds CudaOps (the C
ABI) and NCCL.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib as L
from .layer import Dispatch, dispatch_build, ffn_bwd, ffn_fwd, route


class CudaOps:
    """The EP step's compute, every piece a C-ABI call into libmoeblaze.so."""

    def route(self, x, wg, k, renorm):
        return route(x, wg, k, renorm)

    def dispatch(self, ids, E, dtype):
        return dispatch_build(ids, E, dtype=dtype)

    def row_meta(self, disp, w, experts_per_rank, dtype):
        T, k = w.shape
        R = T * k
        p = L.problem(T, 128, 128, max(experts_per_rank, k), k, dtype)
        row_w = torch.empty(R, dtype=torch.float32, device=w.device)
        row_e = torch.empty(R, dtype=torch.int32, device=w.device)
        L.moe_ep_row_meta(p, disp.c(), w, experts_per_rank, row_w, row_e)
        return row_w, row_e

    def gather_rows(self, src, index):
        n = index.numel()
        dst = torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
        L.moe_gather_rows(src, index.reshape(-1), dst)
        return dst

    def ffn_fwd(self, x, w1, w2, w3, w, disp):
        return ffn_fwd(x, w1, w2, w3, w, disp)

    def ffn_bwd(self, dy, x, w1, w2, w3, w, disp, a, b):
        return ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b)

    def combine(self, rows, tim, T, d, k):
        out = torch.empty(T, d, dtype=rows.dtype, device=rows.device)
        p = L.problem(T, d, 128, max(k, 1), k, rows.dtype)
        L.moe_combine_rows(p, rows, tim, out)
        return out

    def router_backward(self, dg, x, wg, logits, ids, dx_partial, renorm):
        T, d = x.shape
        E = wg.shape[0]
        k = dg.shape[1]
        p = L.problem(T, d, 128, E, k, x.dtype, renorm)
        dwg = torch.empty_like(wg)
        dx = torch.empty_like(dx_partial)
        router = L.MoeRouterBwd(wg.data_ptr(), logits.data_ptr(), ids.data_ptr(), dwg.data_ptr())
        ws = L.workspace(p, L.MOE_OP_ROUTER_BWD, x.device)
        L.moe_router_backward(p, dg, x, router, dx_partial, dx, ws)
        return dx, dwg


def nccl_a2a(send, send_split, recv_split, group=None):
    out = torch.empty((sum(recv_split),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(out, send.contiguous(), recv_split, send_split, group=group)
    return out


class ExpertParallelMoE:
    """One MoE layer, expert-parallel over `group`."""

    def __init__(self, E, k, renormalize=False, group=None, ops=None, a2a=None):
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if E % self.P:
            raise ValueError(f"E={E} not divisible by world size {self.P}")
        self.E, self.k, self.renorm, self.group = E, k, renormalize, group
        self.El = E // self.P
        self.local_experts = (self.rank * self.El, (self.rank + 1) * self.El)
        self.ops = ops or CudaOps()
        self._a2a = a2a or nccl_a2a
        self.last_rows_received = 0

    def a2a(self, send, send_split, recv_split):
        return self._a2a(send, send_split, recv_split, self.group)

    def forward(self, x, wg, w1l, w2l, w3l):
        ops, P, El, k = self.ops, self.P, self.El, self.k
        T, d = x.shape
        logits, ids, w = ops.route(x, wg, k, self.renorm)
        disp = ops.dispatch(ids, self.E, x.dtype)
        row_w, row_e = ops.row_meta(disp, w, El, x.dtype)
        # C1: per-expert counts to the owner ranks; split sizes to the host (one sync)
        recv_counts = self.a2a(disp.counts, [El] * P, [El] * P)
        offs_h = disp.offs.cpu().tolist()
        send_split = [offs_h[(q + 1) * El] - offs_h[q * El] for q in range(P)]
        rc = recv_counts.cpu().view(P, El)
        recv_split = rc.sum(1).tolist()
        self.last_rows_received = int(sum(recv_split))
        # C2: routed rows (exactly T*k rows in expert order; a comm buffer, not an activation)
        xs = ops.gather_rows(x, disp.eti)
        x_recv = self.a2a(xs, send_split, recv_split)
        del xs
        w_recv = self.a2a(row_w, send_split, recv_split).view(-1, 1)
        e_recv = self.a2a(row_e, send_split, recv_split).view(-1, 1)
        disp_l = ops.dispatch(e_recv, El, x.dtype)
        y_rows, a_l, b_l = ops.ffn_fwd(x_recv, w1l, w2l, w3l, w_recv, disp_l)
        del x_recv
        # C3: expert outputs back to their tokens, combined through token_index_map
        y_back = self.a2a(y_rows, recv_split, send_split)
        y = ops.combine(y_back, disp.tim, T, d, k)
        ctx = dict(x=x, wg=wg, w1l=w1l, w2l=w2l, w3l=w3l, logits=logits, ids=ids, w=w, disp=disp,
                   send_split=send_split, recv_split=recv_split, w_recv=w_recv, disp_l=disp_l, a_l=a_l, b_l=b_l)
        return y, ctx

    def backward(self, ctx, dy):
        ops = self.ops
        x, disp = ctx["x"], ctx["disp"]
        T, d = x.shape
        ss, rs = ctx["send_split"], ctx["recv_split"]
        # C4: dY rows and (again) X rows to the expert owners
        dy_recv = self.a2a(ops.gather_rows(dy, disp.eti), ss, rs)
        x_recv = self.a2a(ops.gather_rows(x, disp.eti), ss, rs)
        g = ops.ffn_bwd(dy_recv, x_recv, ctx["w1l"], ctx["w2l"], ctx["w3l"], ctx["w_recv"], ctx["disp_l"],
                        ctx["a_l"], ctx["b_l"])
        del dy_recv, x_recv
        # C5: token-gradient rows and gate-weight gradients back to the sources
        dx_back = self.a2a(g["dx"], rs, ss)
        dg_back = self.a2a(g["dg"].reshape(-1, 1), rs, ss)
        dx_part = ops.combine(dx_back, disp.tim, T, d, self.k)
        dg = ops.gather_rows(dg_back, disp.tim.reshape(-1)).view(T, self.k)
        dx, dwg = ops.router_backward(dg, x, ctx["wg"], ctx["logits"], ctx["ids"], dx_part, self.renorm)
        # C6: replicated router
        acc = dwg.float() if dwg.element_size() < 4 else dwg  # reduce 16-bit grads in fp32
        dist.all_reduce(acc, group=self.group)
        dwg = acc.to(dwg.dtype)
        return dict(dx=dx, dw_gate=dwg, dw1=g["dw1"], dw2=g["dw2"], dw3=g["dw3"], dg=dg)

    def step(self, x, wg, w1l, w2l, w3l, dy):
        y, ctx = self.forward(x, wg, w1l, w2l, w3l)
        return y, self.backward(ctx, dy)
