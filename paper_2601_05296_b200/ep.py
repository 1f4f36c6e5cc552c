"""Expert-parallel MoEBlaze layer over torch.distributed.

The paper is single-GPU and names distribution as future work.  The
layer shards naturally by expert: rank r owns experts [r*E/P, (r+1)*E/P);
tokens stay data-parallel (T per rank); the router W_g is replicated.

Per-destination dedup (NEXT-1).  A token whose k experts live on m <= min(k, P)
ranks travels to each of those ranks once, not k times: the send plan is the
MoEBlaze dispatch itself, applied one level up -- moe_ep_dest marks, per token,
the ranks owning any of its experts (dest [T, P], -1 elsewhere) and
moe_dispatch_build over dest (sparse slots) yields the send order (tokens
grouped by rank, ascending), the per-rank row counts and the inverse map
send_pos [T, P] (P:123-135 with "experts" = ranks).  Each sent row carries the
token's k slots restricted to the receiving rank (moe_ep_send_meta: local expert
id or -1, gate weight), so the receiver runs the SAME fused kernels as a
sparse-slot problem (p.rows = its routed (token, expert) rows): FWD_DOWN's
red.add combine then sums the token's local experts before anything travels
back -- one return row per (token, rank).

Local pairs never travel.  moe_ep_dest excludes the own rank, so a token's slots
on its own rank's experts are computed in place: the receiver's token rows are
[the T local tokens (moe_ep_local_slots: their own-rank slots) | the received
rows], its output rows [0, T) are the local partial outputs, which
moe_combine_rows adds as `base` to the returned rows.  At P = 1 nothing is
exchanged and the step is the single-GPU layer plus the plan bookkeeping.

Forward, per rank:
  1. moe_route + moe_dispatch_build over the global experts (per-expert counts).
  2. send plan (moe_ep_dest without self + moe_dispatch_build); C1: all-to-all of
     the [rows, pairs per local expert] counts; ONE device->host read of the
     split sizes (the only host sync of the step: buffers are sized by it).
  3. C2a: the packed slot metadata of the remote rows; the receiver builds its
     sparse dispatch over [local slots | received slots].  C2b: remote X rows in
     send order (moe_gather_rows), received behind the local tokens' rows, on a
     side stream: moe_ffn_fwd_ex runs the up-projection of every expert's local
     rows (they come first in each expert segment) while it is in flight and
     waits for it only before the received rows' up-projection.
  4. receiver: moe_ffn_fwd_ex (split at row T): the received rows' down projection
     and y first, then (C3 on a side stream) the local rows' down projection;
     C3 returns one row per (remote token, rank); moe_combine_rows adds them to
     the local partial through send_pos.
Backward:
  C4a: remote dY rows to the owners (needed first); C4b: remote X rows again
  (keeping the received X would be a saved permuted activation) on a side
  stream, overlapped with the dH / dX GEMMs -- moe_ffn_bwd waits for it only
  before the dW1/dW2 GEMM (moe_bwd_sync.x_ready).  C5: dX rows and gate-weight
  gradients return on the side stream as soon as moe_ffn_bwd records dx_ready,
  overlapped with the dW3 / dW1,dW2 GEMMs.  moe_combine_rows (local dX partial
  as base) + moe_ep_slot_grad (local dg) + moe_router_backward on the source;
  C6: all_reduce of dW_g.  Expert weight grads stay local.

`ops` (the compute) and `a2a` (the exchange) are injectable so the host-side
bookkeeping is testable with gloo on CPU; the product binds CudaOps (the C ABI)
and NCCL.
"""
from __future__ import annotations

import contextlib

import torch
import torch.distributed as dist

from . import _lib as L
from .layer import Dispatch, route


class CudaOps:
    """The EP step's compute, every piece a C-ABI call into libmoeblaze.so."""

    def route(self, x, wg, k, renorm):
        return route(x, wg, k, renorm)

    def dispatch(self, ids, E, dtype, rows=0):
        """moe_dispatch_build; rows > 0: sparse slots (-1 = empty), R <= rows."""
        T, k = ids.shape
        dev = ids.device
        R = rows if rows > 0 else T * k
        p = L.problem(T, 128, 128, E, k, dtype, rows=rows)
        disp = Dispatch(torch.empty(E, dtype=torch.int32, device=dev), torch.empty(E + 1, dtype=torch.int32, device=dev),
                        torch.empty(max(R, 1), dtype=torch.int32, device=dev)[:R],
                        torch.empty(T, k, dtype=torch.int32, device=dev),
                        torch.empty(max(R, 1), dtype=torch.int32, device=dev)[:R], ids)
        ws = L.workspace(p, L.MOE_OP_DISPATCH, dev)
        L.moe_dispatch_build(p, ids, disp.c(), ws)
        return disp

    def ep_dest(self, ids, E, El, P, self_rank=-1):
        T, k = ids.shape
        dest = torch.empty(T, P, dtype=torch.int32, device=ids.device)
        L.moe_ep_dest(L.problem(T, 128, 128, E, k, torch.bfloat16), ids, El, P, dest, self_rank=self_rank)
        return dest

    def local_slots(self, ids, w, E, El, rank, out_ids, out_w):
        """moe_ep_local_slots into out_ids / out_w ([T, k] views of the receiver's slot arrays)."""
        T, k = ids.shape
        L.moe_ep_local_slots(L.problem(T, 128, 128, E, k, torch.bfloat16), ids, w, El, rank, out_ids, out_w)

    def send_meta(self, ids, w, E, El, P, send_row_slot):
        T, k = ids.shape
        n = send_row_slot.numel()
        sid = torch.empty(n, k, dtype=torch.int32, device=ids.device)
        sw = torch.empty(n, k, dtype=torch.float32, device=ids.device)
        L.moe_ep_send_meta(L.problem(T, 128, 128, E, k, torch.bfloat16), ids, w, El, P, send_row_slot, sid, sw)
        return sid, sw

    def slot_grad(self, ids, E, El, P, send_pos, dg_back, dg_local=None, self_rank=-1):
        T, k = ids.shape
        dg = torch.empty(T, k, dtype=torch.float32, device=ids.device)
        L.moe_ep_slot_grad(L.problem(T, 128, 128, E, k, torch.bfloat16), ids, El, P, send_pos,
                           dg_back if dg_back is not None and dg_back.numel() else None, dg, dg_local=dg_local,
                           self_rank=self_rank)
        return dg

    def read_host(self, t):
        """The split sizes to the host: a kernel writes them into pinned host memory
        and the host waits on an event -- a plain .cpu() would queue its copy behind
        the copy engine's bulk transfers of a host-fed pipeline (tens of ms at
        the EP config), stalling the whole step."""
        if not t.is_cuda:
            return t.clone()
        if getattr(self, "_pinned", None) is None or self._pinned.numel() < t.numel():
            self._pinned = torch.empty(max(t.numel(), 1024), dtype=t.dtype, pin_memory=True)
        out = self._pinned[:t.numel()]
        L.moe_gather_rows(t.reshape(-1, 1), None, out.view(-1, 1))
        ev = torch.cuda.Event()
        ev.record()
        ev.synchronize()
        return out.clone()

    def gather_rows(self, src, index):
        n = index.numel()
        dst = torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
        L.moe_gather_rows(src, index.reshape(-1), dst)
        return dst

    def ffn_fwd(self, x, w1, w2, w3, w, disp, rows, t_ready=None, x_ready=None, y_ready=None, sm_reserve=0):
        """t_ready: x rows [0, t_ready) are resident, the rest arrive at x_ready (a CUDA
        event or None): moe_ffn_fwd_ex runs the up-projection of each expert's resident
        rows first and waits x_ready only before the rest (moe_dispatch_row_split); with
        y_ready it also finishes the y rows from t_ready on first, records y_ready, and
        runs the resident rows' down projection on all but sm_reserve SMs."""
        T, d = x.shape
        E, h, _ = w1.shape
        k = w.shape[1]
        p = L.problem(T, d, h, E, k, x.dtype, rows=rows)
        a = torch.empty(rows, h, dtype=x.dtype, device=x.device)
        b = torch.empty(rows, h, dtype=x.dtype, device=x.device)
        y = torch.empty(T, d, dtype=x.dtype, device=x.device)
        ws = L.workspace(p, L.MOE_OP_FFN_FWD, x.device)
        if t_ready is None and x_ready is None:
            L.moe_ffn_fwd(p, x, w1, w2, w3, w, disp.c(), a, b, None, y, ws)
        else:
            split = None
            if t_ready is not None:
                split = torch.empty(E, dtype=torch.int32, device=x.device)
                L.moe_dispatch_row_split(p, disp.c(), t_ready, split)
            L.moe_ffn_fwd_ex(p, x, w1, w2, w3, w, disp.c(), a, b, None, y, ws, row_split=split, x_ready=x_ready,
                             y_ready=y_ready, t_ready=t_ready or 0, sm_reserve=sm_reserve)
        return y, a, b

    def ffn_bwd(self, dy, x, w1, w2, w3, w, disp, a, b, rows, x_ready=None, dx_ready=None):
        T, d = dy.shape
        E, h, _ = w1.shape
        k = w.shape[1]
        p = L.problem(T, d, h, E, k, dy.dtype, rows=rows)
        dx = torch.empty_like(dy)
        dw1, dw2, dw3 = torch.empty_like(w1), torch.empty_like(w2), torch.empty_like(w3)
        dg = torch.empty(T, k, dtype=torch.float32, device=dy.device)
        ws = L.workspace(p, L.MOE_OP_FFN_BWD, dy.device)
        L.moe_ffn_bwd(p, dy, x, w1, w2, w3, w, disp.c(), a, b, None, dx, dw1, dw2, dw3, dg, None, ws,
                      x_ready=x_ready, dx_ready=dx_ready)
        return dict(dx=dx, dw1=dw1, dw2=dw2, dw3=dw3, dg=dg)

    def combine(self, rows, tim, T, d, k, base=None):
        """out[t] = base[t] + sum of the returned rows of t (moe_combine_rows)."""
        ref = base if base is not None else rows
        out = torch.empty(T, d, dtype=ref.dtype, device=ref.device)
        p = L.problem(T, d, 128, max(k, 1), k, ref.dtype, rows=T * k)  # sparse: -1 entries are expected
        L.moe_combine_rows(p, rows if rows.numel() else None, tim, out, base=base)
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


def nccl_a2a(send, send_split, recv_split, group=None, out=None):
    """all_to_all_single; `out` (optional) = a contiguous receive buffer, e.g. the
    tail of the receiver's row array behind its local tokens."""
    if out is None:
        out = torch.empty((sum(recv_split),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
    if dist.get_world_size(group) > 1:
        dist.all_to_all_single(out, send.contiguous(), recv_split, send_split, group=group)
    elif out.numel():
        out.copy_(send)  # one rank: the exchange is the identity
    return out


class ExpertParallelMoE:
    """One MoE layer, expert-parallel over `group`, with per-destination dedup.

    overlap: run C4b (X rows) and C5 (dX rows, gate grads) on a side CUDA
    stream against the backward GEMMs (default: on for CUDA tensors over NCCL).
    sm_reserve: SMs the local rows' down projection leaves to the C3 all-to-all's kernel
    (moe_fwd_sync.sm_reserve).
    retain_recv_x: keep the X rows received in forward for the dW1/dW2 GEMM
    instead of sending them again in backward: one a2a unit less
    per step, R_recv x d saved activation bytes more (a permuted copy of X, which
    the default -- the north star's no-permuted-buffer rule -- does not keep).
    """

    def __init__(self, E, k, renormalize=False, group=None, ops=None, a2a=None, overlap=None, retain_recv_x=False,
                 sm_reserve=16):
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if E % self.P:
            raise ValueError(f"E={E} not divisible by world size {self.P}")
        self.E, self.k, self.renorm, self.group = E, k, renormalize, group
        self.El = E // self.P
        self.local_experts = (self.rank * self.El, (self.rank + 1) * self.El)
        self.ops = ops or CudaOps()
        self._a2a = a2a or nccl_a2a
        self.overlap = overlap
        self.retain_recv_x = retain_recv_x
        self.sm_reserve = sm_reserve
        self.last_rows_received = 0   # (token, expert) rows computed here
        self.last_rows_sent = 0       # token rows sent (X) to other ranks, after dedup
        self.last_pairs_sent = 0      # (token, expert) pairs they carry

    def a2a(self, send, send_split, recv_split, out=None):
        """Collective: every rank calls it, also with nothing to send or receive."""
        return self._a2a(send, send_split, recv_split, self.group, out=out)

    def _side_stream(self, device):
        """One side stream per layer instance (the exchanges of C2b, C3, C4b and C5 are
        issued on it in program order; creating a stream per step would cost a driver call)."""
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=device)
        return self._side

    def _use_streams(self, x):
        if self.overlap is not None:
            return bool(self.overlap) and x.is_cuda
        return x.is_cuda and dist.get_backend(self.group) == "nccl"

    def _rows(self, local, send_tok, send_split, recv_split):
        """[T + U, ...] buffer: the local rows first, the U received rows behind them (C2 / C4)."""
        T = local.shape[0]
        buf = torch.empty((T + sum(recv_split),) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        buf[:T].copy_(local)
        self.a2a(self.ops.gather_rows(local, send_tok), send_split, recv_split, out=buf[T:])
        return buf

    def forward(self, x, wg, w1l, w2l, w3l):
        ops, P, El, k, E, me = self.ops, self.P, self.El, self.k, self.E, self.rank
        T, d = x.shape
        logits, ids, w = ops.route(x, wg, k, self.renorm)
        disp = ops.dispatch(ids, E, x.dtype)
        # send plan: one row per (token, owning remote rank); own-rank pairs stay here
        dest = ops.ep_dest(ids, E, El, P, self_rank=me)
        plan = ops.dispatch(dest, P, x.dtype, rows=T * min(k, P))
        # C1: [rows to q, pairs per local expert of q] -> owners; one host read of all split sizes
        cnt = torch.cat([plan.counts.view(P, 1), disp.counts.view(P, El)], 1).reshape(-1).contiguous()
        rc = self.a2a(cnt, [El + 1] * P, [El + 1] * P)
        host = ops.read_host(torch.cat([plan.counts, rc]))
        send_split = host[:P].tolist()
        rc_h = host[P:].view(P, El + 1)
        recv_split = rc_h[:, 0].tolist()
        n_pairs = int(rc_h[:, 1:].sum())  # incl. the own rank's pairs (row `me` of rc_h)
        n_send = int(sum(send_split))
        U = int(sum(recv_split))
        self.last_rows_received = n_pairs
        self.last_rows_sent = n_send
        self.last_pairs_sent = T * k
        send_tok = plan.eti[:n_send]
        # receiver slots: [local tokens' own-rank slots | received slots] (packed ids | w bits)
        wcols = k * w.element_size() // 4
        meta = torch.empty(T + U, k + wcols, dtype=torch.int32, device=x.device)
        lid = torch.empty(T, k, dtype=torch.int32, device=x.device)
        lw = torch.empty(T, k, dtype=w.dtype, device=x.device)
        ops.local_slots(ids, w, E, El, me, lid, lw)
        meta[:T, :k] = lid
        meta[:T, k:] = lw.view(torch.int32)
        sid, sw = ops.send_meta(ids, w, E, El, P, plan.row_slot[:n_send])
        # C2a: the received rows' slot metadata first (small: the receiver's dispatch needs it)
        self.a2a(torch.cat([sid, sw.view(torch.int32)], 1), send_split, recv_split, out=meta[T:])
        ids_l = meta[:, :k].contiguous()
        w_l = meta[:, k:].contiguous().view(w.dtype)
        disp_l = ops.dispatch(ids_l, El, x.dtype, rows=n_pairs) if n_pairs else None
        # C2b: the remote X rows, received behind the local rows.  With CUDA streams the
        # all-to-all runs on a side stream, issued BEFORE the expert GEMMs so NCCL's kernel
        # is resident first (the GEMMs' dynamic tile scheduler hands the remaining tiles to
        # the CTAs that start later); the up-projection of every expert's local rows
        # (tokens < T, first in each expert segment) overlaps it, and moe_ffn_fwd_ex waits
        # for the rows only before the received rows' up-projection
        streams = self._use_streams(x)
        x_l = torch.empty((T + U, d), dtype=x.dtype, device=x.device)
        x_l[:T].copy_(x)
        x_send = ops.gather_rows(x, send_tok)
        x_ready = None
        if streams and U:
            main, side = torch.cuda.current_stream(), self._side_stream(x.device)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self.a2a(x_send, send_split, recv_split, out=x_l[T:])
            x_ready = torch.cuda.Event()
            x_ready.record(side)
            x_l.record_stream(side)
            x_send.record_stream(side)
        else:
            self.a2a(x_send, send_split, recv_split, out=x_l[T:])
        del x_send
        y_ready = None
        if streams and U and n_pairs:
            y_ready = torch.cuda.Event()
            y_ready.record(torch.cuda.current_stream())  # created now; re-recorded by the library
        if n_pairs:
            y_rows, a_l, b_l = ops.ffn_fwd(x_l, w1l, w2l, w3l, w_l, disp_l, n_pairs,
                                           t_ready=T if U else None, x_ready=x_ready, y_ready=y_ready,
                                           sm_reserve=self.sm_reserve if y_ready is not None else 0)
        else:
            if x_ready is not None:
                torch.cuda.current_stream().wait_event(x_ready)
            y_rows, a_l, b_l = x_l.new_zeros(T + U, d), None, None
        x_keep = x_l if self.retain_recv_x else None
        del x_l
        # C3: per-(remote token, rank) partial outputs back; token-side sum through send_pos,
        # on top of the local partial (rows [0, T) of the receiver's output).  With streams the
        # received rows' y is final at y_ready, before the local rows' down projection, which
        # leaves sm_reserve SMs to this all-to-all's kernel
        if y_ready is not None:
            main, side = torch.cuda.current_stream(), self._side_stream(x.device)
            side.wait_event(y_ready)
            with torch.cuda.stream(side):
                y_back = self.a2a(y_rows[T:], recv_split, send_split)
            y_rows.record_stream(side)
            main.wait_stream(side)
            y_back.record_stream(main)
        else:
            y_back = self.a2a(y_rows[T:], recv_split, send_split)
        y = ops.combine(y_back, plan.tim, T, d, P, base=y_rows[:T])
        ctx = dict(x=x, wg=wg, w1l=w1l, w2l=w2l, w3l=w3l, logits=logits, ids=ids, w=w, plan=plan, send_tok=send_tok,
                   send_split=send_split, recv_split=recv_split, w_l=w_l, disp_l=disp_l, a_l=a_l, b_l=b_l,
                   n_pairs=n_pairs, x_recv=x_keep, U=U)
        return y, ctx

    def backward(self, ctx, dy):
        ops, P, El, E, k, me = self.ops, self.P, self.El, self.E, self.k, self.rank
        x, plan = ctx["x"], ctx["plan"]
        T, d = x.shape
        ss, rs = ctx["send_split"], ctx["recv_split"]
        n_pairs, U = ctx["n_pairs"], ctx["U"]
        w1l, w2l, w3l = ctx["w1l"], ctx["w2l"], ctx["w3l"]
        streams = self._use_streams(x)
        main = torch.cuda.current_stream() if streams else None
        side = self._side_stream(x.device) if streams else None
        sctx = (lambda: torch.cuda.stream(side)) if streams else contextlib.nullcontext
        # C4a: remote dY rows to the expert owners (the dH GEMM needs them first)
        dy_l = self._rows(dy, ctx["send_tok"], ss, rs)
        # C4b: remote X rows again, on the side stream (only the dW1/dW2 GEMM reads
        # them), unless forward kept them (retain_recv_x)
        x_l = ctx.pop("x_recv", None)
        x_ready = dx_ready = None
        if x_l is None:
            x_l = torch.empty(T + U, d, dtype=x.dtype, device=x.device)
            x_l[:T].copy_(x)
            x_send = ops.gather_rows(x, ctx["send_tok"])
            if streams:
                side.wait_stream(main)
            with sctx():
                self.a2a(x_send, ss, rs, out=x_l[T:])
            if streams:
                x_ready = torch.cuda.Event()
                x_ready.record(side)
                x_l.record_stream(side)
                x_send.record_stream(side)
        elif streams:
            x_ready = torch.cuda.Event()
            x_ready.record(main)
        if streams:
            # torch creates the CUDA event lazily at its first record: create it
            # now so the library gets a real handle to re-record after dX is final
            dx_ready = torch.cuda.Event()
            dx_ready.record(main)
        if n_pairs:
            g = ops.ffn_bwd(dy_l, x_l, w1l, w2l, w3l, ctx["w_l"], ctx["disp_l"], ctx["a_l"], ctx["b_l"],
                            n_pairs, x_ready=x_ready, dx_ready=dx_ready)
        else:  # nothing routed here: zero expert grads
            g = dict(dx=dy_l.new_zeros(T + U, d), dg=torch.zeros(T + U, k, dtype=ctx["w_l"].dtype, device=dy.device),
                     dw1=torch.zeros_like(w1l), dw2=torch.zeros_like(w2l), dw3=torch.zeros_like(w3l))
            if streams:
                dx_ready.record(main)
                main.wait_event(x_ready)
        # C5: per-(remote token, rank) dX partials and the gate-weight gradients back, on the side stream
        with sctx():
            if streams:
                side.wait_event(dx_ready)
                g["dx"].record_stream(side)
                g["dg"].record_stream(side)
            dx_back = self.a2a(g["dx"][T:], rs, ss)
            dg_back = self.a2a(g["dg"][T:], rs, ss)
        if streams:
            main.wait_stream(side)
            dx_back.record_stream(main)
            dg_back.record_stream(main)
        dx_part = ops.combine(dx_back, plan.tim, T, d, P, base=g["dx"][:T])
        dg = ops.slot_grad(ctx["ids"], E, El, P, plan.tim, dg_back, dg_local=g["dg"][:T], self_rank=me)
        dx, dwg = ops.router_backward(dg, x, ctx["wg"], ctx["logits"], ctx["ids"], dx_part, self.renorm)
        # C6: replicated router
        acc = dwg.float() if dwg.element_size() < 4 else dwg  # reduce 16-bit grads in fp32
        if P > 1:
            dist.all_reduce(acc, group=self.group)
        dwg = acc.to(dwg.dtype)
        return dict(dx=dx, dw_gate=dwg, dw1=g["dw1"], dw2=g["dw2"], dw3=g["dw3"], dg=dg)

    def step(self, x, wg, w1l, w2l, w3l, dy):
        y, ctx = self.forward(x, wg, w1l, w2l, w3l)
        return y, self.backward(ctx, dy)
