"""Expert-parallel MoEBlaze layer with a device-initiated exchange over peer
memory: no host sync in the step (the paper names
distribution as future work).

The NCCL path (ep.py) reads the all-to-all split sizes on the host once per
step, because NCCL's all_to_all_single and the receive buffers are sized on
the host.  Here every rank owns a fixed set of receive buffers (the
"symmetric" buffers: one allocation, the same layout on every rank) sized for
the worst case -- P*T token rows, since a rank sends each of its T tokens at
most once to each rank (per-destination dedup) -- and every peer maps them
(CUDA IPC; over NVLink / NVSwitch on a multi-GPU node).  The library's
moe_ep_* kernels then move rows with loads / stores to peer addresses and
order the ranks with epoch flags in peer memory (include/moeblaze.h,
"Device-initiated expert-parallel exchange"), so the host only enqueues.

Step e on rank `me` (every phase signals all ranks, itself included):
  ENTER      signal + wait: every rank has finished step e-1, so its buffers
             (and its count matrix) may be overwritten.
  route, send plan (moe_ep_dest without self + moe_dispatch_build over ranks).
  COUNTS     moe_ep_publish_counts: this rank's row of every rank's count
             matrix; the local tokens are copied into rows [0, T) meanwhile.
  ROWS       moe_ep_push_rows x3: X rows, the tokens' k global expert ids and
             gate weights, gathered straight from the source arrays into the
             owners' buffers at row T + sum_{s<me} cmat[s][q] (no send buffer).
  receiver   moe_ep_recv_prepare (global -> local ids, -1 tail), dispatch over
             the P*T rows (sparse slots, rows = the worst case), moe_ffn_fwd_ex
             into the symmetric `out` buffer: the received rows' down
             projection and y first (rows >= T), then the local rows'.
  Y          signalled from a side stream as soon as the received rows' y is
             final (y_ready), so peers pull while this rank computes its own
             rows; wait; moe_ep_pull_combine: y[t] = local partial + the
             owners' rows of t, read from peer memory (fused combine).
Backward: DY push of dY rows; moe_ffn_bwd data stage (dX rows into `out`, gate
grads into `dg`, X still in the symmetric `x` buffer -- nothing is sent twice);
DX signal; then the dW1/dW2 and dW3 stages on this stream while a side stream
runs the exchange tail: DX wait, pull-combine of dX, moe_ep_pull_slot_grad of
dg, router backward into the symmetric `dwg`, DWG signal + wait,
moe_ep_pull_sum = the all-reduce of the replicated router's gradient (rank
order, identical on every rank); the streams join before returning.

Buffer reuse is safe by these happens-before chains: peers write my x / ids /
w / dy / cmat only after ENTER of the next step (after my whole backward);
my `out` is overwritten by dX only after the DY wait (every peer pushed dY,
so it finished pulling y); `dg` / `dwg` / `out` are read by peers in step e
and rewritten by me only after ENTER e+1.

Kernel loading.  With CUDA's lazy module loading, the first launch of a kernel
may wait for the context to go idle -- i.e. for a pending spin-wait.  With one
process per rank (the deployment) that only delays the first step: every wait
depends on signals the peers issue earlier in the same program order.  A
single process driving several ranks (PeerGroup.virtual, tests) must load
eagerly (CUDA_MODULE_LOADING=EAGER) or it deadlocks until the wait times out.

Cost of host-sync freedom: the receive-side problem has P*T token rows and
P*T*min(k, El) routed-row capacity (A, B and the FFN workspace are sized for
it; the kernels process only the actual rows: the GEMMs read expert_offsets
on the device, the accumulator zeroing / finalize read the T + U bound that
moe_ep_recv_prepare writes into moe_dispatch.token_rows), the same trade as
fixed-capacity low-latency EP dispatch.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import _lib as L
from .ep import CudaOps

_ALIGN = 256


def _round(n, a=_ALIGN):
    return (n + a - 1) // a * a


def _layout(P, T, d, k, E, dtype):
    """Symmetric-buffer layout: name -> (byte offset, shape, dtype)."""
    T_cap = P * T
    fields = [("flags", (L.MOE_EP_NPHASE * P,), torch.int64), ("cmat", (P * P,), torch.int32),
              ("x", (T_cap, d), dtype), ("dy", (T_cap, d), dtype), ("out", (T_cap, d), dtype),
              ("ids", (T_cap, k), torch.int32), ("w", (T_cap, k), torch.float32),
              ("dg", (T_cap, k), torch.float32), ("dwg", (E, d), dtype)]
    out, o = {}, 0
    for name, shape, dt in fields:
        out[name] = (o, shape, dt)
        o += _round(math.prod(shape) * torch.empty((), dtype=dt).element_size())
    return out, o


class PeerGroup:
    """One rank's symmetric buffers and the peers' addresses of theirs."""

    def __init__(self, P, rank, T, d, k, E, dtype, device, timeout_s=30.0):
        self.P, self.rank, self.T, self.d, self.k, self.E, self.dtype = P, rank, T, d, k, E, dtype
        self.T_cap = P * T
        self.layout, nbytes = _layout(P, T, d, k, E, dtype)
        self.raw = torch.zeros(nbytes, dtype=torch.uint8, device=device)  # flags = 0: no epoch seen yet
        self.buf = {n: self.raw[o:o + math.prod(s) * torch.empty((), dtype=dt).element_size()].view(dt).view(s)
                    for n, (o, s, dt) in self.layout.items()}
        self.arrive = torch.zeros(L.MOE_EP_NPHASE, dtype=torch.int32, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.timeout_ns = int(timeout_s * 1e9)
        self._mapped = []
        self.g = None

    def connect(self, bases):
        """bases[q] = rank q's `raw` as addressed from this process."""
        dev = self.raw.device
        self.tables = {n: torch.tensor([b + o for b in bases], dtype=torch.int64, device=dev)
                       for n, (o, _, _) in self.layout.items()}
        self.g = L.MoeEpPeers(self.P, self.rank, self.tables["flags"].data_ptr(), self.tables["cmat"].data_ptr(),
                              self.arrive.data_ptr(), self.status.data_ptr(), self.timeout_ns)

    @classmethod
    def virtual(cls, P, T, d, k, E, dtype, device, timeout_s=30.0):
        """P ranks inside this process on one device (tests): each rank's kernels
        must run on its own stream; the peers' addresses are direct."""
        gs = [cls(P, r, T, d, k, E, dtype, device, timeout_s) for r in range(P)]
        bases = [g.raw.data_ptr() for g in gs]
        for g in gs:
            g.connect(bases)
        torch.cuda.synchronize(device)
        return gs

    @classmethod
    def from_group(cls, T, d, k, E, dtype, device, group=None, timeout_s=30.0):
        """One rank per process: map every rank's buffers through CUDA IPC (the
        handles travel once over `group`, any backend)."""
        P, rank = dist.get_world_size(group), dist.get_rank(group)
        g = cls(P, rank, T, d, k, E, dtype, device, timeout_s)
        torch.cuda.synchronize(device)  # zeroed before any peer can signal into it
        mine = L.ipc_handle(g.raw)
        allh = [None] * P
        dist.all_gather_object(allh, mine, group=group)
        bases = []
        with torch.cuda.device(device):
            for q, (h, off) in enumerate(allh):
                if q == rank:
                    bases.append(g.raw.data_ptr())
                else:
                    ptr, base = L.ipc_open(h, off)
                    g._mapped.append(base)
                    bases.append(ptr)
        g.connect(bases)
        dist.barrier(group)  # every rank mapped (and zeroed) before the first signal
        return g

    def check(self):
        """Raise if a wait of this rank timed out (a host read: call outside timed loops)."""
        s = int(self.status.item())
        if s:
            raise L.MoEError(f"peer exchange: rank {self.rank} timed out waiting for phase {s - 1}")

    def close(self):
        for b in self._mapped:
            L.ipc_close(b)
        self._mapped = []


class P2PExpertParallelMoE:
    """One MoE layer, expert-parallel over the ranks of `peers`, exchange over
    peer memory (no host sync, no NCCL).  Same math and results as
    ep.ExpertParallelMoE (per-destination dedup, local pairs never travel)."""

    SM_RESERVE = 2  # SMs the local rows' down projection leaves free for the Y signal kernel

    def __init__(self, peers: PeerGroup, E, k, renormalize=False):
        self.peers = peers
        self.P, self.rank = peers.P, peers.rank
        if E % self.P:
            raise ValueError(f"E={E} not divisible by {self.P} ranks")
        if E != peers.E or k != peers.k:
            raise ValueError("peer buffers were sized for another (E, k)")
        self.E, self.k, self.renorm = E, k, renormalize
        self.El = E // self.P
        self.local_experts = (self.rank * self.El, (self.rank + 1) * self.El)
        self.ops = CudaOps()
        self.epoch = 0
        self._last = None

    # the last step's row counts live on the device: these read them (host sync,
    # for reports outside timed regions only)
    @property
    def last_rows_received(self):
        return int(self._last[1].offs[-1].item()) if self._last else 0

    @property
    def last_rows_sent(self):
        return int(self._last[0].offs[-1].item()) if self._last else 0

    def forward(self, x, wg, w1l, w2l, w3l):
        pg, ops, P, El, k, E, me = self.peers, self.ops, self.P, self.El, self.k, self.E, self.rank
        G, buf, tab = pg.g, pg.buf, pg.tables
        T, d = x.shape
        if T != pg.T or d != pg.d or x.dtype != pg.dtype:
            raise ValueError("x does not match the peer buffers' (T, d, dtype)")
        h = w1l.shape[1]
        T_cap = pg.T_cap
        self.epoch += 1
        e = self.epoch
        L.moe_ep_signal(G, L.MOE_EP_PH_ENTER, e)
        L.moe_ep_wait(G, L.MOE_EP_PH_ENTER, e)
        logits, ids, w = ops.route(x, wg, k, self.renorm)
        dest = ops.ep_dest(ids, E, El, P, self_rank=me)
        n_send_max = T * min(k, P)
        plan = ops.dispatch(dest, P, x.dtype, rows=n_send_max)
        L.moe_ep_publish_counts(G, plan.counts, e)
        # the local tokens' rows and own-rank slots (no peer involved)
        L.moe_gather_rows(x, None, buf["x"][:T])
        ops.local_slots(ids, w, E, El, me, buf["ids"][:T], buf["w"][:T])
        L.moe_ep_wait(G, L.MOE_EP_PH_COUNTS, e)
        es = x.element_size()
        L.moe_ep_push_rows(G, x, plan.eti, plan.offs, n_send_max, d * es, T, tab["x"], -1, e)
        L.moe_ep_push_rows(G, ids, plan.eti, plan.offs, n_send_max, k * 4, T, tab["ids"], -1, e)
        L.moe_ep_push_rows(G, w, plan.eti, plan.offs, n_send_max, k * 4, T, tab["w"], L.MOE_EP_PH_ROWS, e)
        L.moe_ep_wait(G, L.MOE_EP_PH_ROWS, e)
        token_rows = torch.empty(1, dtype=torch.int32, device=x.device)  # T + U, known on the device only
        L.moe_ep_recv_prepare(G, T, T_cap, k, El, buf["ids"], buf["w"], token_rows)
        n_cap = T_cap * min(k, El)
        disp_l = ops.dispatch(buf["ids"], El, x.dtype, rows=n_cap)
        disp_l.token_rows = token_rows
        p = L.problem(T_cap, d, h, El, k, x.dtype, rows=n_cap)
        a_l = torch.empty(n_cap, h, dtype=x.dtype, device=x.device)
        b_l = torch.empty(n_cap, h, dtype=x.dtype, device=x.device)
        ws = L.workspace(p, L.MOE_OP_FFN_FWD, x.device)
        # the received rows' down projection and y first (rows [T, T + U) of `out`): y_ready
        # fires before the local rows' down projection, and the Y signal goes out from a side
        # stream at that moment, so the owners of those tokens pull them while this rank still
        # computes its own rows (C3 overlap); the GEMM leaves SM_RESERVE SMs free so the signal
        # kernel is not queued behind it
        main = torch.cuda.current_stream()
        split = torch.empty(El, dtype=torch.int32, device=x.device)
        L.moe_dispatch_row_split(p, disp_l.c(), T, split)
        y_ready = torch.cuda.Event()
        y_ready.record(main)  # created now; re-recorded by the library
        L.moe_ffn_fwd_ex(p, buf["x"], w1l, w2l, w3l, buf["w"], disp_l.c(), a_l, b_l, None, buf["out"], ws,
                         row_split=split, y_ready=y_ready, t_ready=T, sm_reserve=self.SM_RESERVE)
        side = self._side_stream(x.device)
        side.wait_event(y_ready)
        with torch.cuda.stream(side):
            L.moe_ep_signal(G, L.MOE_EP_PH_Y, e)
        main.wait_stream(side)  # later work on this stream is ordered after the signal
        del ws
        L.moe_ep_wait(G, L.MOE_EP_PH_Y, e)
        y = torch.empty(T, d, dtype=x.dtype, device=x.device)
        L.moe_ep_pull_combine(G, L.problem(T, d, 128, E, k, x.dtype), tab["out"], T, plan.offs, plan.tim,
                              buf["out"][:T], y)
        self._last = (plan, disp_l)
        ctx = dict(epoch=e, x=x, wg=wg, w1l=w1l, w2l=w2l, w3l=w3l, logits=logits, ids=ids, plan=plan,
                   disp_l=disp_l, a_l=a_l, b_l=b_l, n_cap=n_cap, n_send_max=n_send_max)
        return y, ctx

    def backward(self, ctx, dy):
        pg, P, El, k, E, me = self.peers, self.P, self.El, self.k, self.E, self.rank
        G, buf, tab = pg.g, pg.buf, pg.tables
        e = ctx["epoch"]
        if e != self.epoch:
            raise RuntimeError("P2PExpertParallelMoE: backward must follow its own forward (the symmetric "
                               "buffers hold one step)")
        x, plan, w1l, w2l, w3l = ctx["x"], ctx["plan"], ctx["w1l"], ctx["w2l"], ctx["w3l"]
        T, d = x.shape
        h = w1l.shape[1]
        T_cap, n_cap = pg.T_cap, ctx["n_cap"]
        L.moe_gather_rows(dy, None, buf["dy"][:T])
        L.moe_ep_push_rows(G, dy, plan.eti, plan.offs, ctx["n_send_max"], d * dy.element_size(), T, tab["dy"],
                           L.MOE_EP_PH_DY, e)
        L.moe_ep_wait(G, L.MOE_EP_PH_DY, e)
        p = L.problem(T_cap, d, h, El, k, x.dtype, rows=n_cap)
        ws = L.workspace(p, L.MOE_OP_FFN_BWD, x.device)
        a_l, b_l, dc = ctx.pop("a_l"), ctx.pop("b_l"), ctx["disp_l"].c()
        args = (p, buf["dy"], buf["x"], w1l, w2l, w3l, buf["w"], dc, a_l, b_l, None)
        # data grads: dX rows into `out`, gate grads into `dg` -- then peers may pull them
        L.moe_ffn_bwd(*args, buf["out"], None, None, None, buf["dg"], None, ws, stages=L.MOE_BWD_DATA)
        L.moe_ep_signal(G, L.MOE_EP_PH_DX, e)
        # the exchange tail runs on a side stream while this stream computes dW1/dW2
        # and dW3: wait for every owner's dX rows, pull-combine them and the gate
        # grads, router backward, and the dW_g all-reduce.  Everything it touches
        # is allocated here, on this stream, and stays referenced until the join.
        wg = ctx["wg"]
        dx_part = torch.empty(T, d, dtype=x.dtype, device=x.device)
        dx = torch.empty_like(dx_part)
        dg = torch.empty(T, k, dtype=torch.float32, device=x.device)
        dwg = torch.empty_like(wg)
        pr = L.problem(T, d, 128, E, k, x.dtype, self.renorm)
        ws_r = L.workspace(pr, L.MOE_OP_ROUTER_BWD, x.device)
        main = torch.cuda.current_stream()
        side = self._side_stream(x.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            L.moe_ep_wait(G, L.MOE_EP_PH_DX, e)
            pc = L.problem(T, d, 128, E, k, x.dtype)
            L.moe_ep_pull_combine(G, pc, tab["out"], T, plan.offs, plan.tim, buf["out"][:T], dx_part)
            L.moe_ep_pull_slot_grad(G, pc, El, ctx["ids"], tab["dg"], T, plan.offs, plan.tim, buf["dg"][:T], dg)
            router = L.MoeRouterBwd(wg.data_ptr(), ctx["logits"].data_ptr(), ctx["ids"].data_ptr(),
                                    buf["dwg"].data_ptr())
            L.moe_router_backward(pr, dg, x, router, dx_part, dx, ws_r)
            L.moe_ep_signal(G, L.MOE_EP_PH_DWG, e)
            L.moe_ep_wait(G, L.MOE_EP_PH_DWG, e)
            L.moe_ep_pull_sum(G, tab["dwg"], wg.numel(), L._dtype_code(wg.dtype), dwg)
        dw1, dw2 = torch.empty_like(w1l), torch.empty_like(w2l)
        L.moe_ffn_bwd(*args, buf["out"], dw1, dw2, None, buf["dg"], None, ws, stages=L.MOE_BWD_DW12)
        for t in (a_l, b_l):  # dA / dB are dead after the dW1 / dW2 GEMM
            t.untyped_storage().resize_(0)
        dw3 = torch.empty_like(w3l)
        L.moe_ffn_bwd(*args, buf["out"], None, None, dw3, buf["dg"], None, ws, stages=L.MOE_BWD_DW3)
        main.wait_stream(side)
        del ws, ws_r
        return dict(dx=dx, dw_gate=dwg, dw1=dw1, dw2=dw2, dw3=dw3, dg=dg)

    def _side_stream(self, device):
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=device)
        return self._side

    def step(self, x, wg, w1l, w2l, w3l, dy):
        y, ctx = self.forward(x, wg, w1l, w2l, w3l)
        return y, self.backward(ctx, dy)
