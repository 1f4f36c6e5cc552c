"""Expert-parallel bookkeeping on CPU: world size 2 (and 4) over gloo.

The EP orchestrator (paper_2601_05296_b200/ep.py) is run with oracle-backed
compute ops (fp64, test-only) and gloo all-to-all, so what is tested is the
host logic: split sizes, send order, per-row payload, the receiver's local
index build, the return exchange and the token-side combine through
token_index_map, and the dW_g all-reduce.  Every rank's outputs must equal the
single-process oracle over the concatenated tokens (fp64, 1e-10)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from moe_inputs import make_inputs
from tests._util import dispatch_sparse as _dispatch_sparse


class OracleOps:
    """Test-only compute for the EP orchestrator: the fp64 oracle on CPU, plus
    numpy restatements of the EP helpers' definitions (include/moeblaze.h)."""

    class D:
        def __init__(self, d, ids):
            self.counts = torch.from_numpy(d["counts"].astype(np.int32))
            self.offs = torch.from_numpy(d["offs"].astype(np.int32))
            self.eti = torch.from_numpy(d["eti"].astype(np.int64))
            self.tim = torch.from_numpy(d["tim"].astype(np.int64))
            self.row_slot = torch.from_numpy(d["row_slot"].astype(np.int64))
            self.ids = ids
            self.raw = d

    def route(self, x, wg, k, renorm):
        r = O.route(x.numpy(), wg.numpy(), k, renorm)
        return torch.from_numpy(r["logits"]), torch.from_numpy(r["ids"]), torch.from_numpy(r["w"])

    def dispatch(self, ids, E, dtype, rows=0):
        if rows:
            return OracleOps.D(_dispatch_sparse(ids.numpy(), E), ids)
        return OracleOps.D(O.dispatch_argsort(ids.numpy(), E), ids)

    def ep_dest(self, ids, E, El, P, self_rank=-1):
        owner = ids.long() // El
        dest = torch.full((ids.shape[0], P), -1, dtype=torch.int32)
        for q in range(P):
            if q != self_rank:
                dest[(owner == q).any(1), q] = q
        return dest

    def local_slots(self, ids, w, E, El, rank, out_ids, out_w):
        mine = (ids.long() // El) == rank
        out_ids.copy_(torch.where(mine, ids.long() - rank * El, -1).to(torch.int32))
        out_w.copy_(torch.where(mine, w, 0.0).to(out_w.dtype))

    def send_meta(self, ids, w, E, El, P, row_slot):
        t, q = row_slot.long() // P, row_slot.long() % P
        e = ids[t].long()
        mine = (e // El) == q[:, None]
        return torch.where(mine, e - q[:, None] * El, -1).to(torch.int32), torch.where(mine, w[t], 0.0)

    def slot_grad(self, ids, E, El, P, send_pos, dg_back, dg_local=None, self_rank=-1):
        T, k = ids.shape
        owner = ids.long() // El
        pos = send_pos.long().gather(1, owner)
        back = dg_back[pos.clamp(min=0), torch.arange(k)[None, :].expand(T, k)] if dg_back.numel() else \
            torch.zeros(T, k, dtype=torch.float64)
        return torch.where(owner == self_rank, dg_local, back) if self_rank >= 0 else back

    def gather_rows(self, src, index):
        return src[index.reshape(-1).long()].clone()

    def read_host(self, t):
        return t.clone()

    def ffn_fwd(self, x, w1, w2, w3, w, disp, rows, **overlap):  # t_ready, x_ready, ...: scheduling only
        f = O.ffn_forward(x.numpy(), w1.numpy(), w2.numpy(), w3.numpy(), disp.ids.numpy(), w.numpy(), disp.raw)
        return torch.from_numpy(f["y"]), torch.from_numpy(f["A"][:rows]), torch.from_numpy(f["B"][:rows])

    def ffn_bwd(self, dy, x, w1, w2, w3, w, disp, a, b, rows, x_ready=None, dx_ready=None):
        g = O.ffn_backward(dy.numpy(), x.numpy(), w1.numpy(), w2.numpy(), w3.numpy(), disp.ids.numpy(), w.numpy(),
                           disp.raw, a.numpy(), b.numpy())
        return {n: torch.from_numpy(np.ascontiguousarray(g[n])) for n in ("dx", "dw1", "dw2", "dw3", "dg")}

    def combine(self, rows, tim, T, d, k, base=None):
        t = tim.reshape(T, k).long()
        out = base.clone() if base is not None else torch.zeros(T, d, dtype=torch.float64)
        if rows.numel():
            out = out + torch.where((t >= 0)[..., None], rows[t.clamp(min=0)], 0.0).sum(1)
        return out

    def router_backward(self, dg, x, wg, logits, ids, dx_partial, renorm):
        rb = O.router_backward(dg.numpy(), x.numpy(), wg.numpy(), logits.numpy(), ids.numpy(), renorm)
        return dx_partial + torch.from_numpy(rb["dx"]), torch.from_numpy(rb["dw_gate"])


def gloo_a2a(send, send_split, recv_split, group=None, out=None):
    res = torch.empty((sum(recv_split),) + tuple(send.shape[1:]), dtype=send.dtype)
    dist.all_to_all_single(res, send.contiguous(), recv_split, send_split, group=group)
    if out is None:
        return res
    out.copy_(res)
    return out


CFG = dict(T=40, d=16, h=24, E=8, k=2)
CFG6 = dict(T=40, d=16, h=24, E=8, k=6)   # k > P: tokens hit several experts per rank (dedup)


def _inputs(rank, P, renorm, routing, c=CFG):
    W = make_inputs(c["T"], c["d"], c["h"], c["E"], c["k"], dtype="fp32", seed=100, routing=routing)
    X = [make_inputs(c["T"], c["d"], c["h"], c["E"], c["k"], dtype="fp32", seed=r, routing=routing) for r in range(P)]
    f = lambda t: t.double()  # noqa: E731
    return {n: f(W[n]) for n in ("w_gate", "w1", "w2", "w3")}, [(f(X[r]["x"]), f(X[r]["dy"])) for r in range(P)]


def _worker(rank, P, port, renorm, routing, q, c=CFG, retain=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    from paper_2601_05296_b200.ep import ExpertParallelMoE
    W, XS = _inputs(rank, P, renorm, routing, c)
    ep = ExpertParallelMoE(c["E"], c["k"], renorm, ops=OracleOps(), a2a=gloo_a2a, retain_recv_x=retain)
    lo, hi = ep.local_experts
    x, dy = XS[rank]
    y, g = ep.step(x, W["w_gate"], W["w1"][lo:hi], W["w2"][lo:hi], W["w3"][lo:hi], dy)
    q.put((rank, y.numpy(), {n: v.numpy() for n, v in g.items()}, (lo, hi), ep.last_rows_sent))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("P,renorm,routing,c,retain", [(1, False, "balanced", CFG, False),
                                                      (2, False, "balanced", CFG, False), (2, True, "skewed", CFG, False),
                                                      (4, False, "balanced", CFG, False),
                                                      (4, False, "degenerate", CFG, False),
                                                      (2, False, "balanced", CFG6, False),
                                                      (4, True, "skewed", CFG6, False),
                                                      (4, False, "skewed", CFG6, True)])
def test_ep_matches_single_process_oracle(P, renorm, routing, c, retain):
    """Every rank's y, dx, dg, dW_g and local expert grads equal the fp64 oracle
    over the concatenated tokens; each token row is sent once per owning rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, renorm, routing, q, c, retain)) for r in range(P)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(P)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    W, XS = _inputs(0, P, renorm, routing, c)
    Xall = torch.cat([x for x, _ in XS]).numpy()
    DYall = torch.cat([dy for _, dy in XS]).numpy()
    Wn = {n: v.numpy() for n, v in W.items()}
    fwd = O.layer_forward(Xall, Wn["w_gate"], Wn["w1"], Wn["w2"], Wn["w3"], c["k"], renorm)
    bwd = O.layer_backward(fwd, DYall, Xall, Wn["w_gate"], Wn["w1"], Wn["w2"], Wn["w3"], renorm)
    T = c["T"]
    El = c["E"] // P
    for rank, y, g, (lo, hi), n_sent in res:
        sl = slice(rank * T, (rank + 1) * T)
        owners = fwd["ids"][sl] // El
        # per-destination dedup; own-rank pairs are computed in place and never sent
        assert n_sent == sum(len(set(row) - {rank}) for row in owners.tolist())
        if c["k"] > P:
            assert n_sent < T * c["k"]
        np.testing.assert_allclose(y, fwd["y"][sl], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(g["dx"], bwd["dx"][sl], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(g["dg"], bwd["dg"][sl], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(g["dw_gate"], bwd["dw_gate"], rtol=1e-10, atol=1e-12)
        for n in ("dw1", "dw2", "dw3"):
            np.testing.assert_allclose(g[n], bwd[n][lo:hi], rtol=1e-10, atol=1e-12)
