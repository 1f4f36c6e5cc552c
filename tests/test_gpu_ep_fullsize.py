"""Expert parallel at BASELINE.json's EP shape (T 32768 tokens per rank,
d 4096, h 2048, E 64, k 8), through both exchanges, on one B200: P = 2 ranks
are two processes sharing cuda:0 (the peer-memory exchange maps the other
process's buffers by CUDA IPC; the NCCL-path test stages its all-to-all
through the host over gloo, since NCCL cannot put two ranks on one GPU).

Every rank compares, on every element, its outputs with the single-GPU layer
run on the concatenation of both ranks' tokens (its token slice of y, dX, dg;
its experts' slices of dW1, dW2, dW3; the replicated dW_g).  The single-GPU
layer at this shape is itself checked against the fp64 oracle
(tests/test_gpu_fullsize.py, "ep").  Tolerance 1e-2 normwise: the returned
rows travel in bf16; the rest differs by fp32 summation order."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from moe_inputs import CONFIGS, make_inputs
from tests.test_gpu_ep import _port, staged_a2a

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _nw(a, b):
    a, b = a.float(), b.float()
    den = b.abs().max().item()
    return (a - b).abs().max().item() / den if den else a.abs().max().item()


def _worker(rank, P, port, q, exchange):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    import paper_2601_05296_b200 as M
    c = CONFIGS["ep"]
    T, E, k = c.T, c.E, c.k
    W = make_inputs(T, c.d, c.h, E, k, dtype="bf16", seed=100, device=dev)
    X = [make_inputs(T, c.d, c.h, E, k, dtype="bf16", seed=r, device=dev) for r in range(P)]
    x, dy = X[rank]["x"], X[rank]["dy"]
    if exchange == "p2p":
        from paper_2601_05296_b200.ep_p2p import P2PExpertParallelMoE, PeerGroup
        pg = PeerGroup.from_group(T, c.d, k, E, x.dtype, dev, timeout_s=120.0)
        ep = P2PExpertParallelMoE(pg, E, k)
    else:
        from paper_2601_05296_b200.ep import ExpertParallelMoE
        ep = ExpertParallelMoE(E, k, a2a=staged_a2a)
    lo, hi = ep.local_experts
    wl = [W[n][lo:hi].contiguous() for n in ("w1", "w2", "w3")]
    y, g = ep.step(x, W["w_gate"], *wl, dy)
    torch.cuda.synchronize()
    if exchange == "p2p":
        pg.check()
    rows_received = ep.last_rows_received
    dist.barrier()
    # the single-GPU layer on both ranks' tokens (each rank runs it for itself)
    xa = torch.cat([X[r]["x"] for r in range(P)])
    dya = torch.cat([X[r]["dy"] for r in range(P)])
    logits, ids, w = M.route(xa, W["w_gate"], k)
    disp = M.dispatch_build(ids, E)
    ya, a, b = M.ffn_fwd(xa, W["w1"], W["w2"], W["w3"], w, disp)
    ga = M.ffn_bwd(dya, xa, W["w1"], W["w2"], W["w3"], w, disp, a, b, w_gate=W["w_gate"], logits=logits)
    torch.cuda.synchronize()
    sl = slice(rank * T, (rank + 1) * T)
    errs = {"y": _nw(y, ya[sl]), "dx": _nw(g["dx"], ga["dx"][sl]), "dg": _nw(g["dg"], ga["dg"][sl]),
            "dw_gate": _nw(g["dw_gate"], ga["dw_gate"])}
    for n in ("dw1", "dw2", "dw3"):
        errs[n] = _nw(g[n], ga[n][lo:hi])
    q.put((rank, errs, rows_received))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["p2p", "nccl_path_gloo"])
def test_ep_fullsize_two_ranks_match_single_gpu(exchange):
    P = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, q, exchange)) for r in range(P)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=900) for _ in range(P)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, errs, rows in res:
        print(exchange, "rank", rank, "rows received", rows, {n: round(v, 5) for n, v in errs.items()})
        assert rows > 0
        bad = {n: v for n, v in errs.items() if not v <= TOL}
        assert not bad, (rank, errs)
