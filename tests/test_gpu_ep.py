"""Expert-parallel layer with the real CUDA kernels (C ABI) on one B200.

NCCL cannot place two ranks on one GPU, so the 2-rank case runs two processes
on cuda:0 with gloo and a host-staged all-to-all; every compute step is the
library's (CudaOps).  Compared with the single-GPU path on the concatenated
tokens (ids exact; floats within 1e-2: return rows travel in bf16, SURVEY
§8(e)) and with the fp64 oracle (2e-2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from moe_inputs import make_inputs
from tests._util import BF16_TOL, f64, normwise

pytestmark = pytest.mark.gpu

CFG = dict(T=384, d=256, h=256, E=8, k=2)
CFG_EL1 = dict(T=384, d=256, h=256, E=2, k=2)   # P = 2: one expert per rank, fewer than k


def staged_a2a(send, send_split, recv_split, group=None, out=None):
    res = torch.empty((sum(recv_split),) + tuple(send.shape[1:]), dtype=send.dtype)
    dist.all_to_all_single(res, send.detach().cpu().contiguous(), recv_split, send_split, group=group)
    if out is None:
        return res.to(send.device)
    out.copy_(res)
    return out


def _inputs(P, routing="balanced", c=CFG):
    W = make_inputs(c["T"], c["d"], c["h"], c["E"], c["k"], dtype="bf16", seed=100, routing=routing)
    XS = [make_inputs(c["T"], c["d"], c["h"], c["E"], c["k"], dtype="bf16", seed=r, routing=routing)
          for r in range(P)]
    return W, [(X["x"], X["dy"]) for X in XS]


def _worker(rank, P, port, q, routing, backend="gloo", retain=False, c=CFG):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    gpu = rank if backend == "nccl_multi" else 0
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if backend.startswith("nccl"):  # real NCCL all-to-all and the side-stream overlap of C4b / C5
        dist.init_process_group("nccl", rank=rank, world_size=P, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=P)
    W, XS = _inputs(P, routing, c)
    x, dy = (t.to(dev) for t in XS[rank])
    if backend.startswith("p2p"):  # device-initiated exchange over CUDA-IPC-mapped peer memory
        from paper_2601_05296_b200.ep_p2p import P2PExpertParallelMoE, PeerGroup
        pg = PeerGroup.from_group(c["T"], c["d"], c["k"], c["E"], torch.bfloat16, dev, timeout_s=60.0)
        ep = P2PExpertParallelMoE(pg, c["E"], c["k"])
    else:
        from paper_2601_05296_b200.ep import ExpertParallelMoE
        # gloo_overlap: the side-stream orchestration (C2b / C3 overlap with the row-split
        # GEMMs: x_ready, y_ready, sm_reserve; C4b / C5 in backward) over the host-staged
        # all-to-all -- the only way to run it with received rows on a one-GPU box
        ep = ExpertParallelMoE(c["E"], c["k"], False, a2a=staged_a2a if backend.startswith("gloo") else None,
                               retain_recv_x=retain, overlap=True if backend == "gloo_overlap" else None)
        assert ep._use_streams(x) == (backend.startswith("nccl") or backend == "gloo_overlap")
    lo, hi = ep.local_experts
    wl = [W[n][lo:hi].contiguous().to(dev) for n in ("w1", "w2", "w3")]
    for _ in range(2 if backend.startswith("p2p") else 1):  # p2p: a second step reuses the buffers
        y, g = ep.step(x, W["w_gate"].to(dev), *wl, dy)
    torch.cuda.synchronize()
    if backend.startswith("p2p"):
        pg.check()
    # numpy (pickled by value): torch tensors would be shared by fd and can
    # vanish when this worker exits before the parent reads the queue
    q.put((rank, y.float().cpu().numpy(), {n: v.float().cpu().numpy() for n, v in g.items()}, (lo, hi)))
    dist.barrier()
    dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("P,routing,backend,retain,c", [(2, "balanced", "gloo", False, CFG_EL1),
                                                        (2, "balanced", "nccl_multi", False, CFG_EL1)])
def test_ep_fewer_local_experts_than_k(P, routing, backend, retain, c):
    test_ep_cuda_matches_single_gpu(P, routing, backend, retain, c)


@pytest.mark.parametrize("P,routing,backend,retain", [(1, "balanced", "gloo", False), (2, "balanced", "gloo", False),
                                                      (2, "degenerate", "gloo", False),
                                                      (1, "balanced", "nccl", False), (1, "skewed", "nccl", False),
                                                      (2, "skewed", "gloo", True), (1, "balanced", "nccl", True),
                                                      (2, "balanced", "nccl_multi", False),
                                                      (2, "skewed", "nccl_multi", True),
                                                      # P = 4 and 8 processes sharing one GPU over gloo: the
                                                      # EP config's rank counts (E = 8: 2 experts, then 1 < k)
                                                      (4, "balanced", "gloo", False), (8, "skewed", "gloo", False),
                                                      # the stream orchestration with received rows (U > 0)
                                                      (2, "balanced", "gloo_overlap", False),
                                                      (4, "skewed", "gloo_overlap", False),
                                                      (2, "degenerate", "gloo_overlap", True)])
def test_ep_cuda_matches_single_gpu(P, routing, backend, retain, c=CFG):
    """degenerate routing: every token picks experts 0,1, so rank 1 receives no rows.
    nccl (P = 1): the product path, with C4b / C5 on the side stream.  nccl_multi:
    one rank per GPU over real NCCL all-to-all (skipped with fewer than P GPUs)."""
    if backend.endswith("_multi") and torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs (this box has {torch.cuda.device_count()})")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, q, routing, backend, retain, c)) for r in range(P)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(P)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    compare_with_single_gpu(P, routing, c, res)


@pytest.mark.parametrize("P,routing,backend", [(1, "balanced", "p2p"), (2, "balanced", "p2p"), (2, "skewed", "p2p"),
                                               (2, "degenerate", "p2p"), (4, "balanced", "p2p"),
                                               (2, "balanced", "p2p_multi"), (4, "skewed", "p2p_multi")])
def test_ep_p2p_matches_single_gpu(P, routing, backend):
    """The device-initiated exchange (ep_p2p: CUDA-IPC peer memory, epoch flags,
    no host sync, no NCCL): P processes share cuda:0 (time-sliced contexts, the
    flags spin across them), or one GPU per rank (p2p_multi, skipped with fewer
    GPUs).  Two steps per process: the second reuses the symmetric buffers."""
    test_ep_cuda_matches_single_gpu(P, routing, backend, False, CFG)


@pytest.mark.parametrize("P", [2])
def test_ep_p2p_fewer_local_experts_than_k(P):
    test_ep_cuda_matches_single_gpu(P, "balanced", "p2p", False, CFG_EL1)


def compare_with_single_gpu(P, routing, c, res):
    import paper_2601_05296_b200 as M
    W, XS = _inputs(P, routing, c)
    dev = torch.device("cuda", 0)
    x = torch.cat([a for a, _ in XS]).to(dev)
    dy = torch.cat([b for _, b in XS]).to(dev)
    wg, w1, w2, w3 = (W[n].to(dev) for n in ("w_gate", "w1", "w2", "w3"))
    k = c["k"]
    logits, ids, w = M.route(x, wg, k)
    disp = M.dispatch_build(ids, c["E"])
    y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp)
    g1 = M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits)
    torch.cuda.synchronize()
    fwd = O.layer_forward(f64(x), f64(wg), f64(w1), f64(w2), f64(w3), k, logits=f64(logits))
    bwd = O.layer_backward(fwd, f64(dy), f64(x), f64(wg), f64(w1), f64(w2), f64(w3))
    T = c["T"]
    for rank, ye, ge, (lo, hi) in res:
        sl = slice(rank * T, (rank + 1) * T)
        assert normwise(ye, f64(y[sl])) < 1e-2
        assert normwise(ge["dx"], f64(g1["dx"][sl])) < 1e-2
        assert normwise(ge["dg"], f64(g1["dg"][sl])) < 1e-2
        assert normwise(ge["dw_gate"], f64(g1["dw_gate"])) < 1e-2
        for n in ("dw1", "dw2", "dw3"):
            assert normwise(ge[n], f64(g1[n][lo:hi])) < 1e-2, n
            assert normwise(ge[n], bwd[n][lo:hi]) < BF16_TOL, n
        assert normwise(ye, fwd["y"][sl]) < BF16_TOL
        assert normwise(ge["dx"], bwd["dx"][sl]) < BF16_TOL


@pytest.mark.parametrize("P,routing", [(2, "balanced"), (4, "skewed"), (8, "balanced")])
def test_ep_p2p_virtual_ranks_one_process(P, routing):
    """P ranks in one process on one GPU, one stream each (tests/_p2p_virtual.py):
    the host enqueues all forwards, then all backwards, and never waits -- the
    run can only finish if the EP step has no host sync."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "tests._p2p_virtual", str(P), routing], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ok" in r.stdout
