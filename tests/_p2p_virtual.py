"""P expert-parallel ranks inside ONE process on one GPU, each on its own CUDA
stream, exchanging over the peer-memory kernels (ep_p2p) with direct
addresses.  The host enqueues every rank's whole forward, then every rank's
whole backward, without ever waiting on the GPU: if any step of the EP path
synchronised the host, rank 0's wait for rank 1 would never be satisfied and
the flags' timeout would fail the run.  Run as a subprocess by
tests/test_gpu_ep.py, with two settings that must precede the CUDA context:
CUDA_DEVICE_MAX_CONNECTIONS=32 (with fewer hardware queues than streams two
ranks' streams can share a queue, and a rank's spin-wait would block the peer
kernel queued behind it) and CUDA_MODULE_LOADING=EAGER (a lazily loaded
kernel's first launch waits for the context to go idle, i.e. for rank 0's
spin-wait, which only rank 1's not-yet-enqueued signal can end: with one host
thread driving every rank that is a deadlock; one process per rank, the
deployment, only delays the first step, see ep_p2p.py).

usage: python -m tests._p2p_virtual P routing [steps]"""
import os
import sys

os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"
os.environ["CUDA_MODULE_LOADING"] = "EAGER"

import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.test_gpu_ep import CFG, _inputs, compare_with_single_gpu  # noqa: E402
from paper_2601_05296_b200.ep_p2p import P2PExpertParallelMoE, PeerGroup  # noqa: E402


def main(P, routing, steps=2):
    c = CFG
    dev = torch.device("cuda", 0)
    W, XS = _inputs(P, routing, c)
    pgs = PeerGroup.virtual(P, c["T"], c["d"], c["k"], c["E"], torch.bfloat16, dev, timeout_s=20.0)
    eps = [P2PExpertParallelMoE(pg, c["E"], c["k"]) for pg in pgs]
    streams = [torch.cuda.Stream(dev) for _ in range(P)]
    wg = W["w_gate"].to(dev)
    xs = [(x.to(dev), dy.to(dev)) for x, dy in XS]
    wls = []
    for ep in eps:
        lo, hi = ep.local_experts
        wls.append([W[n][lo:hi].contiguous().to(dev) for n in ("w1", "w2", "w3")])
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    for _ in range(steps):
        outs = []
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                outs.append(eps[r].forward(xs[r][0], wg, *wls[r]))
        grads = []
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                grads.append(eps[r].backward(outs[r][1], xs[r][1]))
    torch.cuda.synchronize()
    for pg in pgs:
        pg.check()
    res = [(r, outs[r][0].float().cpu().numpy(), {n: v.float().cpu().numpy() for n, v in grads[r].items()},
            eps[r].local_experts) for r in range(P)]
    compare_with_single_gpu(P, routing, c, res)
    print(f"p2p virtual P={P} {routing}: ok")


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 2)
