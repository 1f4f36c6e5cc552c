"""HostPipeline: overlapped host<->device transfers give the same results as
sequential steps (different inputs per step, rotating device buffers)."""
import pytest
import torch

from moe_inputs import make_inputs

pytestmark = pytest.mark.gpu


def test_host_pipeline_matches_sequential():
    import paper_2601_05296_b200 as M
    from paper_2601_05296_b200.pipeline import HostPipeline
    dev = torch.device("cuda", 0)
    T, d, h, E, k = 256, 128, 256, 8, 2
    W = make_inputs(T, d, h, E, k, dtype="bf16", seed=5, device=dev)
    params = [torch.nn.Parameter(W[n]) for n in ("w_gate", "w1", "w2", "w3")]
    steps = [make_inputs(T, d, h, E, k, dtype="bf16", seed=50 + i) for i in range(5)]
    xs = [s["x"].pin_memory() for s in steps]
    dys = [s["dy"].pin_memory() for s in steps]

    def layer_step(xd, dyd):
        xl = xd.detach().requires_grad_(True)
        y = M.moe_layer(xl, *params, k)
        y.backward(dyd)
        return y, xl.grad

    ref = []
    for x, dy in zip(xs, dys):
        y, dx = layer_step(x.to(dev), dy.to(dev))
        ref.append((y.cpu(), dx.cpu()))
    ys = [torch.empty_like(x).pin_memory() for x in xs]
    dxs = [torch.empty_like(x).pin_memory() for x in xs]
    HostPipeline(layer_step, xs[0].shape, xs[0].dtype, dev).run(xs, dys, ys, dxs)
    torch.cuda.synchronize()
    for (ry, rdx), y, dx in zip(ref, ys, dxs):
        assert torch.equal(ry, y)
        assert torch.equal(rdx, dx)
    # the traced run (bench.py's e2e diagnostics) gives the same results and sane timings
    from paper_2601_05296_b200.pipeline import trace_summary
    for t in ys + dxs:
        t.zero_()
    tr = []
    HostPipeline(layer_step, xs[0].shape, xs[0].dtype, dev).run(xs, dys, ys, dxs, trace=tr)
    torch.cuda.synchronize()
    for (ry, rdx), y, dx in zip(ref, ys, dxs):
        assert torch.equal(ry, y) and torch.equal(rdx, dx)
    summ = trace_summary(tr)
    assert len(tr) == 1 + len(xs)
    for key in ("h2d", "comp", "d2h", "run_ms_per_step"):
        assert summ[key] > 0, (key, summ)
