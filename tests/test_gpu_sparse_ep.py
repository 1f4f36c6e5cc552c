"""GPU parity of the expert-parallel building blocks
through the C ABI: sparse-slot problems (moe_problem.rows > 0, topk_ids -1 =
empty slot) as run by an EP receiver, and the send-plan helpers moe_ep_dest /
moe_ep_send_meta / moe_ep_slot_grad / moe_combine_rows.  Index work is
bit-exact against the definitions in include/moeblaze.h; floats against the
fp64 oracle (2e-2 bf16, 1e-4 fp32)."""
import numpy as np
import pytest
import torch

import oracle as O
from moe_inputs import make_inputs
from tests._util import BF16_TOL, FP32_TOL, dispatch_sparse, f64, i64, normwise

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def M():
    from paper_2601_05296_b200 import build as B
    B.build()
    import paper_2601_05296_b200 as M
    M._lib.load()
    return M


def _sparse_ids(T, E, k, seed, p_empty):
    """k slots per token, each -1 (empty) or a distinct expert of this rank; with
    E < k (an EP receiver owning fewer experts than a token's k) at most E slots
    of a token are non-empty."""
    g = np.random.default_rng(seed)
    if k <= E:
        ids = np.stack([g.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    else:
        ids = np.full((T, k), -1, np.int32)
        for t in range(T):
            ids[t, g.permutation(k)[:E]] = g.permutation(E)
    ids[g.random((T, k)) < p_empty] = -1
    return ids


@pytest.mark.parametrize("T,E,k,p_empty", [(1, 4, 2, 0.5), (300, 8, 2, 0.3), (5000, 64, 6, 0.7), (4097, 16, 8, 0.9),
                                           (1000, 4, 1, 0.5), (257, 8, 8, 1.0),
                                           # fewer local experts than k (EP with E/P < k)
                                           (600, 1, 2, 0.3), (900, 2, 8, 0.2), (70, 4, 20, 0.5)])
def test_sparse_dispatch_bit_exact(M, T, E, k, p_empty):
    from paper_2601_05296_b200.ep import CudaOps
    ids_np = _sparse_ids(T, E, k, T + k, p_empty)
    n = int((ids_np >= 0).sum())
    d = CudaOps().dispatch(torch.from_numpy(ids_np).to(DEV), E, torch.bfloat16, rows=max(n, 1))
    torch.cuda.synchronize()
    ref = dispatch_sparse(ids_np, E)
    assert np.array_equal(i64(d.counts), ref["counts"])
    assert np.array_equal(i64(d.offs), ref["offs"])
    assert np.array_equal(i64(d.eti)[:n], ref["eti"])
    assert np.array_equal(i64(d.tim), ref["tim"])
    assert np.array_equal(i64(d.row_slot)[:n], ref["row_slot"])


@pytest.mark.parametrize("T,d,h,E,k,dtype,p_empty", [
    (300, 256, 384, 8, 2, "bf16", 0.4), (777, 512, 256, 16, 6, "bf16", 0.6), (200, 128, 128, 4, 1, "bf16", 0.5),
    (96, 64, 96, 4, 3, "fp32", 0.5),
    # E (local experts) < k: Mixtral-like E = 8, k = 2 over 8 ranks -> 1 expert per rank;
    # DeepSeek-like k = 6 over 16 ranks -> 4 experts per rank
    (500, 256, 384, 1, 2, "bf16", 0.3), (640, 128, 256, 4, 6, "bf16", 0.2), (80, 64, 96, 2, 8, "fp32", 0.4),
])
def test_sparse_layer_parity(M, T, d, h, E, k, dtype, p_empty):
    """An EP receiver's problem: token rows with only some slots routed here.
    y_t = sum over the non-empty slots; every gradient as the oracle
    over exactly those (token, expert) rows; d_topk_w = 0 at empty slots."""
    from paper_2601_05296_b200.ep import CudaOps
    inp = make_inputs(T, d, h, E, k, dtype=dtype, seed=5, device=DEV)
    ids_np = _sparse_ids(T, E, k, 11, p_empty)
    n = int((ids_np >= 0).sum())
    ids = torch.from_numpy(ids_np).to(DEV)
    w = torch.rand(T, k, generator=torch.Generator().manual_seed(3)).to(DEV)
    w[ids < 0] = 0
    ops = CudaOps()
    disp = ops.dispatch(ids, E, inp["x"].dtype, rows=n)
    y, a, b = ops.ffn_fwd(inp["x"], inp["w1"], inp["w2"], inp["w3"], w, disp, n)
    g = ops.ffn_bwd(inp["dy"], inp["x"], inp["w1"], inp["w2"], inp["w3"], w, disp, a.clone(), b.clone(), n)
    torch.cuda.synchronize()
    ref = dispatch_sparse(ids_np, E)
    fw = O.ffn_forward(f64(inp["x"]), f64(inp["w1"]), f64(inp["w2"]), f64(inp["w3"]), ids_np, f64(w), ref)
    bw = O.ffn_backward(f64(inp["dy"]), f64(inp["x"]), f64(inp["w1"]), f64(inp["w2"]), f64(inp["w3"]), ids_np,
                        f64(w), ref, fw["A"][:n], fw["B"][:n])
    tol = BF16_TOL if dtype == "bf16" else FP32_TOL
    assert normwise(y, fw["y"]) < tol
    assert normwise(a, fw["A"][:n]) < tol and normwise(b, fw["B"][:n]) < tol
    for name in ("dx", "dw1", "dw2", "dw3"):
        assert normwise(g[name], bw[name]) < tol, name
    assert normwise(g["dg"], bw["dg"]) < tol
    assert torch.all(g["dg"][ids < 0] == 0)
    assert torch.all(y[(ids < 0).all(1)] == 0)


@pytest.mark.parametrize("T,E,k,P", [(1, 8, 2, 2), (1000, 8, 2, 4), (3000, 64, 8, 8), (513, 16, 6, 2), (100, 4, 4, 1)])
def test_ep_plan_helpers_bit_exact(M, T, E, k, P):
    """moe_ep_dest + sparse dispatch = the send plan; moe_ep_send_meta,
    moe_ep_slot_grad and moe_combine_rows (with -1 entries) by definition."""
    from paper_2601_05296_b200.ep import CudaOps
    ops = CudaOps()
    g = np.random.default_rng(T + P)
    ids_np = np.stack([g.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    El = E // P
    ids = torch.from_numpy(ids_np).to(DEV)
    w = torch.from_numpy(g.random((T, k)).astype(np.float32)).to(DEV)
    dest = ops.ep_dest(ids, E, El, P)
    owner = ids_np // El
    ref_dest = np.full((T, P), -1)
    for q in range(P):
        ref_dest[(owner == q).any(1), q] = q
    assert np.array_equal(i64(dest), ref_dest)
    plan = ops.dispatch(dest, P, torch.bfloat16, rows=T * min(k, P))
    n_send = int(plan.offs[P].item())
    assert n_send == sum(len(set(r)) for r in owner.tolist())
    rs = plan.row_slot[:n_send]
    sid, sw = ops.send_meta(ids, w, E, El, P, rs)
    rs_np = i64(rs)
    t, q = rs_np // P, rs_np % P
    mine = owner[t] == q[:, None]
    assert np.array_equal(i64(sid), np.where(mine, ids_np[t] - q[:, None] * El, -1))
    assert np.array_equal(sw.cpu().numpy(), np.where(mine, w.cpu().numpy()[t], 0))
    dg_back = torch.from_numpy(g.random((n_send, k)).astype(np.float32)).to(DEV)
    dg = ops.slot_grad(ids, E, El, P, plan.tim, dg_back)
    pos = i64(plan.tim)[np.arange(T)[:, None], owner]
    assert np.array_equal(dg.cpu().numpy(), dg_back.cpu().numpy()[pos, np.arange(k)[None, :]])
    rows = torch.randn(n_send, 256, device=DEV).to(torch.bfloat16)
    out = ops.combine(rows, plan.tim, T, 256, P)
    tim = i64(plan.tim)
    r64 = f64(rows)
    ref = np.zeros((T, 256))
    for j in range(P):  # fixed slot order, fp32 accumulation
        ref = (ref.astype(np.float32) + np.where(tim[:, j:j + 1] >= 0, r64[np.maximum(tim[:, j], 0)], 0)
               .astype(np.float32)).astype(np.float64)
    assert np.array_equal(f64(out), f64(torch.from_numpy(ref.astype(np.float32)).to(torch.bfloat16)))


@pytest.mark.parametrize("T,n_valid,d,h,E,k,upper", [(900, 300, 256, 384, 4, 2, False), (1024, 1000, 512, 256, 8, 2, True),
                                                     (500, 0, 256, 256, 2, 2, True)])
def test_token_rows_bound_and_upper_bound_rows(M, T, n_valid, d, h, E, k, upper):
    """moe_dispatch.token_rows (the peer-memory EP receiver's T + U bound on the
    device) with token rows >= n_valid carrying no slot, and moe_problem.rows
    given as an upper bound (T*k) instead of the exact count: y, dX, dg of the
    rows < n_valid and every weight gradient are bit-identical to the exact,
    unbounded call (same kernels, same rows; only the zeroing / finalize range
    and the buffer sizes differ)."""
    from paper_2601_05296_b200.ep import CudaOps
    inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=7, device=DEV)
    ids_np = _sparse_ids(T, E, k, 13, 0.3)
    ids_np[n_valid:] = -1
    n = int((ids_np >= 0).sum())
    ids = torch.from_numpy(ids_np).to(DEV)
    w = torch.rand(T, k, generator=torch.Generator().manual_seed(4)).to(DEV)
    w[ids < 0] = 0
    ops = CudaOps()
    res = []
    for bounded in (False, True):
        rows = T * k if (bounded and upper) else max(n, 1)
        disp = ops.dispatch(ids, E, inp["x"].dtype, rows=rows)
        if bounded:
            disp.token_rows = torch.tensor([n_valid], dtype=torch.int32, device=DEV)
        y, a, b = ops.ffn_fwd(inp["x"], inp["w1"], inp["w2"], inp["w3"], w, disp, rows)
        g = ops.ffn_bwd(inp["dy"], inp["x"], inp["w1"], inp["w2"], inp["w3"], w, disp, a, b, rows)
        torch.cuda.synchronize()
        res.append((y[:n_valid].clone(), g))
    (y0, g0), (y1, g1) = res
    assert torch.equal(y0, y1)
    assert torch.equal(g0["dx"][:n_valid], g1["dx"][:n_valid])
    assert torch.equal(g0["dg"][:n_valid], g1["dg"][:n_valid])
    for name in ("dw1", "dw2", "dw3"):
        assert torch.equal(g0[name], g1[name]), name


@pytest.mark.parametrize("T,d,h,E,k,dtype,p_empty,t_ready", [
    (700, 256, 384, 8, 2, "bf16", 0.0, 311),      # dense slots, split inside most segments
    (700, 256, 384, 8, 2, "bf16", 0.0, 0),        # nothing resident: all rows in the second launch
    (700, 256, 384, 8, 2, "bf16", 0.0, 700),      # everything resident: second launch empty
    (2000, 512, 256, 16, 6, "bf16", 0.5, 1337),   # sparse receiver rows (EP), k = 6
    (900, 256, 384, 1, 2, "bf16", 0.3, 450),      # one local expert < k
    (96, 64, 96, 4, 3, "fp32", 0.5, 40),          # fp32: one launch after x_ready
])
def test_ffn_fwd_row_split_identical(M, T, d, h, E, k, dtype, p_empty, t_ready):
    """moe_ffn_fwd_ex (NEXT-1 forward overlap): the up-projection split at the rows
    whose token is < t_ready, the rest after an event; the down projection of the
    rows from the split on first, y rows [t_ready, T) final at y_ready, then the
    rest on fewer SMs -- A, B and y bit-identical to one moe_ffn_fwd call (k <= 2:
    the red.add combine onto zero is order-free), and row_split[e] the lower bound
    of t_ready in expert e's ascending segment."""
    from paper_2601_05296_b200 import _lib as L
    from paper_2601_05296_b200.ep import CudaOps
    inp = make_inputs(T, d, h, E, k, dtype=dtype, seed=9, device=DEV)
    ids_np = _sparse_ids(T, E, k, 21, p_empty)
    n = int((ids_np >= 0).sum())
    ids = torch.from_numpy(ids_np).to(DEV)
    w = torch.rand(T, k, generator=torch.Generator().manual_seed(4)).to(DEV)
    w[ids < 0] = 0
    ops = CudaOps()
    disp = ops.dispatch(ids, E, inp["x"].dtype, rows=n)
    x, w1, w2, w3 = inp["x"], inp["w1"], inp["w2"], inp["w3"]
    y0, a0, b0 = ops.ffn_fwd(x, w1, w2, w3, w, disp, n)
    p = L.problem(T, d, h, E, k, x.dtype, rows=n)
    split = torch.empty(E, dtype=torch.int32, device=DEV)
    L.moe_dispatch_row_split(p, disp.c(), t_ready, split)
    torch.cuda.synchronize()
    offs, eti = i64(disp.offs), i64(disp.eti)[:n]
    ref = [offs[e] + int(np.searchsorted(eti[offs[e]:offs[e + 1]], t_ready, side="left")) for e in range(E)]
    assert np.array_equal(i64(split), np.array(ref))
    # X rows from t_ready on are written only after the event the split launch waits on
    xs = x.clone()
    xs[t_ready:] = 0
    side = torch.cuda.Stream()
    ev = torch.cuda.Event()
    ev.record()
    side.wait_event(ev)
    with torch.cuda.stream(side):
        torch.cuda._sleep(20_000_000)  # the late rows land well after the first launch has started
        xs[t_ready:].copy_(x[t_ready:])
        ready = torch.cuda.Event()
        ready.record(side)
    y_ready = torch.cuda.Event()
    y_ready.record()
    y1, a1, b1 = ops.ffn_fwd(xs, w1, w2, w3, w, disp, n, t_ready=t_ready, x_ready=ready, y_ready=y_ready,
                             sm_reserve=40)
    # what a C3 exchange would read at y_ready: the y rows from t_ready on, already final
    # (the local rows' down projection runs after it, on 148 - 40 SMs)
    grab = torch.cuda.Stream()
    grab.wait_event(y_ready)
    with torch.cuda.stream(grab):
        y_hi = y1[t_ready:].clone()
    torch.cuda.synchronize()
    if k <= 2:  # a token's rows are all in one launch: its red.adds onto zero are order-free
        assert torch.equal(y1, y0)
        assert torch.equal(y_hi, y0[t_ready:])
    else:
        assert normwise(f64(y1), f64(y0)) < 1e-2
        if t_ready < T:
            assert normwise(f64(y_hi), f64(y0[t_ready:])) < 1e-2
    assert torch.equal(a1, a0) and torch.equal(b1, b0)
