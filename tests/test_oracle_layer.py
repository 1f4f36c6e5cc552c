"""Pins for the oracle's routing, forward and backward (CPU only).

Each test checks the oracle against something other than itself: brute-force
sorting, closed-form special cases (textbook SwiGLU MLP via torch.nn.functional),
invariants, an independent dense-masked torch autograd formulation, and central
finite differences in fp64.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
from moe_inputs import make_inputs


def _np(t):
    return t.double().numpy()


def _problem(T=24, d=16, h=24, E=4, k=2, seed=0, routing="balanced"):
    inp = make_inputs(T, d, h, E, k, dtype="fp32", seed=seed, routing=routing)
    return {n: _np(v) for n, v in inp.items()}


# ---------------------------------------------------------------- routing
def test_topk_brute_force_sort():
    """ids = k largest logits, descending, ties -> lower id; checked by a plain
    python sort of each row."""
    rng = np.random.default_rng(1)
    logits = rng.integers(-3, 3, size=(50, 7)).astype(np.float64)  # many exact ties
    p, ids, w = O.topk_from_logits(logits, 3)
    for t in range(50):
        ref = sorted(range(7), key=lambda e: (-logits[t, e], e))[:3]
        assert ids[t].tolist() == ref
        ex = np.exp(logits[t] - logits[t].max())
        assert np.allclose(w[t], (ex / ex.sum())[ref], rtol=1e-15, atol=0)


def test_topk_k_equals_E_sums_to_one():
    rng = np.random.default_rng(2)
    logits = rng.normal(size=(20, 5))
    p, ids, w = O.topk_from_logits(logits, 5)
    assert np.allclose(w.sum(1), 1.0, atol=1e-14)
    assert all(sorted(r) == list(range(5)) for r in ids.tolist())
    _, _, wr = O.topk_from_logits(logits, 2, renormalize=True)
    assert np.allclose(wr.sum(1), 1.0, atol=1e-14)


def test_route_logits_are_matmul():
    P = _problem()
    r = O.route(P["x"], P["w_gate"], 2)
    ref = np.einsum("td,ed->te", P["x"], P["w_gate"])
    assert np.allclose(r["logits"], ref, rtol=1e-13, atol=1e-13)


# ---------------------------------------------------------------- forward special cases
def _mlp_torch(x, w1, w2, w3):
    """Textbook SwiGLU MLP, SiLU(x W1) * (x W2) W3, torch fp64."""
    x, w1, w2, w3 = (torch.from_numpy(np.ascontiguousarray(a)) for a in (x, w1, w2, w3))
    return F.linear(F.silu(F.linear(x, w1)) * F.linear(x, w2), w3).numpy()


def test_single_expert_is_plain_swiglu_mlp():
    """E = k = 1 => g = 1 => y = SwiGLU-MLP(x)."""
    P = _problem(E=1, k=1)
    f = O.layer_forward(P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], 1)
    ref = _mlp_torch(P["x"], P["w1"][0], P["w2"][0], P["w3"][0])
    assert np.allclose(f["y"], ref, rtol=1e-12, atol=1e-12)
    assert np.allclose(f["A"], P["x"] @ P["w1"][0].T, rtol=1e-12, atol=1e-12)
    # Y_swi (Alg. 1 l.11), the activation MOE_CKPT_ABU saves: the MLP's hidden layer
    X = torch.from_numpy(P["x"])
    hid = F.silu(X @ torch.from_numpy(P["w1"][0]).T) * (X @ torch.from_numpy(P["w2"][0]).T)
    assert np.allclose(f["U"], hid.numpy(), rtol=1e-12, atol=1e-12)
    # and U W3 is the expert output: y = U W3 with the gate weight 1
    assert np.allclose(f["U"] @ P["w3"][0].T, ref, rtol=1e-12, atol=1e-12)


def test_identical_experts_with_renorm_is_mlp():
    P = _problem(E=4, k=2)
    for n in ("w1", "w2", "w3"):
        P[n] = np.repeat(P[n][:1], 4, axis=0)
    f = O.layer_forward(P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], 2, renormalize=True)
    ref = _mlp_torch(P["x"], P["w1"][0], P["w2"][0], P["w3"][0])
    assert np.allclose(f["y"], ref, rtol=1e-12, atol=1e-12)


def test_token_permutation_and_expert_relabel_invariance():
    P = _problem(T=30, E=5, k=2, seed=3)
    f = O.layer_forward(P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], 2)
    perm = np.random.default_rng(0).permutation(30)
    fp = O.layer_forward(P["x"][perm], P["w_gate"], P["w1"], P["w2"], P["w3"], 2)
    assert np.allclose(fp["y"], f["y"][perm], rtol=1e-12, atol=1e-12)
    assert np.array_equal(fp["ids"], f["ids"][perm])
    rel = np.array([3, 0, 4, 1, 2])
    fr = O.layer_forward(P["x"], P["w_gate"][rel], P["w1"][rel], P["w2"][rel], P["w3"][rel], 2)
    assert np.allclose(fr["y"], f["y"], rtol=1e-12, atol=1e-12)


def test_forward_dense_masked_formulation():
    """y = sum_e G[:,e] MLP_e(x) with G the top-k-masked softmax, dense
    over all experts (no dispatch structures at all)."""
    P = _problem(T=40, E=6, k=3, seed=5)
    f = O.layer_forward(P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], 3)
    y = _dense_masked_torch(P, 3, False)[0].detach().numpy()
    assert np.allclose(f["y"], y, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- backward
def _dense_masked_torch(P, k, renorm, req_grad=False):
    t = {n: torch.tensor(v, requires_grad=req_grad) for n, v in P.items() if n != "dy"}
    logits = t["x"] @ t["w_gate"].T
    p = torch.softmax(logits, dim=1)
    ids = torch.from_numpy(np.argsort(-logits.detach().numpy(), axis=1, kind="stable")[:, :k].copy())
    mask = torch.zeros_like(p).scatter_(1, ids, 1.0)
    G = p * mask
    if renorm:
        G = G / G.sum(1, keepdim=True)
    E = P["w1"].shape[0]
    y = 0
    for e in range(E):
        o = F.linear(F.silu(F.linear(t["x"], t["w1"][e])) * F.linear(t["x"], t["w2"][e]), t["w3"][e])
        y = y + G[:, e:e + 1] * o
    return y, t


@pytest.mark.parametrize("renorm", [False, True])
@pytest.mark.parametrize("T,d,h,E,k", [(24, 16, 24, 4, 2), (17, 8, 12, 6, 3), (10, 8, 8, 3, 1)])
def test_backward_vs_dense_masked_autograd(renorm, T, d, h, E, k):
    P = _problem(T, d, h, E, k, seed=T + E)
    fwd = O.layer_forward(P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], k, renormalize=renorm)
    bwd = O.layer_backward(fwd, P["dy"], P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], renormalize=renorm)
    y, t = _dense_masked_torch(P, k, renorm, req_grad=True)
    assert np.allclose(y.detach().numpy(), fwd["y"], rtol=1e-12, atol=1e-12)
    (y * torch.from_numpy(P["dy"])).sum().backward()
    for mine, ref in (("dx", "x"), ("dw1", "w1"), ("dw2", "w2"), ("dw3", "w3"), ("dw_gate", "w_gate")):
        g = t[ref].grad.numpy()
        err = np.abs(bwd[mine] - g).max() / max(np.abs(g).max(), 1e-6)  # k=1+renorm: grad is exactly 0
        assert err < 1e-10, (mine, err)


def test_gate_grad_equals_dy_dot_expert_output():
    """dg[t,j] = <dy_t, O_r> where O_r = U_r W3_e (the derivative of P:91 in g)."""
    P = _problem(T=20, E=4, k=2, seed=9)
    fwd = O.layer_forward(P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], 2)
    bwd = O.layer_backward(fwd, P["dy"], P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"])
    for t in range(20):
        for j in range(2):
            e = fwd["ids"][t, j]
            o = _mlp_torch(P["x"][t:t + 1], P["w1"][e], P["w2"][e], P["w3"][e])[0]
            assert abs(bwd["dg"][t, j] - P["dy"][t] @ o) < 1e-12 * (1 + abs(P["dy"][t] @ o))


@pytest.mark.parametrize("renorm", [False, True])
def test_backward_central_finite_differences(renorm):
    """Central FD in fp64, eps = 1e-6, loss = sum(y * dy); coordinates whose
    perturbation changes the routing are redrawn (top-k is piecewise constant)."""
    T, d, h, E, k = 12, 8, 12, 4, 2
    P = _problem(T, d, h, E, k, seed=11)
    fwd = O.layer_forward(P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], k, renormalize=renorm)
    bwd = O.layer_backward(fwd, P["dy"], P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], renormalize=renorm)
    rng = np.random.default_rng(0)
    eps = 1e-6

    def loss(Q):
        f = O.layer_forward(Q["x"], Q["w_gate"], Q["w1"], Q["w2"], Q["w3"], k, renormalize=renorm)
        return float(np.sum(f["y"] * P["dy"])), f["ids"]

    for name, gname in (("x", "dx"), ("w_gate", "dw_gate"), ("w1", "dw1"), ("w2", "dw2"), ("w3", "dw3")):
        checked = 0
        while checked < 12:
            idx = tuple(rng.integers(0, s) for s in P[name].shape)
            Q = {n: v.copy() for n, v in P.items()}
            Q[name][idx] += eps
            lp, idp = loss(Q)
            Q[name][idx] -= 2 * eps
            lm, idm = loss(Q)
            if not (np.array_equal(idp, fwd["ids"]) and np.array_equal(idm, fwd["ids"])):
                continue
            fd = (lp - lm) / (2 * eps)
            an = bwd[gname][idx]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (name, idx, fd, an)
            checked += 1


def test_silu_derivative_closed_form():
    """SiLU'(a) = sigma(a)(1 + a(1 - sigma(a))) (reading #15) vs torch autograd."""
    a = torch.linspace(-30, 30, 601, dtype=torch.float64, requires_grad=True)
    F.silu(a).sum().backward()
    s = O.sigmoid(a.detach().numpy())
    mine = s * (1 + a.detach().numpy() * (1 - s))
    assert np.allclose(mine, a.grad.numpy(), rtol=1e-14, atol=1e-15)
    assert np.allclose(O.silu(a.detach().numpy()), F.silu(a).detach().numpy(), rtol=1e-15, atol=1e-300)


# ---------------------------------------------------------------- memory formulas
def test_paper_memory_formulas():
    """Mem_routing = L*d*k*2 B ~ 94 GB for L~2M, k=4, d=6144 (the exact
    product is 98.3 GB = 91.6 GiB; reading #22).  P:85: Mem_act = 2*L*h ~ 98 GB
    for h = 24576 (bytes, bf16: L*h*2)."""
    L, k, d, h = 2e6, 4, 6144, 24576
    assert math.isclose(L * d * k * 2 / 1e9, 98.304)
    assert 90 < L * d * k * 2 / 2**30 < 95
    assert math.isclose(2 * L * h / 1e9, 98.304)


# ---------------------------------------------------------------- non-gated experts (NEXT-2)
@pytest.mark.parametrize("act", ["silu", "relu"])
def test_nongated_single_expert_is_textbook_mlp(act):
    """E = k = 1: y = W2 sigma(W1 x) via torch.nn.functional, fp64."""
    P = _problem(E=1, k=1)
    f = O.layer_forward(P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], 1, activation=act)
    x, w1, w3 = (torch.from_numpy(np.ascontiguousarray(a)) for a in (P["x"], P["w1"][0], P["w3"][0]))
    sig = F.silu if act == "silu" else F.relu
    ref = F.linear(sig(F.linear(x, w1)), w3).numpy()
    assert np.allclose(f["y"], ref, rtol=1e-12, atol=1e-12)
    assert f["B"] is None


@pytest.mark.parametrize("act", ["silu", "relu"])
@pytest.mark.parametrize("renorm", [False, True])
def test_nongated_backward_vs_dense_masked_autograd(act, renorm):
    T, d, h, E, k = 21, 12, 16, 5, 2
    P = _problem(T, d, h, E, k, seed=4)
    fwd = O.layer_forward(P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], k, renorm, activation=act)
    bwd = O.layer_backward(fwd, P["dy"], P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], renorm)
    t = {n: torch.tensor(v, requires_grad=True) for n, v in P.items() if n != "dy"}
    logits = t["x"] @ t["w_gate"].T
    p = torch.softmax(logits, 1)
    ids = torch.from_numpy(np.argsort(-logits.detach().numpy(), axis=1, kind="stable")[:, :k].copy())
    G = p * torch.zeros_like(p).scatter_(1, ids, 1.0)
    if renorm:
        G = G / G.sum(1, keepdim=True)
    sig = F.silu if act == "silu" else F.relu
    y = sum(G[:, e:e + 1] * F.linear(sig(F.linear(t["x"], t["w1"][e])), t["w3"][e]) for e in range(E))
    assert np.allclose(y.detach().numpy(), fwd["y"], rtol=1e-12, atol=1e-12)
    (y * torch.from_numpy(P["dy"])).sum().backward()
    for mine, ref in (("dx", "x"), ("dw1", "w1"), ("dw3", "w3"), ("dw_gate", "w_gate")):
        g = t[ref].grad.numpy()
        assert np.abs(bwd[mine] - g).max() / max(np.abs(g).max(), 1e-6) < 1e-10, (act, mine)
    assert bwd["dw2"] is None and np.abs(t["w2"].grad.numpy() if t["w2"].grad is not None else 0).max() == 0


def test_nongated_silu_finite_differences():
    T, d, h, E, k = 10, 6, 8, 3, 2
    P = _problem(T, d, h, E, k, seed=13)
    fwd = O.layer_forward(P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"], k, activation="silu")
    bwd = O.layer_backward(fwd, P["dy"], P["x"], P["w_gate"], P["w1"], P["w2"], P["w3"])
    rng = np.random.default_rng(3)
    eps = 1e-6
    for name, gname in (("x", "dx"), ("w1", "dw1"), ("w3", "dw3"), ("w_gate", "dw_gate")):
        done = 0
        while done < 8:
            idx = tuple(rng.integers(0, s) for s in P[name].shape)
            vals, idsl = [], []
            for sgn in (1, -1):
                Q = {n: v.copy() for n, v in P.items()}
                Q[name][idx] += sgn * eps
                f = O.layer_forward(Q["x"], Q["w_gate"], Q["w1"], Q["w2"], Q["w3"], k, activation="silu")
                vals.append(float(np.sum(f["y"] * P["dy"])))
                idsl.append(f["ids"])
            if not all(np.array_equal(i, fwd["ids"]) for i in idsl):
                continue
            fd = (vals[0] - vals[1]) / (2 * eps)
            assert abs(fd - bwd[gname][idx]) <= 1e-6 * max(1.0, abs(fd)), (name, idx)
            done += 1
