"""MoEBlaze oracle: plain, slow, obviously-correct fp64 CPU implementation.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import or call anything under
oracle/.  The product path (paper_2601_05296_b200) never imports it, and it
imports nothing from the product path: the two share no code.

What it computes: the standard dropless top-k SwiGLU MoE layer.  MoEBlaze
reaches exactly this result, only with less memory and traffic (P:25, P:101,
"without sacrificing accuracy"), so the oracle is that definition written
out, streaming expert by expert, in fp64 NumPy.  Citations are
/root/reference/PAPER.md line numbers ("P:n").

Readings of silent/garbled points:
  * gate = softmax over all E, then top-k, no renormalisation by
    default; renormalize=True is the Mixtral variant;
  * top-k is taken on the logits (softmax is monotone), descending, exact
    ties -> lower expert id; slot j = j-th largest;
  * inside an expert segment tokens are in ascending token id;
  * W1 = gate (SiLU) branch, W2 = up branch, W3 = down, stored
    nn.Linear style: w1[e], w2[e] are [h, d], w3[e] is [d, h];
  * Alg. 1's Z is X and its grad-Z is grad-X;
  * the gate-weight gradient and router backward are not in the paper
    (Alg. 1 returns only dW1..3, dZ); they are the analytic derivative of
    y = sum_i g_i(x) E_i(x) through softmax.

Every function here is pinned by a `-m "not gpu"` test (tests/test_oracle_*.py)
against something other than itself: the paper's worked example,
the paper's sort-based construction, brute force, closed forms, an
independent dense-masked torch autograd formulation and central finite
differences.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "softmax_rows", "topk_from_logits", "route", "dispatch_brute", "dispatch_argsort",
    "ffn_forward", "ffn_backward", "router_backward", "layer_forward", "layer_backward",
    "silu", "sigmoid", "ACTIVATIONS",
]

# FFN variants: the paper evaluates SwiGLU experts (§5,
# P:188-192) and non-gated experts E_i(x) = W2,i sigma(W1,i x) (§2.2) with
# sigma = SiLU or ReLU.  Non-gated experts use w1 (gate/
# first layer) and w3 (second layer); w2 is unused and B does not exist.
ACTIVATIONS = ("swiglu", "silu", "relu")


def sigmoid(a):
    """sigma(u) = 1/(1+exp(-u)), evaluated without overflow."""
    a = np.asarray(a, dtype=np.float64)
    out = np.empty_like(a)
    pos = a >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-a[pos]))
    ea = np.exp(a[~pos])
    out[~pos] = ea / (1.0 + ea)
    return out


def silu(a):
    """SiLU(u) = u * sigma(u)."""
    return a * sigmoid(a)


def softmax_rows(z):
    """Row-wise softmax, max-subtracted."""
    z = np.asarray(z, dtype=np.float64)
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    return e / e.sum(axis=1, keepdims=True)


def topk_from_logits(logits, k, renormalize=False):
    """topk_experts = TopK(softmax(W_g x)) given the logits.

    Selection on the logits (monotone with the softmax), descending, ties ->
    lower id (a stable sort of the negated logits keeps the lower index
    first).  Returns (probs [T,E], ids [T,k] int32, w [T,k]) where
    w[t,j] = p[t, ids[t,j]] is the gate score g_i(x) of P:91 (renormalised
    over the k chosen experts when renormalize=True).
    """
    logits = np.asarray(logits, dtype=np.float64)
    p = softmax_rows(logits)
    order = np.argsort(-logits, axis=1, kind="stable")
    ids = order[:, :k].astype(np.int32)
    w = np.take_along_axis(p, ids.astype(np.int64), axis=1)
    if renormalize:
        w = w / w.sum(axis=1, keepdims=True)
    return p, ids, w


def route(x, w_gate, k, renormalize=False):
    """Gating network: logits = x W_g^T, W_g in R^{E x d}, no bias."""
    x = np.asarray(x, dtype=np.float64)
    w_gate = np.asarray(w_gate, dtype=np.float64)
    logits = x @ w_gate.T
    p, ids, w = topk_from_logits(logits, k, renormalize)
    return dict(logits=logits, probs=p, ids=ids, w=w)


def dispatch_brute(ids, E):
    """The four index structures of §4.1, by their definitions.

    counts[e]  = #{(t,j): ids[t,j] = e}                        (expert_lengths)
    offs       = exclusive prefix sum, length E+1               (expert_token_offsets)
    eti        = for e = 0..E-1, tokens t routed to e, ascending (expert_token_indices)
    tim[t,j]   = position of (t, ids[t,j]) inside eti           (token_index_map)
    tei        = ids                                            (token_expert_indices)
    row_slot[r]= t*k + j for the (t, j) stored at eti position r (inverse of tim)
    Pure-Python loops: O(T*E), for small cases.
    """
    ids = np.asarray(ids)
    T, k = ids.shape
    counts = np.zeros(E, dtype=np.int64)
    for t in range(T):
        for j in range(k):
            counts[int(ids[t, j])] += 1
    offs = np.zeros(E + 1, dtype=np.int64)
    for e in range(E):
        offs[e + 1] = offs[e] + counts[e]
    eti = []
    tim = np.full((T, k), -1, dtype=np.int64)
    for e in range(E):
        for t in range(T):
            for j in range(k):
                if int(ids[t, j]) == e:
                    tim[t, j] = len(eti)
                    eti.append(t)
    eti = np.asarray(eti, dtype=np.int64)
    row_slot = np.empty(T * k, dtype=np.int64)
    for t in range(T):
        for j in range(k):
            row_slot[tim[t, j]] = t * k + j
    return dict(counts=counts.astype(np.int32), offs=offs.astype(np.int32), eti=eti.astype(np.int32),
                tim=tim.astype(np.int32), tei=ids.astype(np.int32), row_slot=row_slot.astype(np.int32))


def dispatch_argsort(ids, E):
    """The paper's sort-based construction: flatten the top-k choices
    to (expert, token) pairs, globally sort by expert id (stable => tokens
    ascending inside each expert), recover token ids and per-expert ranges."""
    ids = np.asarray(ids)
    T, k = ids.shape
    flat = ids.reshape(-1).astype(np.int64)
    order = np.argsort(flat, kind="stable")
    eti = (order // k).astype(np.int32)
    tim = np.empty(T * k, dtype=np.int64)
    tim[order] = np.arange(T * k)
    counts = np.bincount(flat, minlength=E).astype(np.int32)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    return dict(counts=counts, offs=offs, eti=eti, tim=tim.reshape(T, k).astype(np.int32),
                tei=ids.astype(np.int32), row_slot=order.astype(np.int32))


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def _act(a, activation):
    """sigma of the non-gated FFN: SiLU(u) = u sigma(u) or ReLU."""
    if activation == "silu":
        return silu(a)
    if activation == "relu":
        return np.maximum(a, 0.0)
    raise ValueError(activation)


def _act_grad(a, activation):
    """d sigma / d a: SiLU' = sigma(a)(1 + a(1 - sigma(a))); ReLU' = 1[a > 0]."""
    if activation == "silu":
        s = sigmoid(a)
        return s * (1.0 + a * (1.0 - s))
    if activation == "relu":
        return (a > 0).astype(np.float64)
    raise ValueError(activation)


def ffn_forward(x, w1, w2, w3, ids, w, disp, activation="swiglu"):
    """Expert computation + output aggregation, forward (Alg. 1
    FusedForward P:221-233, SwiGLU P:190-192, aggregation P:89-93).

    For every expert e and every row r of its segment (token t = eti[r],
    slot j with ids[t,j] = e):
        A_r = x_t W1_e,  B_r = x_t W2_e           (W1_e = w1[e]^T)
        U_r = SiLU(A_r) * B_r                      (Y_swi)
        O_r = U_r W3_e                             (W3_e = w3[e]^T)
        y_t += w[t,j] * O_r
    Returns y [T,d], the checkpointed pre-activations A, B [T*k, h] in
    expert-sorted row order and U (Alg. 1's Y_swi, the
    third tensor Alg. 1 l.11 stores) in the same order.
    Non-gated (activation = "silu" | "relu"): U_r = sigma(A_r), no B
    (returned as None), w2 unused.
    """
    gated = activation == "swiglu"
    x, w1, w3, w = _f64(x), _f64(w1), _f64(w3), _f64(w)
    w2 = _f64(w2) if gated else None
    T, d = x.shape
    E, h, _ = w1.shape
    k = ids.shape[1]
    offs, eti, row_slot = disp["offs"], disp["eti"], disp["row_slot"]
    R = T * k
    y = np.zeros((T, d))
    A = np.zeros((R, h))
    B = np.zeros((R, h)) if gated else None
    U = np.zeros((R, h))
    for e in range(E):
        lo, hi = int(offs[e]), int(offs[e + 1])
        if hi == lo:
            continue
        toks = eti[lo:hi].astype(np.int64)
        slots = row_slot[lo:hi].astype(np.int64)
        xe = x[toks]
        a = xe @ w1[e].T
        if gated:
            b = xe @ w2[e].T
            u = silu(a) * b
            B[lo:hi] = b
        else:
            u = _act(a, activation)
        o = u @ w3[e].T
        wr = w.reshape(-1)[slots]
        np.add.at(y, toks, wr[:, None] * o)
        A[lo:hi] = a
        U[lo:hi] = u
    return dict(y=y, A=A, B=B, U=U)


def ffn_backward(dy, x, w1, w2, w3, ids, w, disp, A, B, activation="swiglu"):
    """Expert backward (Alg. 1 FusedBackward P:236-253, §3.2), with
    the routing weight of P:91 carried through, plus the gate-weight gradient.

    For row r (expert e, token t, slot j), go_r = dy_t (gathered):
        dHu_r = go_r W3_e^T                          (Alg.1 l.20, before w)
        dg[t,j] = <dHu_r, U_r>  (= <dy_t, O_r>)      (gate-weight grad, not in paper)
        dW3_e  = sum_r (w U_r)^T go_r                 (Alg.1 l.18)
        dU_r   = w dHu_r
        S_r    = SiLU(A_r) recomputed                 (Alg.1 l.24)
        dA_r   = dU_r * B_r * SiLU'(A_r)             (Alg.1 l.26)
        dB_r   = dU_r * S_r                           (Alg.1 l.28)
        dW1_e  = sum_r x_t^T dA_r, dW2_e = sum_r x_t^T dB_r   (l.29 FusedBwdW)
        dx_t  += dA_r W1_e^T + dB_r W2_e^T            (l.30 FusedBwdX)
    SiLU'(a) = sigma(a) (1 + a (1 - sigma(a))).
    Returns dx [T,d], dw1, dw2 [E,h,d], dw3 [E,d,h], dg [T,k], dA, dB [R,h].
    Non-gated: U = sigma(A), dA = dU * sigma'(A); dw2, dB are None and
    dx_t += dA_r W1_e^T only.
    """
    gated = activation == "swiglu"
    dy, x, w1, w3, w = _f64(dy), _f64(x), _f64(w1), _f64(w3), _f64(w)
    w2 = _f64(w2) if gated else None
    A = _f64(A)
    B = _f64(B) if gated else None
    T, d = x.shape
    E, h, _ = w1.shape
    k = ids.shape[1]
    offs, eti, row_slot = disp["offs"], disp["eti"], disp["row_slot"]
    dx = np.zeros((T, d))
    dw1 = np.zeros_like(w1)
    dw2 = np.zeros_like(w2) if gated else None
    dw3 = np.zeros_like(w3)
    dg = np.zeros(T * k)
    dA = np.zeros_like(A)
    dB = np.zeros_like(B) if gated else None
    for e in range(E):
        lo, hi = int(offs[e]), int(offs[e + 1])
        if hi == lo:
            continue
        toks = eti[lo:hi].astype(np.int64)
        slots = row_slot[lo:hi].astype(np.int64)
        wr = w.reshape(-1)[slots][:, None]
        a = A[lo:hi]
        if gated:
            b = B[lo:hi]
            sg = sigmoid(a)
            s = a * sg
            u = s * b
        else:
            u = _act(a, activation)
        go = dy[toks]
        dhu = go @ w3[e]                      # [n, h]  (w3[e] is [d, h])
        dg[slots] = np.sum(dhu * u, axis=1)
        dw3[e] = go.T @ (wr * u)              # [d, h]
        du = wr * dhu
        xe = x[toks]
        if gated:
            da = du * b * sg * (1.0 + a * (1.0 - sg))
            db = du * s
            dw2[e] = db.T @ xe
            dB[lo:hi] = db
            np.add.at(dx, toks, da @ w1[e] + db @ w2[e])
        else:
            da = du * _act_grad(a, activation)
            np.add.at(dx, toks, da @ w1[e])
        dw1[e] = da.T @ xe                    # [h, d]
        dA[lo:hi] = da
    return dict(dx=dx, dw1=dw1, dw2=dw2, dw3=dw3, dg=dg.reshape(T, k), dA=dA, dB=dB)


def router_backward(dg, x, w_gate, logits, ids, renormalize=False):
    """Backward of w = TopK-gather(softmax(x W_g^T)).

    dsel = dg                                   (no renorm)
    dsel_j = (dg_j - sum_i dg_i w_i) / sum_i p_sel_i   (renorm: w = p_sel / sum p_sel)
    dp[t, ids[t,j]] = dsel[t,j];  dlogits = p * (dp - <p, dp>)
    dW_g = dlogits^T x;  dx_router = dlogits W_g
    """
    dg, x, w_gate, logits = _f64(dg), _f64(x), _f64(w_gate), _f64(logits)
    T, k = dg.shape
    p = softmax_rows(logits)
    psel = np.take_along_axis(p, ids.astype(np.int64), axis=1)
    if renormalize:
        ssum = psel.sum(axis=1, keepdims=True)
        wsel = psel / ssum
        dsel = (dg - np.sum(dg * wsel, axis=1, keepdims=True)) / ssum
    else:
        dsel = dg
    dp = np.zeros_like(p)
    for j in range(k):
        dp[np.arange(T), ids[:, j].astype(np.int64)] += dsel[:, j]
    dlogits = p * (dp - np.sum(p * dp, axis=1, keepdims=True))
    return dict(dlogits=dlogits, dw_gate=dlogits.T @ x, dx=dlogits @ w_gate)


def layer_forward(x, w_gate, w1, w2, w3, k, renormalize=False, logits=None, dispatch="argsort", activation="swiglu"):
    """Whole layer forward.  `logits` given => forced routing on those logits
    (used with the GPU's fp32 logits so near-ties resolve identically)."""
    if logits is None:
        r = route(x, w_gate, k, renormalize)
    else:
        p, ids, w = topk_from_logits(logits, k, renormalize)
        r = dict(logits=_f64(logits), probs=p, ids=ids, w=w)
    E = _f64(w_gate).shape[0]
    disp = (dispatch_brute if dispatch == "brute" else dispatch_argsort)(r["ids"], E)
    f = ffn_forward(x, w1, w2, w3, r["ids"], r["w"], disp, activation)
    return dict(**r, disp=disp, activation=activation, **f)


def layer_backward(fwd, dy, x, w_gate, w1, w2, w3, renormalize=False):
    """Whole layer backward: expert part + router part; dx includes both."""
    b = ffn_backward(dy, x, w1, w2, w3, fwd["ids"], fwd["w"], fwd["disp"], fwd["A"], fwd["B"],
                     fwd.get("activation", "swiglu"))
    rb = router_backward(b["dg"], x, w_gate, fwd["logits"], fwd["ids"], renormalize)
    out = dict(b)
    out["dx_ffn"] = b["dx"]
    out["dx"] = b["dx"] + rb["dx"]
    out["dw_gate"] = rb["dw_gate"]
    out["dlogits"] = rb["dlogits"]
    return out
