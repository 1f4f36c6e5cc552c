"""Shared test helpers (comparators, oracle wiring).  Test infrastructure."""
import numpy as np
import torch

BF16_TOL = 2e-2   # BASELINE.json north_star: bf16 max-relative-error 2e-2
FP32_TOL = 1e-4   # fp32 mode 1e-4


def normwise(gpu, ref):
    """max|gpu - ref| / max|ref| (reading #18: normwise infinity relative error)."""
    g = gpu.detach().double().cpu().numpy() if isinstance(gpu, torch.Tensor) else np.asarray(gpu, np.float64)
    r = np.asarray(ref, np.float64)
    den = np.abs(r).max() if r.size else 0.0
    if den == 0.0:
        return float(np.abs(g).max()) if g.size else 0.0
    return float(np.abs(g - r).max() / den)


def f64(t):
    return t.detach().double().cpu().numpy()


def i64(t):
    return t.detach().cpu().numpy().astype(np.int64)


def dispatch_sparse(ids, E):
    """Test-only: the index structures of §4.1 over the non-empty slots (ids >= 0)
    of a sparse-slot problem, by a stable argsort -- the definition the
    C ABI states for p.rows > 0 (empty slots: token_index_map = -1)."""
    T, k = ids.shape
    flat = ids.reshape(-1).astype(np.int64)
    valid = flat >= 0
    n = int(valid.sum())
    order = np.argsort(np.where(valid, flat, E), kind="stable")[:n]
    counts = np.bincount(flat[valid], minlength=E)
    offs = np.concatenate([[0], np.cumsum(counts)])
    tim = np.full(T * k, -1, dtype=np.int64)
    tim[order] = np.arange(n)
    return dict(counts=counts, offs=offs, eti=order // k, tim=tim.reshape(T, k), row_slot=order, tei=ids)
