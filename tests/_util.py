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
