"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the MoEBlaze method (no routing, no
dispatch, no FFN): it only draws random tensors with the shapes and value
distributions of the paper's workloads and rounds them to the run dtype.
Both `oracle/` (via the tests / bench) and the CUDA path consume exactly the
same values; the oracle upcasts them exactly to fp64.

Recipe (DESIGN.md §"Input recipe"):
  X  ~ N(0,1)                [T, d]
  Wg ~ N(0,1)/sqrt(d)        [E, d]      -> logits ~ N(0,1)
  W1, W2 ~ N(0,1)/sqrt(d)    [E, h, d]   (nn.Linear (out, in) layout; paper's W1 = w1[e]^T)
  W3 ~ N(0,1)/sqrt(h)        [E, d, h]
  dY ~ N(0,1)                [T, d]
The paper's workloads are synthetic single-layer shapes (Table 1);
it states no value distribution, so unit-variance activations are our choice.

Routing structure:
  balanced   - iid logits (multinomial expert loads), the headline case;
  skewed     - X += u, Wg[e] -= alpha*ln(1+e)*u/|u|^2  => Zipf-like per-expert logit bias;
  degenerate - every token picks experts 0..k-1 (E>k leaves experts empty).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, asdict

import torch

__all__ = ["MoEConfig", "CONFIGS", "make_inputs", "make_ids", "SWEEP_T"]


@dataclass(frozen=True)
class MoEConfig:
    name: str
    T: int          # tokens (paper: L)
    d: int          # model dim
    h: int          # FFN hidden dim (d_ff)
    E: int          # experts
    k: int          # top-k
    dtype: str      # "bf16" | "fp32"

    def as_dict(self):
        return asdict(self)

    @property
    def R(self):
        return self.T * self.k


SWEEP_T = (4096, 8192, 16384, 32768, 65536, 131072)

# BASELINE.json "configs" (index order kept), plus the sweep points.
CONFIGS = {
    "tiny": MoEConfig("tiny", 256, 64, 128, 4, 2, "fp32"),
    "mixtral": MoEConfig("mixtral", 8192, 4096, 14336, 8, 2, "bf16"),
    "deepseek": MoEConfig("deepseek", 16384, 2048, 1408, 64, 6, "bf16"),
    "ep": MoEConfig("ep", 32768, 4096, 2048, 64, 8, "bf16"),
}
for _t in SWEEP_T:
    CONFIGS[f"sweep_{_t // 1024}k"] = MoEConfig(f"sweep_{_t // 1024}k", _t, 4096, 16384, 16, 2, "bf16")


def _torch_dtype(dtype: str):
    return {"bf16": torch.bfloat16, "fp32": torch.float32}[dtype]


def make_inputs(T, d, h, E, k, dtype="bf16", seed=0, routing="balanced", alpha=0.25,
                device="cpu", with_dy=True):
    """Draw one problem instance. Returns a dict of tensors in the run dtype.

    Values are drawn in fp32 from a seeded torch generator on `device`, scaled,
    then rounded (RNE) to the run dtype.  Same (seed, device) => same values.
    """
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    f32 = dict(dtype=torch.float32, device=device, generator=g)
    td = _torch_dtype(dtype)
    x = torch.randn(T, d, **f32)
    wg = torch.randn(E, d, **f32) / math.sqrt(d)
    w1 = torch.randn(E, h, d, **f32).mul_(1.0 / math.sqrt(d)).to(td)
    w2 = torch.randn(E, h, d, **f32).mul_(1.0 / math.sqrt(d)).to(td)
    w3 = torch.randn(E, d, h, **f32).mul_(1.0 / math.sqrt(h)).to(td)
    dy = torch.randn(T, d, **f32) if with_dy else None
    if routing == "skewed":
        u = torch.randn(d, **f32)
        x += u
        bias = alpha * torch.log1p(torch.arange(E, dtype=torch.float32, device=device))
        wg -= bias[:, None] * (u / (u * u).sum())[None, :]
    elif routing == "degenerate":
        if E > 1:
            x[:, 0] = x[:, 0].abs() + 1.0
            wg[:, 1:] *= 0.1
            e = torch.arange(E, dtype=torch.float32, device=device)
            wg[:, 0] = torch.where(e < k, 4.0 + 0.5 * (k - e), torch.full_like(e, -4.0))
    elif routing != "balanced":
        raise ValueError(routing)
    out = dict(x=x.to(td), w_gate=wg.to(td), w1=w1, w2=w2, w3=w3)
    if with_dy:
        out["dy"] = dy.to(td)
    return out


def make_ids(T, E, k, seed=0, kind="random", alpha=1.0):
    """Random routing decisions [T, k] int32 (distinct experts per token) for
    dispatch-only tests.  kind: random | skewed | degenerate | all_same_first."""
    g = torch.Generator().manual_seed(int(seed))
    if kind == "degenerate":
        return torch.arange(k, dtype=torch.int32).repeat(T, 1)
    if kind == "random":
        scores = torch.rand(T, E, generator=g)
    elif kind == "skewed":
        scores = torch.rand(T, E, generator=g).log() - alpha * torch.log1p(torch.arange(E, dtype=torch.float32))
    else:
        raise ValueError(kind)
    # a random permutation per token, first k entries: distinct ids
    return torch.argsort(scores, dim=1, descending=True)[:, :k].to(torch.int32).contiguous()
