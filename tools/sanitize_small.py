"""Small bf16 layers for compute-sanitizer: ragged tails, h % 256 == 128, the d >= 3072
BWD_DH variant, k = 6; the three checkpoint policies through the staged autograd
backward; an expert-parallel receiver with fewer local experts than k (sparse slots)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2601_05296_b200 as M  # noqa: E402
from moe_inputs import make_inputs  # noqa: E402
from paper_2601_05296_b200.ep import CudaOps  # noqa: E402

for (T, d, h, E, k) in [(700, 256, 640, 8, 2), (300, 3072, 384, 4, 2), (500, 512, 256, 16, 6)]:
    inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=1, routing="skewed", device="cuda")
    x, wg, w1, w2, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
    logits, ids, w = M.route(x, wg, k)
    disp = M.dispatch_build(ids, E, dtype=x.dtype)
    y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp)
    g = M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits)
    for ck in ("ab", "abu", "none"):
        xl = x.clone().requires_grad_(True)
        ps = [t.clone().requires_grad_(True) for t in (wg, w1, w2, w3)]
        M.moe_layer(xl, *ps, k, False, ck).backward(dy)
    torch.cuda.synchronize()
    print("ok", T, d, h, E, k, float(y.float().abs().sum()))

# EP receiver: E = 1 local expert, k = 2 slots (one of them empty on most rows)
T, d, h, E, k = 400, 256, 384, 1, 2
inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=2, device="cuda")
g = np.random.default_rng(0)
ids = np.full((T, k), -1, np.int32)
ids[np.arange(T), g.integers(0, k, T)] = 0
n = int((ids >= 0).sum())
ids_t = torch.from_numpy(ids).cuda()
w = torch.rand(T, k, device="cuda") * (ids_t >= 0)
ops = CudaOps()
disp = ops.dispatch(ids_t, E, torch.bfloat16, rows=n)
y, a, b = ops.ffn_fwd(inp["x"], inp["w1"], inp["w2"], inp["w3"], w, disp, n)
ops.ffn_bwd(inp["dy"], inp["x"], inp["w1"], inp["w2"], inp["w3"], w, disp, a, b, n)
torch.cuda.synchronize()
print("ok ep receiver", n)
