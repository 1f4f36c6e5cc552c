"""One small bf16 layer fwd+bwd (ragged tails, h % 256 == 128, d >= 3072 variant) for compute-sanitizer."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2601_05296_b200 as M
from moe_inputs import make_inputs
for (T, d, h, E, k) in [(700, 256, 640, 8, 2), (300, 3072, 384, 4, 2), (500, 512, 256, 16, 6)]:
    inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=1, routing="skewed", device="cuda")
    x, wg, w1, w2, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
    logits, ids, w = M.route(x, wg, k)
    disp = M.dispatch_build(ids, E, dtype=x.dtype)
    y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp)
    g = M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits)
    torch.cuda.synchronize()
    print("ok", T, d, h, E, k, float(y.float().abs().sum()))
