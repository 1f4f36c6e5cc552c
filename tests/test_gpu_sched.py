"""GPU: the die-aware dynamic tile scheduler of the expert GEMMs (gemm_tc.cu,
topology.cu).  The scheduler only changes which SM computes which output tile
(every tile is still computed exactly once, with the same k-order), so the
layer's results must be bit-identical with the die split on (default) and off
(MOEBLAZE_DIE=0).  k <= 2 keeps the red.add combine order-free (reading #12)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, json, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2601_05296_b200 as M
from moe_inputs import make_inputs
T, d, h, E, k = (int(v) for v in sys.argv[2].split(","))
inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=3, routing="skewed", device="cuda")
x, wg, w1, w2, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))
logits, ids, w = M.route(x, wg, k)
disp = M.dispatch_build(ids, E, dtype=x.dtype)
y, a, b = M.ffn_fwd(x, w1, w2, w3, w, disp)
A, B = a.clone(), b.clone()
g = M.ffn_bwd(dy, x, w1, w2, w3, w, disp, a, b, w_gate=wg, logits=logits)
torch.cuda.synchronize()
out = dict(y=y, A=A, B=B, dA=a, dB=b, **{n: v for n, v in g.items() if isinstance(v, torch.Tensor)})
dies, n = M._lib.sm_topology()
print(json.dumps({"n": n, "h": {name: hashlib.sha256(t.contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()
                                 for name, t in sorted(out.items())}}))
"""


def _run(shape, die_env):
    env = dict(os.environ)
    if die_env is not None:
        env["MOEBLAZE_DIE"] = die_env
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, shape], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-6000:] + r.stdout[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_topology_counts():
    import torch
    import paper_2601_05296_b200 as M
    dies, n = M._lib.sm_topology()
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    reached = [d for d in dies if d >= 0]
    if n[1] == 0:  # no split measured: the die-agnostic schedule
        assert n[0] == 0
        return
    assert n[0] + n[1] == len(reached) <= nsm
    assert n[0] == reached.count(0) and n[1] == reached.count(1)
    assert min(n) >= nsm // 4  # two dies of comparable size


@pytest.mark.parametrize("shape", ["3000,512,768,8,2", "5000,1024,1408,16,1", "4096,768,512,4,2"])
def test_die_split_is_bit_identical(shape):
    on = _run(shape, None)
    off = _run(shape, "0")
    assert off["n"][1] == 0
    assert on["h"] == off["h"]
