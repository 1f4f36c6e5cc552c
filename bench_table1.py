#!/usr/bin/env python
"""bench_table1.py — the paper's own experiment grid.

Table 1: conf1..conf7 (d, E, k, batch, seq; h = 4d), single MoE
layer, fwd+bwd excluding the optimizer, activation memory by
saved-tensor hooks, for SwiGLU experts (§6.5-6.6) and non-gated SiLU
experts (§6.3-6.4).  The paper compares against Megablocks on an H100; here
the comparator is the in-repo materialise-everything PyTorch baseline
(materialized_baseline.py: argsort dispatch, routed-token buffer, torch
grouped_mm) on the same B200.  One JSON line per (conf, activation).

    python bench_table1.py [--confs conf1 conf4] [--acts swiglu silu] [--steps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TABLE1 = {  # name: (d, E, k, batch, seq) — P:261-269
    "conf1": (512, 4, 1, 32, 2048), "conf2": (1024, 8, 2, 32, 2048), "conf3": (1024, 16, 4, 32, 2048),
    "conf4": (2048, 16, 4, 32, 1024), "conf5": (512, 16, 4, 32, 1024), "conf6": (1024, 16, 4, 16, 1024),
    "conf7": (2048, 8, 4, 16, 512),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--confs", nargs="*", default=list(TABLE1))
    ap.add_argument("--acts", nargs="*", default=["swiglu", "silu"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import torch
    from materialized_baseline import materialized_moe
    from moe_inputs import make_inputs
    from paper_2601_05296_b200 import build as B
    B.build()
    import paper_2601_05296_b200 as M

    dev = torch.device("cuda", 0)
    for name in a.confs:
        d, E, k, bs, seq = TABLE1[name]
        T, h = bs * seq, 4 * d
        inp = make_inputs(T, d, h, E, k, dtype="bf16", seed=0, device=dev)
        for act in a.acts:
            params = [torch.nn.Parameter(inp[n].clone()) for n in ("w_gate", "w1", "w2", "w3")]

            def run(fn):
                xl = inp["x"].detach().clone().requires_grad_(True)
                for p in params:
                    p.grad = None
                y = fn(xl, *params)
                y.backward(inp["dy"])

            ours = lambda xx, g_, w1, w2, w3: M.moe_layer(xx, g_, w1, w2, w3, k, False, "ab", act)  # noqa: E731
            base = lambda xx, g_, w1, w2, w3: materialized_moe(xx, g_, w1, w2, w3, k, False, act)  # noqa: E731
            row = {"conf": name, "activation": act, "T": T, "d": d, "h": h, "E": E, "k": k}
            for tag, fn in (("moeblaze", ours), ("materialized", base)):
                try:
                    for _ in range(a.warmup):
                        run(fn)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.steps):
                        run(fn)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / a.steps
                    saved = {}

                    def pack(t):
                        s = t.untyped_storage()
                        if s.data_ptr() not in {p.untyped_storage().data_ptr() for p in params}:
                            saved[s.data_ptr()] = s.nbytes()
                        return t

                    xl = inp["x"].detach().clone().requires_grad_(True)
                    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
                        y = fn(xl, *params)
                    del y
                    # peak of one fwd+bwd (max_memory_allocated delta), minus the parameter gradients
                    for p in params:
                        p.grad = None
                    torch.cuda.synchronize()
                    base_b = torch.cuda.memory_allocated()
                    torch.cuda.reset_peak_memory_stats()
                    run(fn)
                    torch.cuda.synchronize()
                    peak = torch.cuda.max_memory_allocated() - base_b
                    grads = sum(p.grad.numel() * p.grad.element_size() for p in params if p.grad is not None)
                    row[tag] = {"ms": round(ms, 3), "tokens_per_s": round(T / (ms / 1e3), 1),
                                "saved_gb": round(sum(saved.values()) / 1e9, 4), "peak_gb": round(peak / 1e9, 4),
                                "activation_peak_gb": round((peak - grads) / 1e9, 4)}
                except Exception as exc:  # report, never fake
                    row[tag] = {"error": repr(exc)[:200]}
            if "ms" in row.get("moeblaze", {}) and "ms" in row.get("materialized", {}):
                row["speedup"] = round(row["materialized"]["ms"] / row["moeblaze"]["ms"], 3)
                row["memory_ratio"] = round(row["materialized"]["saved_gb"] / row["moeblaze"]["saved_gb"], 3)
                row["peak_ratio"] = round(row["materialized"]["peak_gb"] / row["moeblaze"]["peak_gb"], 3)
            print(json.dumps(row), flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
