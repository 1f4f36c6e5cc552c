#!/usr/bin/env python
"""bench_sweep.py — BASELINE.json configs[3]: sequence-length / batch sweep
T = 4K..128K at d = 4096, h = 16384 (4d, Table 1 rule P:259), E = 16, top-2,
reporting fwd+bwd tokens/s and activation memory (saved-tensor hooks)
next to the materialise-everything PyTorch baseline.

    python bench_sweep.py [--T 4096 8192 ...] [--steps 3] [--no-baseline]

One JSON line per T, then a summary line.  The paper's claim checked here:
activation savings "scale proportionally with the sequence length L"
 — the saved-bytes gap grows linearly in T.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, nargs="*", default=None)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--no-baseline", action="store_true")
    a = ap.parse_args()
    import torch
    import bench
    from moe_inputs import CONFIGS, SWEEP_T, make_inputs
    from paper_2601_05296_b200 import build as B
    B.build()
    import paper_2601_05296_b200 as M

    dev = torch.device("cuda", 0)
    rows = []
    for T in (a.T or SWEEP_T):
        cfg = CONFIGS[f"sweep_{T // 1024}k"]
        inp = make_inputs(cfg.T, cfg.d, cfg.h, cfg.E, cfg.k, dtype="bf16", seed=0, device=dev)
        x, wg, w1, w2, w3, dy = (inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy"))

        def step():
            logits, ids, w = M.route(x, wg, cfg.k)
            disp = M.dispatch_build(ids, cfg.E)
            y, A, Bs = M.ffn_fwd(x, w1, w2, w3, w, disp)
            return M.ffn_bwd(dy, x, w1, w2, w3, w, disp, A, Bs, w_gate=wg, logits=logits)

        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        mem = bench.measure_memory(M, x, wg, w1, w2, w3, dy, cfg.k, False) if not a.no_baseline else None
        row = {"workload": cfg.name, "T": T, "d": cfg.d, "h": cfg.h, "E": cfg.E, "k": cfg.k,
               "tokens_per_s": round(T / (ms / 1e3), 1), "ms_per_step": round(ms, 3),
               "tflops": round(18 * T * cfg.k * cfg.d * cfg.h / (ms / 1e3) / 1e12, 1), "memory": mem}
        print(json.dumps(row), flush=True)
        rows.append(row)
        del inp, x, wg, w1, w2, w3, dy
        torch.cuda.empty_cache()
    if rows and rows[0]["memory"] and "saved_gb" in rows[0]["memory"].get("materialized_baseline", {}):
        gaps = [(r["T"], r["memory"]["materialized_baseline"]["saved_gb"] - r["memory"]["ours"]["saved_gb"]) for r in rows]
        per_tok = [g / t * 1e9 for t, g in gaps]
        print(json.dumps({"summary": "saved-activation gap (materialised - ours) per token, bytes",
                          "per_token_bytes": [round(p, 1) for p in per_tok],
                          "ratios": [r["memory"].get("saved_ratio") for r in rows]}), flush=True)


if __name__ == "__main__":
    main()
