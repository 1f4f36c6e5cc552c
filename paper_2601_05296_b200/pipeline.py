"""Host-fed step pipelining: overlap host<->device copies with the MoE layer.

A training/serving loop that feeds each step from host memory pays the PCIe
transfers of its inputs and outputs.  HostPipeline runs steps with the
host->device copy of step i+1 and the device->host copy of step i on their own
CUDA streams, so they overlap step i's kernels on the compute stream (B200
has independent copy engines per direction).  Every step still moves all of
its bytes; only the serialisation is removed.
"""
from __future__ import annotations

import torch


class HostPipeline:
    """step_fn(x_dev, dy_dev) -> (y_dev, dx_dev), enqueued on the current stream.

    `depth` device input buffers rotate; step i+1's inputs are copied while
    step i computes (a buffer is reused only after the step that read it has
    finished).  Results are copied into the caller's pinned host buffers on a
    separate stream."""

    def __init__(self, step_fn, shape, dtype, device, depth=2):
        if depth < 2:
            # load(i + 1) reuses buffer (i + 1) % depth, last read by step i + 1 - depth: with
            # depth 1 that is step i itself, whose completion event is not recorded yet
            raise ValueError("HostPipeline needs depth >= 2 (step i+1's copy must not overwrite step i's inputs)")
        self.step_fn = step_fn
        self.depth = depth
        self.dev = torch.device(device)
        self.h2d = torch.cuda.Stream(self.dev)
        self.d2h = torch.cuda.Stream(self.dev)
        self.x = [torch.empty(shape, dtype=dtype, device=self.dev) for _ in range(depth)]
        self.dy = [torch.empty(shape, dtype=dtype, device=self.dev) for _ in range(depth)]

    def run(self, xs_h, dys_h, ys_h, dxs_h, trace=None):
        """xs_h/dys_h: per-step pinned host inputs; ys_h/dxs_h: per-step pinned
        host outputs (lists of equal length).  Returns when all work is queued;
        the compute stream is made to wait for the last device->host copy.
        trace: a list that receives, per step, timing events bracketing its
        host->device copy, its kernels and its device->host copy (diagnostics;
        read them with trace_summary after a synchronize)."""
        comp = torch.cuda.current_stream(self.dev)
        n = len(xs_h)
        timing = trace is not None
        ev_in = [torch.cuda.Event(enable_timing=timing) for _ in range(n)]
        ev_done = [torch.cuda.Event(enable_timing=timing) for _ in range(n)]
        mk = (lambda: torch.cuda.Event(enable_timing=True)) if timing else None
        marks = [dict(h2d0=mk(), comp0=mk(), d2h0=mk(), d2h1=mk()) for _ in range(n)] if timing else None
        start = torch.cuda.Event(enable_timing=timing)
        start.record(comp)
        if timing:
            trace.append(start)

        def load(i):
            s = i % self.depth
            with torch.cuda.stream(self.h2d):
                self.h2d.wait_event(start)
                if i >= self.depth:  # buffer s was last read by step i - depth
                    self.h2d.wait_event(ev_done[i - self.depth])
                if timing:
                    marks[i]["h2d0"].record(self.h2d)
                self.x[s].copy_(xs_h[i], non_blocking=True)
                self.dy[s].copy_(dys_h[i], non_blocking=True)
                ev_in[i].record(self.h2d)

        if n:
            load(0)
        for i in range(n):
            if i + 1 < n:
                load(i + 1)
            s = i % self.depth
            comp.wait_event(ev_in[i])
            if timing:
                marks[i]["comp0"].record(comp)
            y, dx = self.step_fn(self.x[s], self.dy[s])
            ev_done[i].record(comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(ev_done[i])
                if timing:
                    marks[i]["d2h0"].record(self.d2h)
                ys_h[i].copy_(y.detach(), non_blocking=True)
                dxs_h[i].copy_(dx.detach(), non_blocking=True)
                if timing:
                    marks[i]["d2h1"].record(self.d2h)
                y.record_stream(self.d2h)
                dx.record_stream(self.d2h)
        comp.wait_stream(self.d2h)
        if timing:
            for i in range(n):
                trace.append(dict(marks[i], h2d1=ev_in[i], comp1=ev_done[i]))


def trace_summary(trace):
    """Per-step medians (ms) of a run(trace=...) after synchronize: each leg's
    duration and how much of the copies overlapped the kernels of another step."""
    import statistics
    t0, steps = trace[0], trace[1:]

    def at(ev):
        return t0.elapsed_time(ev)

    rows = []
    for i, m in enumerate(steps):
        r = {k: at(m[k + "1"]) - at(m[k + "0"]) for k in ("h2d", "comp", "d2h")}
        # the kernels of step i run in [comp0_i, comp1_i]; a copy is hidden when it runs inside
        # some step's kernel window
        r["h2d_exposed"] = max(0.0, at(m["comp0"]) - at(steps[i - 1]["comp1"])) if i else 0.0
        rows.append(r)
    med = {k: round(statistics.median(r[k] for r in rows), 4) for k in rows[0]} if rows else {}
    med["gap_between_steps_ms_max"] = round(max((r["h2d_exposed"] for r in rows), default=0.0), 4)
    if steps:
        med["run_ms_per_step"] = round(at(steps[-1]["d2h1"]) / len(steps), 4)
    return med
