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

    def run(self, xs_h, dys_h, ys_h, dxs_h):
        """xs_h/dys_h: per-step pinned host inputs; ys_h/dxs_h: per-step pinned
        host outputs (lists of equal length).  Returns when all work is queued;
        the compute stream is made to wait for the last device->host copy."""
        comp = torch.cuda.current_stream(self.dev)
        n = len(xs_h)
        ev_in = [torch.cuda.Event() for _ in range(n)]
        ev_done = [torch.cuda.Event() for _ in range(n)]
        start = torch.cuda.Event()
        start.record(comp)

        def load(i):
            s = i % self.depth
            with torch.cuda.stream(self.h2d):
                self.h2d.wait_event(start)
                if i >= self.depth:  # buffer s was last read by step i - depth
                    self.h2d.wait_event(ev_done[i - self.depth])
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
            y, dx = self.step_fn(self.x[s], self.dy[s])
            ev_done[i].record(comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(ev_done[i])
                ys_h[i].copy_(y.detach(), non_blocking=True)
                dxs_h[i].copy_(dx.detach(), non_blocking=True)
                y.record_stream(self.d2h)
                dx.record_stream(self.d2h)
        comp.wait_stream(self.d2h)
