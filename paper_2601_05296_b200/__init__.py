"""MoEBlaze (arXiv 2601.05296) hot path on B200 / sm_100a.

The MoE layer forward+backward runs in hand-written CUDA kernels behind the C
ABI of include/moeblaze.h (libmoeblaze.so, built in-tree).  This package is
the thin binding: argument marshalling, device-memory allocation via torch,
and expert-parallel orchestration over torch.distributed.  There is no CPU
fallback.
"""
from .layer import (Dispatch, MoEBlazeFunction, MoEBlazeLayer, dispatch_build, ffn_bwd, ffn_fwd, moe_layer,
                    route)
from . import _lib

__all__ = ["Dispatch", "MoEBlazeFunction", "MoEBlazeLayer", "dispatch_build", "ffn_bwd", "ffn_fwd", "moe_layer",
           "route", "_lib"]
