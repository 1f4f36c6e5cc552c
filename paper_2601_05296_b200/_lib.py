"""ctypes binding of libmoeblaze.so (the C ABI in include/moeblaze.h).

Argument marshalling only: every step of the MoE layer runs in the library's
CUDA kernels.  Torch is used for device memory (the caller-owned buffers and
the scratch workspace) and for the current CUDA stream.  There is no CPU or
PyTorch fallback: if the library cannot be loaded, or a call fails, this
module raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# MOEBLAZE_LIB: an alternative in-tree build of the same library (compile-time
# tuning variants, tools/tune_*.sh); never a different implementation
LIB_PATH = os.environ.get("MOEBLAZE_LIB") or os.path.join(_PKG, "libmoeblaze.so")

MOE_BF16, MOE_FP32 = 0, 1
MOE_OP_ROUTE, MOE_OP_DISPATCH, MOE_OP_FFN_FWD, MOE_OP_FFN_BWD, MOE_OP_ROUTER_BWD = 0, 1, 2, 3, 4

EXPORTS = ("moe_workspace_size", "moe_route", "moe_dispatch_build", "moe_ffn_fwd", "moe_ffn_bwd",
           "moe_gather_rows", "moe_combine_rows", "moe_status_string", "moe_launch_count", "moe_version",
           "moe_profile_enable", "moe_profile_reset", "moe_profile_read", "moe_router_backward", "moe_ep_dest",
           "moe_ep_send_meta", "moe_ep_slot_grad", "moe_ep_local_slots", "moe_sm_topology", "moe_ep_signal",
           "moe_ep_wait", "moe_ep_publish_counts", "moe_ep_push_rows", "moe_ep_recv_prepare", "moe_ep_pull_combine",
           "moe_ep_pull_slot_grad", "moe_ep_pull_sum", "moe_ep_ipc_handle", "moe_ep_ipc_open", "moe_ep_ipc_close",
           "moe_profile_read_named", "moe_ffn_fwd_ex", "moe_dispatch_row_split")
GEMM_KINDS = ("FWD_UP", "FWD_DOWN", "BWD_DH", "BWD_DX", "DW3", "DW12")


class MoeProblem(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int64), ("d", ctypes.c_int32), ("h", ctypes.c_int32), ("E", ctypes.c_int32),
                ("k", ctypes.c_int32), ("dtype", ctypes.c_int32), ("renormalize", ctypes.c_int32),
                ("check_routing", ctypes.c_int32), ("checkpoint", ctypes.c_int32), ("activation", ctypes.c_int32),
                ("deterministic", ctypes.c_int32), ("rows", ctypes.c_int64)]


class MoeDispatch(ctypes.Structure):
    _fields_ = [("expert_counts", ctypes.c_void_p), ("expert_offsets", ctypes.c_void_p),
                ("expert_token_indices", ctypes.c_void_p), ("token_index_map", ctypes.c_void_p),
                ("row_slot", ctypes.c_void_p), ("token_expert_indices", ctypes.c_void_p),
                ("token_rows", ctypes.c_void_p)]


class MoeBwdSync(ctypes.Structure):
    _fields_ = [("x_ready", ctypes.c_void_p), ("dx_ready", ctypes.c_void_p), ("stages", ctypes.c_int32)]


MOE_BWD_DATA, MOE_BWD_DW3, MOE_BWD_DW12, MOE_BWD_ALL = 1, 2, 4, 7


class MoeFwdSync(ctypes.Structure):
    _fields_ = [("row_split", ctypes.c_void_p), ("x_ready", ctypes.c_void_p), ("y_ready", ctypes.c_void_p),
                ("t_ready", ctypes.c_int64), ("sm_reserve", ctypes.c_int32)]


class MoeRouterBwd(ctypes.Structure):
    _fields_ = [("w_gate", ctypes.c_void_p), ("logits", ctypes.c_void_p), ("topk_ids", ctypes.c_void_p),
                ("dw_gate", ctypes.c_void_p)]


# peer-memory exchange phases (moeblaze.h "Device-initiated expert-parallel exchange")
(MOE_EP_PH_ENTER, MOE_EP_PH_COUNTS, MOE_EP_PH_ROWS, MOE_EP_PH_Y, MOE_EP_PH_DY, MOE_EP_PH_DX, MOE_EP_PH_DWG,
 MOE_EP_NPHASE) = range(8)


class MoeEpPeers(ctypes.Structure):
    _fields_ = [("n_ranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("peer_flags", ctypes.c_void_p),
                ("peer_cmat", ctypes.c_void_p), ("arrive", ctypes.c_void_p), ("status", ctypes.c_void_p),
                ("timeout_ns", ctypes.c_int64)]


class MoEError(RuntimeError):
    pass


_lib = None


def load():
    """Load the shared library (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with `python -m paper_2601_05296_b200.build` "
                          "(there is no CPU/PyTorch fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, V, I32, I64, SZ = ctypes.POINTER, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    lib.moe_workspace_size.argtypes = [P(MoeProblem), I32, P(SZ)]
    lib.moe_route.argtypes = [P(MoeProblem), V, V, V, V, V, V, SZ, V]
    lib.moe_dispatch_build.argtypes = [P(MoeProblem), V, P(MoeDispatch), V, SZ, V]
    lib.moe_ffn_fwd.argtypes = [P(MoeProblem), V, V, V, V, V, P(MoeDispatch), V, V, V, V, V, SZ, V]
    lib.moe_ffn_bwd.argtypes = [P(MoeProblem), V, V, V, V, V, V, P(MoeDispatch), V, V, V, V, V, V, V, V,
                                P(MoeRouterBwd), P(MoeBwdSync), V, SZ, V]
    lib.moe_gather_rows.argtypes = [V, I64, V, I64, I64, I32, V, V]
    lib.moe_combine_rows.argtypes = [P(MoeProblem), V, V, V, V, V]
    lib.moe_router_backward.argtypes = [P(MoeProblem), V, V, P(MoeRouterBwd), V, V, V, SZ, V]
    lib.moe_ep_dest.argtypes = [P(MoeProblem), V, I32, I32, I32, V, V]
    lib.moe_ep_local_slots.argtypes = [P(MoeProblem), V, V, I32, I32, V, V, V]
    lib.moe_ep_send_meta.argtypes = [P(MoeProblem), V, V, I32, I32, V, I64, V, V, V]
    lib.moe_ep_slot_grad.argtypes = [P(MoeProblem), V, I32, I32, V, V, V, I32, V, V]
    lib.moe_sm_topology.argtypes = [P(I32), I32, P(I32)]
    U64, G = ctypes.c_uint64, P(MoeEpPeers)
    lib.moe_ep_signal.argtypes = [G, I32, U64, V]
    lib.moe_ep_wait.argtypes = [G, I32, U64, V]
    lib.moe_ep_publish_counts.argtypes = [G, V, U64, V]
    lib.moe_ep_push_rows.argtypes = [G, V, V, V, I64, I64, I64, V, I32, U64, V]
    lib.moe_ep_recv_prepare.argtypes = [G, I64, I64, I32, I32, V, V, V, V]
    lib.moe_ep_pull_combine.argtypes = [G, P(MoeProblem), V, I64, V, V, V, V, V]
    lib.moe_ep_pull_slot_grad.argtypes = [G, P(MoeProblem), I32, V, V, I64, V, V, V, V, V]
    lib.moe_ep_pull_sum.argtypes = [G, V, I64, I32, V, V]
    lib.moe_ep_ipc_handle.argtypes = [V, V, P(I64)]
    lib.moe_ep_ipc_open.argtypes = [V, I64, P(V), P(V)]
    lib.moe_ep_ipc_close.argtypes = [V]
    lib.moe_profile_read_named.argtypes = [ctypes.c_char_p, P(ctypes.c_double), P(I64)]
    lib.moe_ffn_fwd_ex.argtypes = [P(MoeProblem), V, V, V, V, V, P(MoeDispatch), V, V, V, V, P(MoeFwdSync), V, SZ, V]
    lib.moe_dispatch_row_split.argtypes = [P(MoeProblem), P(MoeDispatch), I64, V, V]
    lib.moe_sm_topology.restype = I32
    for fn in ("moe_workspace_size", "moe_route", "moe_dispatch_build", "moe_ffn_fwd", "moe_ffn_bwd",
               "moe_gather_rows", "moe_combine_rows", "moe_router_backward", "moe_ep_dest", "moe_ep_send_meta",
               "moe_ep_slot_grad", "moe_ep_local_slots"):
        getattr(lib, fn).restype = I32
    lib.moe_status_string.argtypes = [I32]
    lib.moe_status_string.restype = ctypes.c_char_p
    lib.moe_launch_count.restype = ctypes.c_uint64
    lib.moe_version.restype = I32
    lib.moe_profile_enable.argtypes = [I32]
    lib.moe_profile_read.argtypes = [I32, P(ctypes.c_double), P(I64)]
    for fn in ("moe_profile_enable", "moe_profile_reset", "moe_profile_read", "moe_router_backward", "moe_ep_dest",
               "moe_ep_send_meta", "moe_ep_slot_grad") + EXPORTS[EXPORTS.index("moe_ep_signal"):]:
        getattr(lib, fn).restype = I32
    _lib = lib
    if torch.cuda.is_available():
        # measure the SM -> die map now (synchronous, ~ms): a first GEMM call inside a
        # CUDA-graph capture must not have to run the probe
        d = (ctypes.c_int32 * 256)()
        n = (ctypes.c_int32 * 2)()
        lib.moe_sm_topology(d, 256, n)
    return lib


def sm_topology(max_sm=256):
    """(die of each SM id (-1 = not reached), SMs per die) as measured by the
    library for the expert GEMMs' tile scheduler (moe_sm_topology)."""
    lib = load()
    dies = (ctypes.c_int32 * max_sm)()
    n = (ctypes.c_int32 * 2)()
    _check(lib.moe_sm_topology(dies, max_sm, n), "moe_sm_topology")
    return list(dies), [n[0], n[1]]


def _check(status, what):
    if status != 0:
        msg = load().moe_status_string(status).decode()
        raise MoEError(f"{what}: {msg} (status {status})")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dtype_code(dt):
    if dt == torch.bfloat16:
        return MOE_BF16
    if dt == torch.float32:
        return MOE_FP32
    raise MoEError(f"unsupported dtype {dt} (bf16 or fp32)")


MOE_CKPT_AB, MOE_CKPT_NONE, MOE_CKPT_ABU = 0, 1, 2
CHECKPOINT = {"ab": MOE_CKPT_AB, "none": MOE_CKPT_NONE, "abu": MOE_CKPT_ABU}


ACTIVATION = {"swiglu": 0, "silu": 1, "relu": 2}


def problem(T, d, h, E, k, dtype, renormalize=False, check_routing=False, checkpoint="ab", activation="swiglu",
            deterministic=False, rows=0):
    """rows > 0: sparse slots (topk_ids -1 = empty slot), R = rows routed rows."""
    return MoeProblem(int(T), int(d), int(h), int(E), int(k), _dtype_code(dtype), int(bool(renormalize)),
                      int(bool(check_routing)), CHECKPOINT[checkpoint], ACTIVATION[activation], int(bool(deterministic)),
                      int(rows))


def workspace_size(p, op):
    n = ctypes.c_size_t(0)
    _check(load().moe_workspace_size(ctypes.byref(p), op, ctypes.byref(n)), "moe_workspace_size")
    return n.value


def workspace(p, op, device):
    n = workspace_size(p, op)
    return torch.empty(max(n, 256), dtype=torch.uint8, device=device)


def launch_count():
    return int(load().moe_launch_count())


# ----------------------------------------------------------------- entry points (same names as the C ABI)
def moe_route(p, x, w_gate, logits, topk_ids, topk_w, stream=None):
    _check(load().moe_route(ctypes.byref(p), _ptr(x), _ptr(w_gate), _ptr(logits), _ptr(topk_ids), _ptr(topk_w),
                            None, 0, _stream(stream)), "moe_route")


def make_dispatch(counts, offs, eti, tim, row_slot, ids, token_rows=None):
    """token_rows: optional device int32 [1], the moe_dispatch.token_rows bound."""
    return MoeDispatch(counts.data_ptr(), offs.data_ptr(), eti.data_ptr(), tim.data_ptr(), row_slot.data_ptr(),
                       ids.data_ptr(), token_rows.data_ptr() if token_rows is not None else None)


def moe_dispatch_build(p, topk_ids, disp, ws, stream=None):
    _check(load().moe_dispatch_build(ctypes.byref(p), _ptr(topk_ids), ctypes.byref(disp), _ptr(ws), ws.numel(),
                                     _stream(stream)), "moe_dispatch_build")


def moe_ffn_fwd(p, x, w1, w2, w3, topk_w, disp, a_save, b_save, u_save, y, ws, stream=None):
    _check(load().moe_ffn_fwd(ctypes.byref(p), _ptr(x), _ptr(w1), _ptr(w2), _ptr(w3), _ptr(topk_w),
                              ctypes.byref(disp), _ptr(a_save), _ptr(b_save), _ptr(u_save), _ptr(y), _ptr(ws),
                              ws.numel(), _stream(stream)), "moe_ffn_fwd")


def moe_ffn_fwd_ex(p, x, w1, w2, w3, topk_w, disp, a_save, b_save, u_save, y, ws, row_split=None, x_ready=None,
                   y_ready=None, t_ready=0, sm_reserve=0, stream=None):
    """moe_ffn_fwd with x rows [0, t_ready) resident and the rest ready at x_ready, y rows
    [t_ready, T) signalled by y_ready (torch.cuda.Event or None) before the down projection of
    the resident rows, which leaves sm_reserve SMs free; row_split from
    moe_dispatch_row_split(t_ready) (moe_fwd_sync)."""
    for ev in (x_ready, y_ready):
        if ev is not None and not ev.cuda_event:
            raise MoEError("moe_ffn_fwd_ex: events must be created (recorded once) before the call")
    sync = MoeFwdSync(_ptr(row_split), x_ready.cuda_event if x_ready is not None else None,
                      y_ready.cuda_event if y_ready is not None else None, int(t_ready), int(sm_reserve))
    _check(load().moe_ffn_fwd_ex(ctypes.byref(p), _ptr(x), _ptr(w1), _ptr(w2), _ptr(w3), _ptr(topk_w),
                                 ctypes.byref(disp), _ptr(a_save), _ptr(b_save), _ptr(u_save), _ptr(y),
                                 ctypes.byref(sync), _ptr(ws), ws.numel(), _stream(stream)), "moe_ffn_fwd_ex")


def moe_dispatch_row_split(p, disp, t_ready, row_split, stream=None):
    _check(load().moe_dispatch_row_split(ctypes.byref(p), ctypes.byref(disp), int(t_ready), _ptr(row_split),
                                         _stream(stream)), "moe_dispatch_row_split")


def moe_ffn_bwd(p, dy, x, w1, w2, w3, topk_w, disp, a_save, b_save, u_save, dx, dw1, dw2, dw3, d_topk_w, router, ws,
                stream=None, x_ready=None, dx_ready=None, stages=0):
    """x_ready / dx_ready: torch.cuda.Event or None; stages: MOE_BWD_* mask, 0 = all (moe_bwd_sync)."""
    sync = None
    for ev in (x_ready, dx_ready):
        if ev is not None and not ev.cuda_event:
            raise MoEError("moe_ffn_bwd: sync events must be created (recorded once) before the call")
    if x_ready is not None or dx_ready is not None or stages:
        sync = MoeBwdSync(x_ready.cuda_event if x_ready is not None else None,
                          dx_ready.cuda_event if dx_ready is not None else None, int(stages))
    _check(load().moe_ffn_bwd(ctypes.byref(p), _ptr(dy), _ptr(x), _ptr(w1), _ptr(w2), _ptr(w3), _ptr(topk_w),
                              ctypes.byref(disp), _ptr(a_save), _ptr(b_save), _ptr(u_save), _ptr(dx), _ptr(dw1),
                              _ptr(dw2), _ptr(dw3), _ptr(d_topk_w),
                              ctypes.byref(router) if router is not None else None,
                              ctypes.byref(sync) if sync is not None else None,
                              _ptr(ws), ws.numel(), _stream(stream)), "moe_ffn_bwd")


def moe_router_backward(p, d_topk_w, x, router, dx_partial, dx, ws, stream=None):
    _check(load().moe_router_backward(ctypes.byref(p), _ptr(d_topk_w), _ptr(x), ctypes.byref(router),
                                      _ptr(dx_partial), _ptr(dx), _ptr(ws), ws.numel(), _stream(stream)),
           "moe_router_backward")


def moe_ep_dest(p, topk_ids, experts_per_rank, n_ranks, dest, stream=None, self_rank=-1):
    _check(load().moe_ep_dest(ctypes.byref(p), _ptr(topk_ids), int(experts_per_rank), int(n_ranks), int(self_rank),
                              _ptr(dest), _stream(stream)), "moe_ep_dest")


def moe_ep_local_slots(p, topk_ids, topk_w, experts_per_rank, rank, local_ids, local_w, stream=None):
    _check(load().moe_ep_local_slots(ctypes.byref(p), _ptr(topk_ids), _ptr(topk_w), int(experts_per_rank), int(rank),
                                     _ptr(local_ids), _ptr(local_w), _stream(stream)), "moe_ep_local_slots")


def moe_ep_send_meta(p, topk_ids, topk_w, experts_per_rank, n_ranks, send_row_slot, send_ids, send_w, stream=None):
    _check(load().moe_ep_send_meta(ctypes.byref(p), _ptr(topk_ids), _ptr(topk_w), int(experts_per_rank),
                                   int(n_ranks), _ptr(send_row_slot), send_row_slot.numel(), _ptr(send_ids),
                                   _ptr(send_w), _stream(stream)), "moe_ep_send_meta")


def moe_ep_slot_grad(p, topk_ids, experts_per_rank, n_ranks, send_pos, dg_back, dg, stream=None, dg_local=None,
                     self_rank=-1):
    _check(load().moe_ep_slot_grad(ctypes.byref(p), _ptr(topk_ids), int(experts_per_rank), int(n_ranks),
                                   _ptr(send_pos), _ptr(dg_back), _ptr(dg_local), int(self_rank), _ptr(dg),
                                   _stream(stream)), "moe_ep_slot_grad")


def moe_gather_rows(src, index, dst, stream=None):
    """index None: dst[i] = src[i] for the rows of dst (a kernel copy; dst may be pinned host memory)."""
    n_src = src.shape[0]
    width = 1
    for s_ in src.shape[1:]:
        width *= s_
    n = index.numel() if index is not None else dst.shape[0]
    _check(load().moe_gather_rows(_ptr(src), n_src, _ptr(index), n, width, src.element_size(), _ptr(dst),
                                  _stream(stream)), "moe_gather_rows")


def moe_combine_rows(p, rows, token_index_map, out, stream=None, base=None):
    _check(load().moe_combine_rows(ctypes.byref(p), _ptr(rows), _ptr(token_index_map), _ptr(base), _ptr(out),
                                   _stream(stream)), "moe_combine_rows")


def moe_ep_signal(g, phase, epoch, stream=None):
    _check(load().moe_ep_signal(ctypes.byref(g), int(phase), int(epoch), _stream(stream)), "moe_ep_signal")


def moe_ep_wait(g, phase, epoch, stream=None):
    _check(load().moe_ep_wait(ctypes.byref(g), int(phase), int(epoch), _stream(stream)), "moe_ep_wait")


def moe_ep_publish_counts(g, counts, epoch, stream=None):
    _check(load().moe_ep_publish_counts(ctypes.byref(g), _ptr(counts), int(epoch), _stream(stream)),
           "moe_ep_publish_counts")


def moe_ep_push_rows(g, src, index, send_offs, n_max, row_bytes, dst_row0, peer_dst, phase, epoch, stream=None):
    """peer_dst: device int64 tensor [P] of the peers' destination addresses."""
    _check(load().moe_ep_push_rows(ctypes.byref(g), _ptr(src), _ptr(index), _ptr(send_offs), int(n_max),
                                   int(row_bytes), int(dst_row0), _ptr(peer_dst), int(phase), int(epoch),
                                   _stream(stream)), "moe_ep_push_rows")


def moe_ep_recv_prepare(g, T, T_cap, k, experts_per_rank, ids, w, token_rows=None, stream=None):
    _check(load().moe_ep_recv_prepare(ctypes.byref(g), int(T), int(T_cap), int(k), int(experts_per_rank), _ptr(ids),
                                      _ptr(w), _ptr(token_rows), _stream(stream)), "moe_ep_recv_prepare")


def moe_ep_pull_combine(g, p, peer_rows, row0, send_offs, send_pos, base, out, stream=None):
    _check(load().moe_ep_pull_combine(ctypes.byref(g), ctypes.byref(p), _ptr(peer_rows), int(row0), _ptr(send_offs),
                                      _ptr(send_pos), _ptr(base), _ptr(out), _stream(stream)), "moe_ep_pull_combine")


def moe_ep_pull_slot_grad(g, p, experts_per_rank, topk_ids, peer_dg, row0, send_offs, send_pos, dg_local, dg,
                          stream=None):
    _check(load().moe_ep_pull_slot_grad(ctypes.byref(g), ctypes.byref(p), int(experts_per_rank), _ptr(topk_ids),
                                        _ptr(peer_dg), int(row0), _ptr(send_offs), _ptr(send_pos), _ptr(dg_local),
                                        _ptr(dg), _stream(stream)), "moe_ep_pull_slot_grad")


def moe_ep_pull_sum(g, peer_src, n, dtype, out, stream=None):
    _check(load().moe_ep_pull_sum(ctypes.byref(g), _ptr(peer_src), int(n), int(dtype), _ptr(out), _stream(stream)),
           "moe_ep_pull_sum")


def ipc_handle(t):
    """(64-byte CUDA IPC handle of the allocation holding t, byte offset of t in it)."""
    h = (ctypes.c_char * 64)()
    off = ctypes.c_int64(0)
    _check(load().moe_ep_ipc_handle(_ptr(t), h, ctypes.byref(off)), "moe_ep_ipc_handle")
    return bytes(h), off.value


def ipc_open(handle, offset):
    """Map a peer's (handle, offset) on the current device: (address, mapping base)."""
    h = (ctypes.c_char * 64).from_buffer_copy(handle)
    ptr, base = ctypes.c_void_p(), ctypes.c_void_p()
    _check(load().moe_ep_ipc_open(h, int(offset), ctypes.byref(ptr), ctypes.byref(base)), "moe_ep_ipc_open")
    return ptr.value, base.value


def ipc_close(base):
    _check(load().moe_ep_ipc_close(ctypes.c_void_p(base)), "moe_ep_ipc_close")


def profile_enable(on=True):
    _check(load().moe_profile_enable(int(bool(on))), "moe_profile_enable")


def profile_reset():
    _check(load().moe_profile_reset(), "moe_profile_reset")


NAMED_STEPS = ("route", "dispatch", "zero_acc", "combine", "dg_reduce", "router_bwd", "finalize_dx")


def profile_read_named(names=NAMED_STEPS):
    """{step name: (total_ms, launches)} for the non-GEMM steps (moe_profile_read_named)."""
    out = {}
    for name in names:
        t, n = ctypes.c_double(0), ctypes.c_int64(0)
        _check(load().moe_profile_read_named(name.encode(), ctypes.byref(t), ctypes.byref(n)),
               "moe_profile_read_named")
        out[name] = (t.value, n.value)
    return out


def profile_read():
    """{kind name: (total_ms, launches)} for the six expert-GEMM kinds."""
    out = {}
    for i, name in enumerate(GEMM_KINDS):
        ms, n = ctypes.c_double(0), ctypes.c_int64(0)
        _check(load().moe_profile_read(i, ctypes.byref(ms), ctypes.byref(n)), "moe_profile_read")
        out[name] = (ms.value, n.value)
    return out
