"""C-ABI library: loads, exports every symbol include/moeblaze.h declares,
validates arguments and sizes its workspace without a GPU (CPU test)."""
import torch
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "moeblaze.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2601_05296_b200 import build as B
    B.build()
    from paper_2601_05296_b200 import _lib as L
    return L.load()


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(moe_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("moe_route", "moe_dispatch_build", "moe_ffn_fwd", "moe_ffn_bwd", "moe_workspace_size"):
        assert s in syms


def test_every_declared_symbol_is_exported(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s
    from paper_2601_05296_b200 import _lib as L
    assert set(L.EXPORTS) == set(declared_symbols())


def test_nm_exports_are_c_symbols():
    import subprocess
    so = os.path.join(ROOT, "paper_2601_05296_b200", "libmoeblaze.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    names = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for s in declared_symbols():
        assert s in names, s  # unmangled: extern "C"


def _problem(L, T=1024, d=256, h=512, E=8, k=2, dtype=0, renorm=0):
    return L.MoeProblem(T, d, h, E, k, dtype, renorm, 0)


def test_workspace_has_no_routed_token_term(lib):
    """By construction (SURVEY §8(c) audit 1): the fwd/bwd workspace is a closed
    form with no T*k*d term.  Its growth in d is the same for k = 2 and k = 8
    (only the [T, d] fp32 accumulators and router terms depend on d); k = 1
    stores each token's single row directly and needs no more than that."""
    from paper_2601_05296_b200 import _lib as L
    for (T, d, h, E) in [(1024, 256, 512, 8), (4096, 512, 256, 64), (2048, 1024, 1024, 16)]:
        for op in (L.MOE_OP_FFN_FWD, L.MOE_OP_FFN_BWD):
            grow = []
            for k in (1, 2, 8):
                s1 = L.workspace_size(_problem(L, T, d, h, E, k), op)
                s2 = L.workspace_size(_problem(L, T, 2 * d, h, E, k), op)
                grow.append(s2 - s1)
            assert abs(grow[2] - grow[1]) <= 2048, (T, d, h, E, op, grow)
            assert grow[0] <= grow[1] + 2048
            assert grow[1] <= T * d * 4 + 64 * E * d * 4 + 4096


def test_deterministic_workspace_is_the_row_buffer(lib):
    """deterministic = 1 (NEXT-4) replaces the [T, d] fp32 accumulator by the
    transient [T*k, d] fp32 row-result buffer -- exactly that, nothing else."""
    from paper_2601_05296_b200 import _lib as L
    for (T, d, h, E, k) in [(1024, 256, 512, 8, 2), (4096, 512, 256, 64, 6), (300, 128, 128, 16, 8)]:
        for op in (L.MOE_OP_FFN_FWD, L.MOE_OP_FFN_BWD):
            base = L.workspace_size(L.problem(T, d, h, E, k, torch.bfloat16), op)
            det = L.workspace_size(L.problem(T, d, h, E, k, torch.bfloat16, deterministic=True), op)
            assert abs((det - base) - (T * k - T) * d * 4) <= 512, (T, d, h, E, k, op, det - base)
        one = [L.workspace_size(L.problem(T, d, h, E, 1, torch.bfloat16, deterministic=det), L.MOE_OP_FFN_FWD)
               for det in (False, True)]
        assert one[0] == one[1]  # k = 1 ignores the flag


def test_argument_validation(lib):
    from paper_2601_05296_b200 import _lib as L
    n = ctypes.c_size_t(0)
    bad = [
        _problem(L, k=9, E=8),          # k > E
        _problem(L, E=300, k=2),        # E > 256
        _problem(L, T=-1),
        _problem(L, d=100),             # bf16 needs d % 128 == 0
        _problem(L, h=96),
    ]
    nd = _problem(L)
    nd.deterministic = 2            # only 0 / 1
    bad.append(nd)
    codes = [lib.moe_workspace_size(ctypes.byref(p), 2, ctypes.byref(n)) for p in bad]
    assert codes == [1, 1, 1, 2, 2, 1]
    ok = _problem(L, T=0)
    assert lib.moe_workspace_size(ctypes.byref(ok), 3, ctypes.byref(n)) == 0
    fp32 = _problem(L, d=64, h=96, dtype=1)
    assert lib.moe_workspace_size(ctypes.byref(fp32), 2, ctypes.byref(n)) == 0
    # null pointers are rejected synchronously, nothing is launched
    assert lib.moe_route(ctypes.byref(_problem(L)), None, None, None, None, None, None, 0, None) == 1
    assert lib.moe_status_string(4) == b"workspace too small"


def test_sparse_slot_rows_validation(lib):
    """moe_problem.rows (sparse slots, NEXT-1 EP receivers): 0 <= rows <= T*k;
    the workspace scales with rows, not T*k (no routed-token term either way)."""
    from paper_2601_05296_b200 import _lib as L
    n = ctypes.c_size_t(0)
    for rows, code in ((-1, 1), (1024 * 2 + 1, 1), (1, 0), (1024 * 2, 0)):
        p = L.problem(1024, 256, 512, 8, 2, torch.bfloat16, rows=rows)
        assert lib.moe_workspace_size(ctypes.byref(p), L.MOE_OP_FFN_FWD, ctypes.byref(n)) == code, rows
    dense = L.workspace_size(L.problem(1024, 256, 512, 8, 2, torch.bfloat16), L.MOE_OP_FFN_FWD)
    half = L.workspace_size(L.problem(1024, 256, 512, 8, 2, torch.bfloat16, rows=1024), L.MOE_OP_FFN_FWD)
    assert abs((dense - half) - 1024 * 512 * 2) <= 512  # the transient U buffer holds R = rows rows


def test_ep_helpers_validation(lib):
    """moe_ep_* reject a rank split that does not tile the experts and sparse
    source problems, synchronously (nothing launched: no GPU needed)."""
    from paper_2601_05296_b200 import _lib as L
    p = L.problem(16, 128, 128, 8, 2, torch.bfloat16)
    assert lib.moe_ep_dest(ctypes.byref(p), None, 3, 2, -1, None, None) == 1    # 3*2 != 8
    assert lib.moe_ep_dest(ctypes.byref(p), None, 4, 2, -1, None, None) == 1    # null pointers, T > 0
    assert lib.moe_ep_dest(ctypes.byref(p), None, 4, 2, 2, None, None) == 1     # self_rank out of range
    p0 = L.problem(0, 128, 128, 8, 2, torch.bfloat16)
    assert lib.moe_ep_dest(ctypes.byref(p0), None, 4, 2, 1, None, None) == 0    # T = 0: nothing to do
    assert lib.moe_ep_send_meta(ctypes.byref(p), None, None, 4, 2, None, 33, None, None, None) == 1  # n > T*P
    assert lib.moe_ep_send_meta(ctypes.byref(p0), None, None, 4, 2, None, 0, None, None, None) == 0
    ps = L.problem(16, 128, 128, 8, 2, torch.bfloat16, rows=8)
    assert lib.moe_ep_slot_grad(ctypes.byref(ps), None, 4, 2, None, None, None, -1, None, None) == 1  # sparse source
    assert lib.moe_ep_slot_grad(ctypes.byref(p0), None, 4, 2, None, None, None, 0, None, None) == 0
    assert lib.moe_ep_local_slots(ctypes.byref(p), None, None, 4, 2, None, None, None) == 1  # rank 2 of 8/4
    assert lib.moe_ep_local_slots(ctypes.byref(p0), None, None, 4, 1, None, None, None) == 0


def test_sparse_slots_allow_fewer_experts_than_k(lib):
    """an EP receiver owns E/P experts, possibly fewer than k
    (Mixtral-like E = 8, k = 2 on 8 ranks; DeepSeek-like k = 6 on 16 ranks): with
    sparse slots (rows > 0) k > E is valid; with every slot routed it is not."""
    from paper_2601_05296_b200 import _lib as L
    n = ctypes.c_size_t(0)
    for E, k in ((1, 2), (4, 6), (2, 8), (1, 64)):
        sp = L.problem(1024, 256, 512, E, k, torch.bfloat16, rows=1024)
        assert lib.moe_workspace_size(ctypes.byref(sp), L.MOE_OP_FFN_FWD, ctypes.byref(n)) == 0, (E, k)
        dense = L.problem(1024, 256, 512, E, k, torch.bfloat16)
        assert lib.moe_workspace_size(ctypes.byref(dense), L.MOE_OP_FFN_FWD, ctypes.byref(n)) == 1, (E, k)
    assert lib.moe_workspace_size(ctypes.byref(L.problem(64, 256, 512, 8, 300, torch.bfloat16, rows=10)),
                                  L.MOE_OP_FFN_FWD, ctypes.byref(n)) == 1   # k <= 256 with sparse slots


def test_checkpoint_policy_workspaces(lib):
    """MOE_CKPT_ABU (Alg. 1 literally): U lives in the caller's u_save, not
    in ws -- both workspaces shrink by exactly one [T*k, h] activation; every
    FFN workspace starts with the 256-byte tile-scheduler counter block."""
    from paper_2601_05296_b200 import _lib as L
    for (T, d, h, E, k) in [(1024, 256, 512, 8, 2), (300, 128, 384, 16, 6)]:
        for op in (L.MOE_OP_FFN_FWD, L.MOE_OP_FFN_BWD):
            ab = L.workspace_size(L.problem(T, d, h, E, k, torch.bfloat16), op)
            abu = L.workspace_size(L.problem(T, d, h, E, k, torch.bfloat16, checkpoint="abu"), op)
            assert abs((ab - abu) - T * k * h * 2) <= 256, (op, ab, abu)
        # MOE_CKPT_NONE: backward recomputes A, B into the caller's scratch a_save/b_save
        none_b = L.workspace_size(L.problem(T, d, h, E, k, torch.bfloat16, checkpoint="none"), L.MOE_OP_FFN_BWD)
        assert none_b == L.workspace_size(L.problem(T, d, h, E, k, torch.bfloat16), L.MOE_OP_FFN_BWD)


def test_staged_backward_validation(lib):
    """moe_bwd_sync.stages: an unknown bit is rejected; a stage whose output
    pointer is missing is rejected; nothing is launched (no GPU here)."""
    from paper_2601_05296_b200 import _lib as L
    p = L.problem(16, 128, 128, 4, 2, torch.bfloat16)
    disp = L.MoeDispatch(256, 256, 256, 256, 256, 256)
    f = ctypes.c_void_p(256)
    for stages, dws in ((8, (f, f, f)), (L.MOE_BWD_DW3, (f, f, None)), (L.MOE_BWD_DW12, (None, f, f)),
                        (L.MOE_BWD_DW12, (f, None, f))):
        sync = L.MoeBwdSync(None, None, stages)
        code = lib.moe_ffn_bwd(ctypes.byref(p), f, f, f, f, f, f, ctypes.byref(disp), f, f, None, f, *dws, f, None,
                               ctypes.byref(sync), f, 1 << 40, None)
        assert code == 1, (stages, code)


def test_sm_topology_validation(lib):
    import ctypes
    n = (ctypes.c_int32 * 2)()
    assert lib.moe_sm_topology(None, 4, n) != 0
    dies = (ctypes.c_int32 * 4)()
    assert lib.moe_sm_topology(dies, 4, None) != 0
    assert lib.moe_sm_topology(dies, -1, n) != 0


def test_ep_peer_exchange_validation(lib):
    """The peer-memory exchange entry points reject a missing / inconsistent
    peer description and bad phases synchronously; calls with nothing to move
    return OK without launching (no GPU needed)."""
    from paper_2601_05296_b200 import _lib as L
    fake = ctypes.c_void_p(0x1000)  # never dereferenced: every call below returns before a launch
    g = L.MoeEpPeers(2, 0, fake, fake, fake, fake, 0)
    bad_rank = L.MoeEpPeers(2, 2, fake, fake, fake, fake, 0)
    no_tables = L.MoeEpPeers(2, 0, None, None, fake, fake, 0)
    for gg in (bad_rank, no_tables):
        assert lib.moe_ep_signal(ctypes.byref(gg), 0, 1, None) == 1
        assert lib.moe_ep_wait(ctypes.byref(gg), 0, 1, None) == 1
    assert lib.moe_ep_signal(None, 0, 1, None) == 1
    assert lib.moe_ep_signal(ctypes.byref(g), L.MOE_EP_NPHASE, 1, None) == 1       # phase out of range
    assert lib.moe_ep_wait(ctypes.byref(g), -1, 1, None) == 1
    assert lib.moe_ep_publish_counts(ctypes.byref(g), None, 1, None) == 1          # no counts
    assert lib.moe_ep_push_rows(ctypes.byref(g), None, None, fake, 4, 6, 0, fake, -1, 1, None) == 1  # row_bytes % 4
    assert lib.moe_ep_push_rows(ctypes.byref(g), None, None, fake, 4, 8, 0, fake, -1, 1, None) == 1  # src null, n > 0
    assert lib.moe_ep_recv_prepare(ctypes.byref(g), 16, 8, 2, 4, None, None, None, None) == 1  # T_cap < T
    assert lib.moe_ep_recv_prepare(ctypes.byref(g), 16, 16, 2, 4, None, None, None, None) == 0  # nothing received
    p = L.problem(16, 100, 128, 8, 2, torch.bfloat16)                                    # d % 8 != 0
    assert lib.moe_ep_pull_combine(ctypes.byref(g), ctypes.byref(p), fake, 16, fake, fake, None, fake, None) == 1
    p0 = L.problem(0, 128, 128, 8, 2, torch.bfloat16)
    assert lib.moe_ep_pull_combine(ctypes.byref(g), ctypes.byref(p0), None, 0, None, None, None, None, None) == 0
    p8 = L.problem(16, 128, 128, 8, 2, torch.bfloat16)
    assert lib.moe_ep_pull_slot_grad(ctypes.byref(g), ctypes.byref(p8), 3, None, None, 16, None, None, None, None,
                                      None) == 1                                         # 3 * 2 ranks != 8 experts
    assert lib.moe_ep_pull_sum(ctypes.byref(g), None, 10, 7, None, None) == 1            # unknown dtype
    assert lib.moe_ep_pull_sum(ctypes.byref(g), None, 0, 0, None, None) == 0
    h = (ctypes.c_char * 64)()
    off = ctypes.c_int64()
    assert lib.moe_ep_ipc_handle(None, h, ctypes.byref(off)) == 1
    assert lib.moe_ep_ipc_close(None) == 1


def test_forward_overlap_validation(lib):
    """moe_dispatch_row_split / moe_ffn_fwd_ex (NEXT-1 forward overlap) reject bad
    arguments synchronously: t_ready outside [0, T], missing dispatch arrays, null
    operands -- and T = 0 launches nothing (no GPU needed)."""
    from paper_2601_05296_b200 import _lib as L
    p = L.problem(1024, 256, 512, 8, 2, torch.bfloat16)
    fake = ctypes.c_void_p(256)  # never dereferenced: validation fails first
    d = L.MoeDispatch(fake, fake, fake, fake, fake, fake, None)
    for t_ready in (-1, 1025):
        assert lib.moe_dispatch_row_split(ctypes.byref(p), ctypes.byref(d), t_ready, fake, None) == 1
    assert lib.moe_dispatch_row_split(ctypes.byref(p), None, 0, fake, None) == 1
    assert lib.moe_dispatch_row_split(ctypes.byref(p), ctypes.byref(d), 0, None, None) == 1
    nod = L.MoeDispatch(fake, None, fake, fake, fake, fake, None)
    assert lib.moe_dispatch_row_split(ctypes.byref(p), ctypes.byref(nod), 0, fake, None) == 1
    sync = L.MoeFwdSync(None, None, None, 0, 0)
    ws_n = L.workspace_size(p, L.MOE_OP_FFN_FWD)
    # null x / y / weights: invalid before anything is launched
    assert lib.moe_ffn_fwd_ex(ctypes.byref(p), None, None, None, None, None, ctypes.byref(d), None, None, None, None,
                              ctypes.byref(sync), fake, ws_n, None) == 1
    # workspace too small
    assert lib.moe_ffn_fwd_ex(ctypes.byref(p), fake, fake, fake, fake, fake, ctypes.byref(d), fake, fake, None, fake,
                              ctypes.byref(sync), fake, ws_n - 1, None) == 4
    # the struct layout the binding passes matches the header's field order
    assert [f[0] for f in L.MoeFwdSync._fields_] == ["row_split", "x_ready", "y_ready", "t_ready", "sm_reserve"]
