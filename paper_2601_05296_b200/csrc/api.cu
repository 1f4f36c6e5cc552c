// api.cu — the C ABI declared in include/moeblaze.h: validation, workspace
// layout, and the launch sequence of every entry point.
#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "gemm.h"

namespace moeb {

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// launchers defined in the other translation units
moe_status launch_route(const moe_problem*, const void*, const void*, float*, int32_t*, float*, cudaStream_t);
moe_status launch_dispatch(const moe_problem*, const int32_t*, const moe_dispatch*, int32_t*, int32_t*, cudaStream_t);
size_t dispatch_ws_bytes(const moe_problem*);
moe_status launch_dg_reduce(const float*, int, const int32_t*, int64_t, float*, cudaStream_t);
int dwg_chunks(const moe_problem* p);
moe_status launch_router_bwd(const moe_problem*, const float*, const int32_t*, const float*, const void*, float*,
                             __nv_bfloat16*, float*, void*, cudaStream_t);
moe_status launch_zero_acc(float*, int64_t, int, const int32_t*, cudaStream_t);
// row0: acc / out start at token row row0 of the problem (t_rows stays the absolute bound)
moe_status launch_finalize(const moe_problem*, const void*, const float*, const __nv_bfloat16*, const void*, void*,
                           cudaStream_t, bool, const int32_t*, const int32_t*, int64_t row0 = 0);
int router_ep8(int E);
moe_status launch_ep_dest(const int32_t*, int64_t, int, int, int, int, int32_t*, cudaStream_t);
moe_status launch_ep_local_slots(const int32_t*, const float*, int64_t, int, int, int32_t*, float*, cudaStream_t);
moe_status launch_ep_send_meta(const int32_t*, const float*, int, int, int, const int32_t*, int64_t, int32_t*, float*,
                               cudaStream_t);
moe_status launch_ep_slot_grad(const int32_t*, int64_t, int, int, int, const int32_t*, const float*, const float*, int,
                               float*, cudaStream_t);
moe_status launch_gather_rows(const void*, const int32_t*, int64_t, int64_t, void*, cudaStream_t);
moe_status launch_combine_rows(const moe_problem*, const void*, const int32_t*, const void*, void*, cudaStream_t);
moe_status launch_row_split(const int32_t*, const int32_t*, int, int64_t, int32_t*, cudaStream_t);

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

static moe_status validate(const moe_problem* p) {
  if (!p) return MOE_ERR_INVALID_ARG;
  if (p->T < 0 || p->d < 1 || p->h < 1 || p->E < 1 || p->k < 1) return MOE_ERR_INVALID_ARG;
  if (p->E > 256) return MOE_ERR_INVALID_ARG;
  // every slot routed: k distinct experts per token (k <= E), top-k selection keeps <= 16.
  // Sparse slots (rows > 0, -1 = empty slot): a receiver may own fewer experts than k
  // (expert parallel with E/P < k), and the rank-level send plan uses k = P
  if (p->rows == 0 && (p->k > p->E || p->k > 16)) return MOE_ERR_INVALID_ARG;
  if (p->rows > 0 && p->k > 256) return MOE_ERR_INVALID_ARG;
  if (p->T * (int64_t)p->k >= (int64_t(1) << 31)) return MOE_ERR_INVALID_ARG;
  if (p->dtype != MOE_BF16 && p->dtype != MOE_FP32) return MOE_ERR_INVALID_ARG;
  if (p->dtype == MOE_BF16 && (p->d % 128 != 0 || p->h % 128 != 0)) return MOE_ERR_UNSUPPORTED;
  if (p->dtype == MOE_FP32 && (p->d % 8 != 0)) return MOE_ERR_UNSUPPORTED;
  if (p->checkpoint != MOE_CKPT_AB && p->checkpoint != MOE_CKPT_NONE && p->checkpoint != MOE_CKPT_ABU)
    return MOE_ERR_INVALID_ARG;
  if (p->activation < MOE_ACT_SWIGLU || p->activation > MOE_ACT_RELU) return MOE_ERR_INVALID_ARG;
  if (p->deterministic != 0 && p->deterministic != 1) return MOE_ERR_INVALID_ARG;
  if (p->rows < 0 || p->rows > p->T * (int64_t)p->k) return MOE_ERR_INVALID_ARG;
  return MOE_OK;
}

// routed rows R: T*k, or p->rows with sparse slots (empty slots = -1 in topk_ids)
static int64_t routed_rows(const moe_problem* p) { return p->rows > 0 ? p->rows : p->T * p->k; }
static bool sparse_slots(const moe_problem* p) { return p->rows > 0; }

static bool aligned16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; }

static size_t esize(const moe_problem* p) { return p->dtype == MOE_BF16 ? 2 : 4; }

// dg partial columns per routed row: the max over the GEMM backends
static int dg_parts(const moe_problem* p) { return (int)ceil_div(p->h, 64); }

// Output mode of the down-projection GEMMs (gemm.h OutMode) and the fp32 rows
// of the accumulator it needs.  k = 1: every token has exactly one routed row,
// so it is stored, not added (bit-identical to red.add onto zero) -- straight
// into the output when nothing else is added to it.  deterministic: one fp32
// row per routed row, summed per token in slot order by the finalize pass.
static int out_mode(const moe_problem* p, bool more_terms) {
  if (p->k == 1 && !sparse_slots(p)) return more_terms ? OUT_TOK : OUT_TOKN;  // sparse: a token may have no row
  return p->deterministic ? OUT_ROWS : OUT_RED;
}
static int64_t acc_rows(const moe_problem* p, int mode) {
  return mode == OUT_TOKN ? 0 : (mode == OUT_ROWS ? routed_rows(p) : p->T);
}

// The FFN workspaces start with the tile-scheduler claim counters of the expert GEMMs: one
// 16-byte slot per GEMM launch of the call (zeroed on the stream right before that launch),
// so concurrent calls on other streams and CUDA-graph replays never share counters.
constexpr size_t SCHED_BYTES = 256;
enum { SCHED_UP = 0, SCHED_DOWN = 1, SCHED_DH = 2, SCHED_DX = 3, SCHED_DW3 = 4, SCHED_DW12 = 5 };
static int* sched_at(void* ws, int slot) { return reinterpret_cast<int*>(ws) + 4 * slot; }

// U (or wU under MOE_CKPT_ABU, then the caller's u_save) between the two forward GEMMs
struct FwdWs { void* u; float* yacc; void* a; void* b; size_t total; };
static FwdWs fwd_layout(const moe_problem* p, void* base) {
  const int64_t R = routed_rows(p);
  char* b = (char*)base;
  size_t o = SCHED_BYTES;
  FwdWs w;
  w.u = nullptr;
  if (p->checkpoint != MOE_CKPT_ABU) { w.u = b + o; o += align256((size_t)R * p->h * esize(p)); }
  w.yacc = (float*)(b + o); o += align256((size_t)acc_rows(p, out_mode(p, false)) * p->d * 4);
  w.a = w.b = nullptr;
  if (p->checkpoint == MOE_CKPT_NONE) {  // A, B are transient: not checkpointed
    w.a = b + o; o += align256((size_t)R * p->h * esize(p));
    w.b = b + o; o += align256((size_t)R * p->h * esize(p));
  }
  w.total = o;
  return w;
}

// dl hi/lo split (bf16 runs): [2, T, ep8] bf16, the router tensor-core operands
static size_t dlhl_bytes(const moe_problem* p) {
  return p->dtype == MOE_BF16 ? align256((size_t)2 * p->T * router_ep8(p->E) * 2) : 0;
}

struct RouterWs { float* dlogits; __nv_bfloat16* dlhl; float* dwgpart; size_t total; };
static RouterWs router_layout(const moe_problem* p, void* base) {
  char* b = (char*)base;
  size_t o = 0;
  RouterWs w;
  w.dlogits = (float*)(b + o); o += align256((size_t)p->T * p->E * 4);
  w.dlhl = (__nv_bfloat16*)(b + o); o += dlhl_bytes(p);
  w.dwgpart = (float*)(b + o); o += align256((size_t)dwg_chunks(p) * p->E * p->d * 4);
  w.total = o;
  return w;
}

// wU (written by the dH GEMM, read by the dW3 GEMM; under MOE_CKPT_ABU the caller's saved
// u_save instead) and the transients of the data-gradient stage
struct BwdWs { void* wu; float* dxacc; float* dgpart; float* dlogits; __nv_bfloat16* dlhl; float* dwgpart; float* dg; size_t total; };
static BwdWs bwd_layout(const moe_problem* p, void* base) {
  const int64_t R = routed_rows(p);
  char* b = (char*)base;
  size_t o = SCHED_BYTES;
  BwdWs w;
  w.wu = nullptr;
  if (p->checkpoint != MOE_CKPT_ABU) { w.wu = b + o; o += align256((size_t)R * p->h * esize(p)); }
  w.dxacc = (float*)(b + o); o += align256((size_t)acc_rows(p, out_mode(p, true)) * p->d * 4);  // router or not
  w.dgpart = (float*)(b + o); o += align256((size_t)R * dg_parts(p) * 4);
  w.dlogits = (float*)(b + o); o += align256((size_t)p->T * p->E * 4);
  w.dlhl = (__nv_bfloat16*)(b + o); o += dlhl_bytes(p);
  w.dwgpart = (float*)(b + o); o += align256((size_t)dwg_chunks(p) * p->E * p->d * 4);
  w.dg = (float*)(b + o); o += align256((size_t)p->T * p->k * 4);
  w.total = o;
  return w;
}

}  // namespace moeb

using namespace moeb;

extern "C" {

const char* moe_status_string(moe_status s) {
  switch (s) {
    case MOE_OK: return "ok";
    case MOE_ERR_INVALID_ARG: return "invalid argument";
    case MOE_ERR_UNSUPPORTED: return "unsupported configuration";
    case MOE_ERR_MISALIGNED: return "pointer not 16-byte aligned";
    case MOE_ERR_WORKSPACE: return "workspace too small";
    case MOE_ERR_BAD_ROUTING: return "invalid routing (expert id out of range or repeated within a token)";
    case MOE_ERR_CUDA: return "CUDA launch error";
  }
  return "unknown status";
}

uint64_t moe_launch_count(void) { return g_launches.load(); }
int32_t moe_version(void) { return 100; }

moe_status moe_workspace_size(const moe_problem* p, moe_op op, size_t* bytes) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  if (!bytes) return MOE_ERR_INVALID_ARG;
  switch (op) {
    case MOE_OP_ROUTE: *bytes = 0; break;
    case MOE_OP_DISPATCH: *bytes = dispatch_ws_bytes(p); break;
    case MOE_OP_FFN_FWD: *bytes = fwd_layout(p, nullptr).total; break;
    case MOE_OP_FFN_BWD: *bytes = bwd_layout(p, nullptr).total; break;
    case MOE_OP_ROUTER_BWD: *bytes = router_layout(p, nullptr).total; break;
    default: return MOE_ERR_INVALID_ARG;
  }
  return MOE_OK;
}

moe_status moe_route(const moe_problem* p, const void* x, const void* w_gate, float* logits, int32_t* topk_ids,
                     float* topk_w, void* ws, size_t ws_bytes, void* stream) {
  (void)ws; (void)ws_bytes;
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  if (p->T > 0 && (!x || !w_gate || !logits || !topk_ids || !topk_w)) return MOE_ERR_INVALID_ARG;
  ProfScope prof("route", (cudaStream_t)stream);
  return launch_route(p, x, w_gate, logits, topk_ids, topk_w, (cudaStream_t)stream);
}

moe_status moe_dispatch_build(const moe_problem* p, const int32_t* topk_ids, const moe_dispatch* out, void* ws,
                              size_t ws_bytes, void* stream) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  if (!out || !out->expert_counts || !out->expert_offsets) return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && (!topk_ids || !out->expert_token_indices || !out->token_index_map || !ws)) return MOE_ERR_INVALID_ARG;
  if (ws_bytes < dispatch_ws_bytes(p)) return MOE_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* status = (int32_t*)ws;
  if (p->check_routing) MOE_CUDA_CHECK(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
  ProfScope prof("dispatch", st);
  return launch_dispatch(p, topk_ids, out, (int32_t*)((char*)ws + 256), status, st);  // rows checked if check_routing
}

moe_status moe_ffn_fwd(const moe_problem* p, const void* x, const void* w1, const void* w2, const void* w3,
                       const float* topk_w, const moe_dispatch* disp, void* a_save, void* b_save, void* u_save,
                       void* y, void* ws, size_t ws_bytes, void* stream) {
  return moe_ffn_fwd_ex(p, x, w1, w2, w3, topk_w, disp, a_save, b_save, u_save, y, nullptr, ws, ws_bytes, stream);
}

moe_status moe_dispatch_row_split(const moe_problem* p, const moe_dispatch* disp, int64_t t_ready, int32_t* row_split,
                                  void* stream) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  if (!disp || !disp->expert_offsets || !row_split || t_ready < 0 || t_ready > p->T) return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && !disp->expert_token_indices) return MOE_ERR_INVALID_ARG;
  return launch_row_split(disp->expert_offsets, disp->expert_token_indices, p->E, t_ready, row_split,
                          (cudaStream_t)stream);
}

moe_status moe_ffn_fwd_ex(const moe_problem* p, const void* x, const void* w1, const void* w2, const void* w3,
                          const float* topk_w, const moe_dispatch* disp, void* a_save, void* b_save, void* u_save,
                          void* y, const moe_fwd_sync* sync, void* ws, size_t ws_bytes, void* stream) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  const bool gated = p->activation == MOE_ACT_SWIGLU;
  if (!disp || !w1 || (gated && !w2) || !w3) return MOE_ERR_INVALID_ARG;
  const bool ckpt = p->checkpoint != MOE_CKPT_NONE;
  const bool abu = p->checkpoint == MOE_CKPT_ABU;
  if (p->T > 0 && (!x || !y || !topk_w || (ckpt && (!a_save || (gated && !b_save))) || (abu && !u_save) || !ws ||
                   !disp->expert_offsets || !disp->expert_token_indices || !disp->row_slot ||
                   (out_mode(p, false) == OUT_ROWS && !disp->token_index_map)))
    return MOE_ERR_INVALID_ARG;
  if (!aligned16(x) || !aligned16(w1) || !aligned16(w2) || !aligned16(w3) || !aligned16(a_save) ||
      !aligned16(b_save) || !aligned16(u_save) || !aligned16(y))
    return MOE_ERR_MISALIGNED;
  FwdWs w = fwd_layout(p, ws);
  if (ws_bytes < w.total) return MOE_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->T == 0) {
    if (sync && sync->y_ready) MOE_CUDA_CHECK(cudaEventRecord((cudaEvent_t)sync->y_ready, st));
    return MOE_OK;
  }
  if (!ckpt) {
    a_save = w.a;
    b_save = w.b;
  }
  const int mode = out_mode(p, false);
  if (mode == OUT_RED) {
    ProfScope prof("zero_acc", st);
    if ((s = launch_zero_acc(w.yacc, p->T, p->d, disp->token_rows, st)) != MOE_OK) return s;
  }
  GemmCall c{};
  c.out_mode = mode; c.out_tok = y;
  c.x = x; c.w1 = w1; c.w2 = w2; c.w3 = w3; c.topw = topk_w;
  c.offs = disp->expert_offsets; c.eti = disp->expert_token_indices; c.row_slot = disp->row_slot;
  c.a_save = a_save; c.b_save = b_save; c.u = abu ? u_save : w.u; c.acc_out = w.yacc;
  c.u_weighted = abu;  // ABU: U carries the gate weight (Alg. 1's saved Y_swi, scaled by w)
  c.T = p->T; c.R = routed_rows(p); c.d = p->d; c.h = p->h; c.E = p->E; c.bf16 = p->dtype == MOE_BF16;
  c.act = p->activation;
  c.which = GEMM_FWD_UP;
  c.sched = sched_at(ws, SCHED_UP);
  cudaEvent_t x_ready = sync ? (cudaEvent_t)sync->x_ready : nullptr;
  cudaEvent_t y_ready = sync ? (cudaEvent_t)sync->y_ready : nullptr;
  const bool split = sync && sync->row_split && c.bf16 && tc_splits_rows();
  if (split) {
    // the rows whose X is resident first, then (after x_ready) the rest: A, B, U land in
    // the same rows as one launch would write
    c.row_split = sync->row_split;
    c.split_half = 1;
    if ((s = run_gemm(c, st)) != MOE_OK) return s;
    if (x_ready) MOE_CUDA_CHECK(cudaStreamWaitEvent(st, x_ready, 0));
    c.split_half = 2;
    if ((s = run_gemm(c, st)) != MOE_OK) return s;
  } else {
    if (x_ready) MOE_CUDA_CHECK(cudaStreamWaitEvent(st, x_ready, 0));
    if ((s = run_gemm(c, st)) != MOE_OK) return s;
  }
  c.which = GEMM_FWD_DOWN;
  c.sched = sched_at(ws, SCHED_DOWN);
  const int64_t t_ready = split ? sync->t_ready : 0;
  if (split && y_ready && mode == OUT_RED && t_ready >= 0 && t_ready <= p->T) {
    // the received rows' y first (their tokens are >= t_ready: they red.add only into rows
    // [t_ready, T)), finalised and signalled so their return overlaps the local rows' down
    // projection, which leaves sm_reserve SMs to the exchange kernel
    const size_t es = esize(p);
    moe_problem hi = *p, lo = *p;
    hi.T = p->T - t_ready;
    lo.T = t_ready;
    c.split_half = 2;
    if ((s = run_gemm(c, st)) != MOE_OK) return s;
    {
      ProfScope prof("combine", st);
      if ((s = launch_finalize(&hi, w.yacc + t_ready * p->d, nullptr, nullptr, nullptr,
                               (char*)y + (size_t)t_ready * p->d * es, st, false, nullptr, disp->token_rows,
                               t_ready)) != MOE_OK)
        return s;
    }
    MOE_CUDA_CHECK(cudaEventRecord(y_ready, st));
    c.split_half = 1;
    c.sm_reserve = sync->sm_reserve;
    if ((s = run_gemm(c, st)) != MOE_OK) return s;
    ProfScope prof("combine", st);
    return launch_finalize(&lo, w.yacc, nullptr, nullptr, nullptr, y, st, false, nullptr, disp->token_rows);
  }
  c.row_split = nullptr;
  c.split_half = 0;
  if ((s = run_gemm(c, st)) != MOE_OK) return s;
  if (mode != OUT_TOKN) {
    ProfScope prof("combine", st);
    if ((s = launch_finalize(p, w.yacc, nullptr, nullptr, nullptr, y, st, false,
                             mode == OUT_ROWS ? disp->token_index_map : nullptr, disp->token_rows)) != MOE_OK)
      return s;
  }
  if (y_ready) MOE_CUDA_CHECK(cudaEventRecord(y_ready, st));
  return MOE_OK;
}

moe_status moe_ffn_bwd(const moe_problem* p, const void* dy, const void* x, const void* w1, const void* w2,
                       const void* w3, const float* topk_w, const moe_dispatch* disp, void* a_save, void* b_save,
                       void* u_save, void* dx, void* dw1, void* dw2, void* dw3, float* d_topk_w,
                       const moe_router_bwd* router, const moe_bwd_sync* sync, void* ws, size_t ws_bytes,
                       void* stream) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  const int stages = (sync && sync->stages) ? sync->stages : MOE_BWD_ALL;
  if (stages & ~MOE_BWD_ALL) return MOE_ERR_INVALID_ARG;
  const bool s_data = stages & MOE_BWD_DATA, s_dw3 = stages & MOE_BWD_DW3, s_dw12 = stages & MOE_BWD_DW12;
  const bool gated = p->activation == MOE_ACT_SWIGLU;
  const bool abu = p->checkpoint == MOE_CKPT_ABU;
  if (!disp || (s_dw12 && (!dw1 || (gated && !dw2))) || (s_dw3 && !dw3)) return MOE_ERR_INVALID_ARG;
  if (s_data && (!w1 || !w3 || (gated && !w2))) return MOE_ERR_INVALID_ARG;
  if (router && (!router->w_gate || !router->dw_gate)) return MOE_ERR_INVALID_ARG;
  if (router && p->T > 0 && (!router->logits || !router->topk_ids)) return MOE_ERR_INVALID_ARG;
  if (router && sparse_slots(p)) return MOE_ERR_INVALID_ARG;  // the router sees every slot of its own tokens
  if (p->T > 0 && (!ws || !disp->expert_offsets || !disp->expert_token_indices || !disp->token_index_map ||
                   !disp->row_slot || !topk_w))
    return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && (s_data || s_dw12) && (!a_save || (gated && !b_save))) return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && s_data && (!dy || !x || !dx)) return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && s_dw3 && (!dy || (abu && !u_save))) return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && s_dw12 && !x) return MOE_ERR_INVALID_ARG;
  if (!aligned16(dy) || !aligned16(x) || !aligned16(a_save) || !aligned16(b_save) || !aligned16(u_save) ||
      !aligned16(dx) || !aligned16(dw1) || !aligned16(dw2) || !aligned16(dw3))
    return MOE_ERR_MISALIGNED;
  BwdWs w = bwd_layout(p, ws);
  if (ws_bytes < w.total) return MOE_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t x_ready = sync ? (cudaEvent_t)sync->x_ready : nullptr;
  cudaEvent_t dx_ready = sync ? (cudaEvent_t)sync->dx_ready : nullptr;
  const int64_t R = routed_rows(p);
  GemmCall c{};
  c.x = x; c.dy = dy; c.w1 = w1; c.w2 = w2; c.w3 = w3; c.topw = topk_w;
  c.offs = disp->expert_offsets; c.eti = disp->expert_token_indices; c.row_slot = disp->row_slot;
  c.a_save = a_save; c.b_save = b_save; c.u = abu ? u_save : w.wu; c.acc_out = w.dxacc; c.dg_part = w.dgpart;
  c.dh_skip_u = abu;  // ABU: wU is saved, the dH GEMM does not write it
  c.T = p->T; c.R = R; c.d = p->d; c.h = p->h; c.E = p->E; c.bf16 = p->dtype == MOE_BF16;
  c.act = p->activation;
  const int mode = out_mode(p, router != nullptr);
  c.out_mode = mode; c.out_tok = dx;
  if (s_data) {
    if (p->T > 0) {
      if (mode == OUT_RED) {
        ProfScope prof("zero_acc", st);
        if ((s = launch_zero_acc(w.dxacc, p->T, p->d, disp->token_rows, st)) != MOE_OK) return s;
      }
      if (p->checkpoint == MOE_CKPT_NONE) {  // recompute A, B (and U into the wU buffer) with the fused up-projection
        c.which = GEMM_FWD_UP;
        c.sched = sched_at(ws, SCHED_UP);
        if ((s = run_gemm(c, st)) != MOE_OK) return s;
      }
      c.which = GEMM_BWD_DH;  // dH, SwiGLU bwd: dA/dB in place, wU, dg partials
      c.sched = sched_at(ws, SCHED_DH);
      if ((s = run_gemm(c, st)) != MOE_OK) return s;
      float* dg = d_topk_w ? d_topk_w : w.dg;
      {
        ProfScope prof("dg_reduce", st);
        if ((s = launch_dg_reduce(w.dgpart, gemm_dg_parts(c), disp->token_index_map, p->T * p->k, dg, st)) != MOE_OK)
          return s;
      }
      c.which = GEMM_BWD_DX;   // dXacc += [dA|dB][W1;W2]
      c.sched = sched_at(ws, SCHED_DX);
      if ((s = run_gemm(c, st)) != MOE_OK) return s;
      if (mode != OUT_TOKN) {  // (k = 1 without router: dx already written by the dX GEMM)
        const float* dl = nullptr;
        if (router) {
          if (x_ready) MOE_CUDA_CHECK(cudaStreamWaitEvent(st, x_ready, 0));  // dW_g = dlogits^T x reads x
          ProfScope prof("router_bwd", st);
          if ((s = launch_router_bwd(p, router->logits, router->topk_ids, dg, x, w.dlogits, w.dlhl, w.dwgpart,
                                     router->dw_gate, st)) != MOE_OK)
            return s;
          dl = w.dlogits;
        }
        ProfScope prof("finalize_dx", st);
        if ((s = launch_finalize(p, w.dxacc, dl, w.dlhl, router ? router->w_gate : nullptr, dx, st, false,
                                 mode == OUT_ROWS ? disp->token_index_map : nullptr, disp->token_rows)) != MOE_OK)
          return s;
      }
    } else if (router) {
      MOE_CUDA_CHECK(cudaMemsetAsync(router->dw_gate, 0, (size_t)p->E * p->d * esize(p), st));
    }
    if (dx_ready) MOE_CUDA_CHECK(cudaEventRecord(dx_ready, st));
  }
  if (s_dw3) {
    c.which = GEMM_DW3;      // dW3 = dY^T (wU)
    c.dw_a = dw3; c.dw_b = nullptr;
    c.sched = sched_at(ws, SCHED_DW3);
    if ((s = run_gemm(c, st)) != MOE_OK) return s;
  }
  if (s_dw12) {
    if (x_ready) MOE_CUDA_CHECK(cudaStreamWaitEvent(st, x_ready, 0));
    c.which = GEMM_DW12;     // dW1, dW2 = [dA|dB]^T X
    c.dw_a = dw1; c.dw_b = dw2;
    c.sched = sched_at(ws, SCHED_DW12);
    if ((s = run_gemm(c, st)) != MOE_OK) return s;
  }
  return MOE_OK;
}

moe_status moe_router_backward(const moe_problem* p, const float* d_topk_w, const void* x, const moe_router_bwd* router,
                               const void* dx_partial, void* dx, void* ws, size_t ws_bytes, void* stream) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  if (!router || !router->w_gate || !router->dw_gate) return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && (!d_topk_w || !x || !router->logits || !router->topk_ids || !dx_partial || !dx || !ws))
    return MOE_ERR_INVALID_ARG;
  RouterWs w = router_layout(p, ws);
  if (ws_bytes < w.total) return MOE_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->T == 0) {
    MOE_CUDA_CHECK(cudaMemsetAsync(router->dw_gate, 0, (size_t)p->E * p->d * esize(p), st));
    return MOE_OK;
  }
  if ((s = launch_router_bwd(p, router->logits, router->topk_ids, d_topk_w, x, w.dlogits, w.dlhl, w.dwgpart,
                             router->dw_gate, st)) != MOE_OK)
    return s;
  return launch_finalize(p, dx_partial, w.dlogits, w.dlhl, router->w_gate, dx, st, true, nullptr, nullptr);
}

moe_status moe_ep_dest(const moe_problem* p, const int32_t* topk_ids, int32_t experts_per_rank, int32_t n_ranks,
                       int32_t self_rank, int32_t* dest, void* stream) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  if (experts_per_rank < 1 || n_ranks < 1 || (int64_t)experts_per_rank * n_ranks != p->E || sparse_slots(p))
    return MOE_ERR_INVALID_ARG;
  if (self_rank < -1 || self_rank >= n_ranks) return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && (!topk_ids || !dest)) return MOE_ERR_INVALID_ARG;
  return launch_ep_dest(topk_ids, p->T, p->k, experts_per_rank, n_ranks, self_rank, dest, (cudaStream_t)stream);
}

moe_status moe_ep_local_slots(const moe_problem* p, const int32_t* topk_ids, const float* topk_w,
                              int32_t experts_per_rank, int32_t rank, int32_t* local_ids, float* local_w,
                              void* stream) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  if (experts_per_rank < 1 || rank < 0 || (int64_t)experts_per_rank * (rank + 1) > p->E || sparse_slots(p))
    return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && (!topk_ids || !topk_w || !local_ids || !local_w)) return MOE_ERR_INVALID_ARG;
  return launch_ep_local_slots(topk_ids, topk_w, p->T * p->k, experts_per_rank, rank, local_ids, local_w,
                               (cudaStream_t)stream);
}

moe_status moe_ep_send_meta(const moe_problem* p, const int32_t* topk_ids, const float* topk_w, int32_t experts_per_rank,
                            int32_t n_ranks, const int32_t* send_row_slot, int64_t n_send, int32_t* send_ids,
                            float* send_w, void* stream) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  if (experts_per_rank < 1 || n_ranks < 1 || (int64_t)experts_per_rank * n_ranks != p->E || sparse_slots(p))
    return MOE_ERR_INVALID_ARG;
  if (n_send < 0 || n_send > p->T * (int64_t)n_ranks) return MOE_ERR_INVALID_ARG;
  if (n_send > 0 && (!topk_ids || !topk_w || !send_row_slot || !send_ids || !send_w)) return MOE_ERR_INVALID_ARG;
  return launch_ep_send_meta(topk_ids, topk_w, p->k, experts_per_rank, n_ranks, send_row_slot, n_send, send_ids, send_w,
                             (cudaStream_t)stream);
}

moe_status moe_ep_slot_grad(const moe_problem* p, const int32_t* topk_ids, int32_t experts_per_rank, int32_t n_ranks,
                            const int32_t* send_pos, const float* dg_back, const float* dg_local, int32_t self_rank,
                            float* dg, void* stream) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  if (experts_per_rank < 1 || n_ranks < 1 || (int64_t)experts_per_rank * n_ranks != p->E || sparse_slots(p))
    return MOE_ERR_INVALID_ARG;
  if (self_rank < -1 || self_rank >= n_ranks || (self_rank >= 0 && p->T > 0 && !dg_local)) return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && (!topk_ids || !send_pos || !dg)) return MOE_ERR_INVALID_ARG;  // dg_back: NULL iff no slot is remote
  return launch_ep_slot_grad(topk_ids, p->T, p->k, experts_per_rank, n_ranks, send_pos, dg_back, dg_local, self_rank,
                             dg, (cudaStream_t)stream);
}

moe_status moe_gather_rows(const void* src, int64_t n_src, const int32_t* index, int64_t n, int64_t width,
                           int32_t elem_bytes, void* dst, void* stream) {
  if (n < 0 || n_src < 0 || width < 1 || (elem_bytes != 2 && elem_bytes != 4)) return MOE_ERR_INVALID_ARG;
  if (n > 0 && (!src || !dst)) return MOE_ERR_INVALID_ARG;
  if (!index && n > n_src) return MOE_ERR_INVALID_ARG;  // identity copy of the first n rows
  if ((width * elem_bytes) % 4 != 0) return MOE_ERR_MISALIGNED;
  if ((width * elem_bytes) % 16 == 0 && (!aligned16(src) || !aligned16(dst))) return MOE_ERR_MISALIGNED;
  return launch_gather_rows(src, index, n, width * elem_bytes, dst, (cudaStream_t)stream);
}

moe_status moe_combine_rows(const moe_problem* p, const void* rows, const int32_t* token_index_map, const void* base,
                            void* out, void* stream) {
  moe_status s = validate(p);
  if (s != MOE_OK) return s;
  if (p->T > 0 && (!token_index_map || !out)) return MOE_ERR_INVALID_ARG;
  if (p->d % 8 != 0) return MOE_ERR_UNSUPPORTED;
  if (!aligned16(rows) || !aligned16(base) || !aligned16(out)) return MOE_ERR_MISALIGNED;
  return launch_combine_rows(p, rows, token_index_map, base, out, (cudaStream_t)stream);
}

}  // extern "C"
