/*
 * moeblaze.h — C ABI of the B200 (sm_100a) MoEBlaze hot path.
 *
 * The operation is one dropless top-k SwiGLU Mixture-of-Experts layer,
 * forward and backward, computed MoEBlaze-style: no routed-token buffer and
 * no padded per-expert buffer ever exists; experts gather token rows through
 * compact index structures and reduce their outputs back by index.
 * Citations "P:n" are lines of the paper text (arXiv 2601.05296, PAPER.md).
 *
 * Problem statement (Alg. 1):
 *   X   [T, d]      tokens ("x in R^{L x d}", L = T)
 *   W_g [E, d]      router, logits = X W_g^T (no bias)
 *   w1, w2 [E, h, d]  SwiGLU gate (SiLU) and up projections, nn.Linear (out,in)
 *                    layout: the paper's W1_e = w1[e]^T, W2_e = w2[e]^T
 *   w3  [E, d, h]   down projection, W3_e = w3[e]^T
 *   y_t = sum_j w[t,j] * ( SiLU(x_t W1_e) * (x_t W2_e) ) W3_e,  e = ids[t,j]
 *
 * Conventions common to every entry point
 *  - All tensor pointers are DEVICE pointers to dense row-major arrays owned by
 *    the caller.  The library never allocates device memory and keeps no
 *    per-call state; scratch comes from the caller's `ws` (size from
 *    moe_workspace_size).  Pointers must be 16-byte aligned.
 *  - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t
 *    passed as void*; NULL = legacy default stream).  No call synchronises the
 *    host: per-expert sizes are read on the device.
 *  - dtype MOE_BF16: X, W*, A/B checkpoints, Y and all gradients are bf16;
 *    logits, topk_w, d_topk_w are fp32; accumulation is fp32 (tcgen05 TMEM).
 *    dtype MOE_FP32: every tensor is fp32 and the arithmetic is true fp32
 *    (CUDA-core FMA, no TF32).
 *  - Argument errors are returned synchronously and nothing is launched:
 *    MOE_ERR_INVALID_ARG (null pointer, bad shape: T < 0, d/h/E/k < 1, E > 256,
 *    T*k >= 2^31; with every slot routed (rows = 0) also k > E or k > 16; with
 *    sparse slots (rows > 0) k <= 256 and k > E is valid, since empty slots are
 *    -1), MOE_ERR_UNSUPPORTED (bf16 with d or h not
 *    a multiple of 128, fp32 with d not a multiple of 8), MOE_ERR_MISALIGNED,
 *    MOE_ERR_WORKSPACE (ws too small).  Launch failures return MOE_ERR_CUDA.
 *    The library never aborts the process.
 *  - T = 0 is valid: nothing is launched except zero-fills of outputs.
 */
#ifndef MOEBLAZE_H_
#define MOEBLAZE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MOE_OK = 0,
  MOE_ERR_INVALID_ARG = 1,
  MOE_ERR_UNSUPPORTED = 2,
  MOE_ERR_MISALIGNED = 3,
  MOE_ERR_WORKSPACE = 4,
  MOE_ERR_BAD_ROUTING = 5,
  MOE_ERR_CUDA = 6
} moe_status;

typedef enum { MOE_BF16 = 0, MOE_FP32 = 1 } moe_dtype;

typedef enum { MOE_OP_ROUTE = 0, MOE_OP_DISPATCH = 1, MOE_OP_FFN_FWD = 2, MOE_OP_FFN_BWD = 3,
               MOE_OP_ROUTER_BWD = 4 } moe_op;

typedef struct {
  int64_t T;              /* tokens in the step (paper's L) */
  int32_t d;              /* model dim */
  int32_t h;              /* FFN hidden dim (d_ff) */
  int32_t E;              /* experts, 1..256 */
  int32_t k;              /* experts per token, 1..min(E,16) */
  int32_t dtype;          /* moe_dtype */
  int32_t renormalize;    /* 0: w = softmax over all E, then pick (paper default);
                             1: w renormalised over the k picked experts (Mixtral) */
  int32_t check_routing;  /* 1: moe_dispatch_build validates ids (range, per-token
                             uniqueness) and records violations in the device status
                             word at ws offset 0 (int32; 0 = ok, else MOE_ERR_BAD_ROUTING) */
  int32_t checkpoint;     /* activation-checkpoint policy:
                             MOE_CKPT_AB (0, default) = the paper's smart checkpoint: save
                             the pre-activations A, B, recompute SiLU in backward;
                             MOE_CKPT_NONE (1) = save nothing but X and the routing: A, B
                             live in ws during moe_ffn_fwd (a_save/b_save may be NULL) and
                             moe_ffn_bwd recomputes them with the fused up-projection into
                             the caller's a_save/b_save, which are then scratch [R, h]
                             buffers (+4 T*k*d*h flops; results bit-identical to MOE_CKPT_AB);
                             MOE_CKPT_ABU (2) = Alg. 1 literally ("Store A, B, Y_swi"):
                             A, B and the gate-weighted activation wU_r = w_r SiLU(A_r) B_r
                             are saved (u_save [R, h]); the down projection consumes wU
                             (y += wU W3, the same sum as w (U W3)), the dW3 GEMM reads the
                             saved wU and the dH GEMM no longer writes it (+R*h
                             saved elements, -R*h written in backward) */
  int32_t activation;     /* expert FFN: MOE_ACT_SWIGLU (0, default) =
                             SiLU(x W1) * (x W2) W3; MOE_ACT_SILU (1) / MOE_ACT_RELU (2)
                             = the non-gated expert W2 sigma(W1 x) of P:75 (the paper's SiLU /
                             ReLU experiments): uses w1 and w3 only; w2, b_save and
                             dw2 are unused (may be NULL); A alone is checkpointed */
  int32_t deterministic;  /* combine of the k expert outputs of a token (SURVEY §8(f) NEXT-4,
                             P:111 vs P:134): 0 (default) = fused red.add of w*O into an fp32
                             [T,d] accumulator in the down-GEMM epilogue (bitwise reproducible
                             for k <= 2, order-dependent in the last bit for k >= 3);
                             1 = ordered: the epilogue stores each routed row's fp32 result at
                             its expert-sorted row index ([T*k, d] fp32 transient ws) and a
                             token-side pass sums a token's rows in slot order j = 0..k-1
                             through token_index_map (bitwise reproducible for every k; for
                             k <= 2 bit-identical to mode 0).  Applies to y and dx.  k = 1
                             ignores it: each token has one row, stored directly. */
  int64_t rows;           /* routed (token, expert) rows R.  0 (default): R = T*k, every slot of
                             topk_ids holds an expert id.  > 0: "sparse slots" -- topk_ids entries
                             equal to -1 are empty slots (no expert), skipped by the dispatch
                             (token_index_map = -1 there, d_topk_w = 0), and rows is the
                             number of non-empty slots or any upper bound on it: buffers and
                             workspace are sized for `rows` (a_save/b_save hold rows rows), the
                             kernels take the actual count from expert_offsets[E] on the
                             device.  Used by the expert-parallel receiver, whose received
                             token rows carry only the slots of this rank's experts (SURVEY
                             §8(f) NEXT-1 dedup); the peer-memory exchange, which never reads
                             counts on the host, passes the worst case.
                             0 <= rows <= T*k. */
} moe_problem;

enum { MOE_CKPT_AB = 0, MOE_CKPT_NONE = 1, MOE_CKPT_ABU = 2 };
enum { MOE_ACT_SWIGLU = 0, MOE_ACT_SILU = 1, MOE_ACT_RELU = 2 };

/* The compact dispatch index structures of §4.1.  R = T*k (or
 * p->rows with sparse slots; token_index_map is then -1 at empty slots).
 *   expert_counts[E]         tokens routed to each expert (expert_lengths)
 *   expert_offsets[E+1]      exclusive prefix sum of counts; offsets[E] = R
 *   expert_token_indices[R]  token ids grouped by expert, ascending inside an
 *                            expert
 *   token_index_map[T*k]     position of (t, ids[t,j]) inside expert_token_indices
 *                            (P:130-135); a permutation of [0, R)
 *   row_slot[R]              inverse of token_index_map: t*k + j for row r
 *   token_expert_indices     == topk_ids [T*k], input only
 * Built by moe_dispatch_build (written), read by moe_ffn_fwd/bwd (read only). */
typedef struct {
  int32_t* expert_counts;
  int32_t* expert_offsets;
  int32_t* expert_token_indices;
  int32_t* token_index_map;
  int32_t* row_slot;
  const int32_t* token_expert_indices;
  const int32_t* token_rows;   /* optional device int32 scalar n <= T: token rows [n, T) carry no
                                  routed slot (sparse problems: their topk_ids rows are all -1).
                                  moe_ffn_fwd/bwd then zero and finalise the fp32 combine
                                  accumulator for rows < n only, and leave y / dx rows >= n
                                  unspecified.  NULL: n = T.  Not read by moe_dispatch_build.
                                  Set by the peer-memory EP receiver (moe_ep_recv_prepare). */
} moe_dispatch;

/* Router backward inputs/outputs for moe_ffn_bwd (not in the paper: the
 * derivative of P:42/P:91 through softmax; reading #14). */
typedef struct {
  const void* w_gate;     /* [E, d] dtype */
  const float* logits;    /* [T, E] fp32, as written by moe_route */
  const int32_t* topk_ids;/* [T, k] */
  void* dw_gate;          /* [E, d] dtype, written */
} moe_router_bwd;

/* Bytes of device scratch `ws` that `op` needs for problem `p` (closed form;
 * with deterministic = 0 it has no T*k*d term: no routed-token buffer exists;
 * deterministic = 1 adds the transient [T*k, d] fp32 row-result buffer).  The
 * first 256 bytes of the FFN workspaces hold the expert GEMMs' tile-scheduler
 * claim counters (zeroed on the stream by every call that uses them). */
moe_status moe_workspace_size(const moe_problem* p, moe_op op, size_t* bytes);

/* Gating.  logits = X W_g^T accumulated in fp32; ids[t,:] = the k
 * largest logits in descending order, exact ties -> lower expert id;
 * topk_w[t,j] = softmax(logits[t,:])[ids[t,j]] (renormalised over the k
 * picked experts if p->renormalize).
 *   x [T,d] dtype, w_gate [E,d] dtype -> logits [T,E] fp32, topk_ids [T,k]
 *   int32, topk_w [T,k] fp32.  ws may be NULL (needs 0 bytes). */
moe_status moe_route(const moe_problem* p, const void* x, const void* w_gate,
                     float* logits, int32_t* topk_ids, float* topk_w,
                     void* ws, size_t ws_bytes, void* stream);

/* Buffer-free dispatch construction (§4.2): from topk_ids [T,k]
 * build counts, offsets, expert_token_indices, token_index_map and row_slot
 * in `out` (all device arrays, written).  Atomic-free and deterministic:
 * results are bit-identical to a stable sort of (expert, token) pairs.
 * Two launches: per-tile histogram, then scan + scatter. */
moe_status moe_dispatch_build(const moe_problem* p, const int32_t* topk_ids, const moe_dispatch* out,
                              void* ws, size_t ws_bytes, void* stream);

/* Expert forward (§3.1, Alg. 1 FusedForward P:221-233):
 *   for each expert e and row r in [offsets[e], offsets[e+1]), t = eti[r]:
 *     A_r = X[t] W1_e,  B_r = X[t] W2_e   (X rows gathered through eti, never copied)
 *     U_r = SiLU(A_r) * B_r               (transient, in ws)
 *     y[t] += topk_w[row_slot[r]] * (U_r W3_e)     (combine fused into the down GEMM)
 *   a_save, b_save [T*k, h] dtype: the checkpointed pre-activations A, B in
 *   expert-sorted row order, written (ignored, may be NULL,
 *   under MOE_CKPT_NONE).  u_save [T*k, h] dtype: MOE_CKPT_ABU only (else
 *   ignored, may be NULL): the saved wU_r = topk_w[row_slot[r]] * U_r, written.
 *   y [T,d] dtype, written. */
moe_status moe_ffn_fwd(const moe_problem* p, const void* x, const void* w1, const void* w2,
                       const void* w3, const float* topk_w, const moe_dispatch* disp,
                       void* a_save, void* b_save, void* u_save, void* y,
                       void* ws, size_t ws_bytes, void* stream);

/* moe_ffn_fwd with the exchanges of an expert-parallel receiver overlapped
 * (SURVEY §8(f) NEXT-1): its token rows are [t_ready local | received], the
 * received rows' x arrives from the all-to-all (C2) and their y goes back by
 * another (C3).  Token rows [0, t_ready) of x are ready at the call; the rows
 * from t_ready on only once sync->x_ready (a cudaEvent_t) has fired.  Each
 * expert's rows [offsets[e], row_split[e]) are those whose token is < t_ready
 * (ascending inside an expert, so they come first).  Launch order:
 *   up-projection of the rows before row_split; wait x_ready; up-projection
 *   of the rest; then, with y_ready set (bf16, red.add combine): down-
 *   projection of the rows from row_split on, y rows
 *   [t_ready, T) finalised, y_ready recorded, down-projection of the rows
 *   before row_split leaving sm_reserve SMs free (for the C3 exchange kernel),
 *   y rows [0, t_ready) finalised; without y_ready: one down-projection and
 *   one finalise (y_ready, if set, recorded at the end).
 * A, B, U and y are the same as one moe_ffn_fwd call (every row is computed
 * by the same tile arithmetic; the red.add combine of a token's rows runs in
 * one launch either way).  sync NULL, or row_split NULL: exactly moe_ffn_fwd
 * (x_ready, if set, waited first; y_ready recorded at the end).  fp32 runs
 * (CUDA-core path) do not split. */
typedef struct {
  const int32_t* row_split;  /* [E] device, from moe_dispatch_row_split(t_ready) */
  void* x_ready;             /* cudaEvent_t or NULL */
  void* y_ready;             /* cudaEvent_t or NULL, recorded (see above) */
  int64_t t_ready;           /* the split token row (as given to moe_dispatch_row_split) */
  int32_t sm_reserve;        /* SMs left free by the launches after y_ready; 0 = none */
} moe_fwd_sync;

moe_status moe_ffn_fwd_ex(const moe_problem* p, const void* x, const void* w1, const void* w2,
                          const void* w3, const float* topk_w, const moe_dispatch* disp,
                          void* a_save, void* b_save, void* u_save, void* y, const moe_fwd_sync* sync,
                          void* ws, size_t ws_bytes, void* stream);

/* row_split[e] = offsets[e] + #{r in [offsets[e], offsets[e+1]) : eti[r] < t_ready}
 * (a binary search per expert: eti is ascending inside an expert).
 * row_split [E] int32 device, written; one launch.  0 <= t_ready <= p->T. */
moe_status moe_dispatch_row_split(const moe_problem* p, const moe_dispatch* disp, int64_t t_ready,
                                  int32_t* row_split, void* stream);

/* Expert backward (§3.2, Alg. 1 FusedBackward P:236-253) with the
 * SiLU recomputed from the checkpoint:
 *   dH_r = dy[eti[r]] W3_e^T;  d_topk_w[t,j] = <dH_r, U_r>
 *   dw3[e] = sum_r (w_r U_r)^T dy[eti[r]]
 *   dA_r = w_r dH_r * B_r * SiLU'(A_r);  dB_r = w_r dH_r * SiLU(A_r)
 *   dw1[e] = sum_r dA_r^T X[eti[r]],  dw2[e] = sum_r dB_r^T X[eti[r]]
 *   dx[t]  = sum_{r: eti[r]=t} (dA_r W1_e^T + dB_r W2_e^T)  [+ router path]
 * a_save/b_save are read (A, B) and OVERWRITTEN with dA, dB (in place); under
 * MOE_CKPT_NONE they are caller-provided scratch [R, h] buffers (contents on
 * entry ignored) that the recomputed A, B, then dA, dB occupy.  u_save
 * (MOE_CKPT_ABU only, else ignored) is the saved wU, read by the dW3 GEMM.
 * dw1/dw2/dw3 are written (experts with no rows get zeros), not accumulated.
 * d_topk_w [T,k] fp32 may be NULL only if router is NULL.
 * router != NULL: also computes the router backward (renorm-aware) and adds
 * dlogits W_g into dx; router->dw_gate is written.
 *
 * Stages (sync->stages; 0 or NULL sync = all, in the order below).  The three
 * stages may be issued as separate calls with the SAME ws (its contents carry
 * wU and the tile counters from one stage to the next), so that a caller can
 * allocate each weight gradient only when its GEMM runs and release A/B
 * (then dA/dB) as soon as the last GEMM that reads them is done:
 *   MOE_BWD_DATA: dH GEMM (dA, dB in place, wU into ws unless ABU, gate-grad
 *                 partials) -> d_topk_w -> dX GEMM -> router backward / dx
 *                 finalise [-> sync->dx_ready recorded].  Needs dy, x (router
 *                 or recompute), w1..w3, dx, d_topk_w; dw1..dw3 may be NULL.
 *   MOE_BWD_DW3:  dW3 = dy^T wU.  Needs dy and dw3; reads wU (ws or u_save).
 *   MOE_BWD_DW12: [dW1; dW2] = [dA | dB]^T x (the only kernel after the
 *                 optional recompute that reads x: [sync->x_ready waited]).
 * In one call the order is DATA -> DW3 -> DW12 (x_ready lets an expert-parallel
 * receiver overlap the arrival of x with everything before DW12). */
enum { MOE_BWD_DATA = 1, MOE_BWD_DW3 = 2, MOE_BWD_DW12 = 4, MOE_BWD_ALL = 7 };
typedef struct {
  void* x_ready;   /* cudaEvent_t or NULL: the stream waits on it (cudaStreamWaitEvent) before
                      the first kernel that reads x after the dX GEMM (the dW1/dW2 GEMM, and
                      the router's dW_g when router != NULL); lets an expert-parallel
                      receiver overlap the arrival of x with the dH / dX GEMMs.  With
                      MOE_CKPT_NONE x is read at the start (recompute), so x must be ready
                      before the call. */
  void* dx_ready;  /* cudaEvent_t or NULL: recorded once dx and d_topk_w are final, before the
                      weight-gradient GEMMs; lets the caller return dx rows while dW1..3 run. */
  int32_t stages;  /* MOE_BWD_* mask; 0 = MOE_BWD_ALL */
} moe_bwd_sync;

moe_status moe_ffn_bwd(const moe_problem* p, const void* dy, const void* x, const void* w1,
                       const void* w2, const void* w3, const float* topk_w,
                       const moe_dispatch* disp, void* a_save, void* b_save, void* u_save,
                       void* dx, void* dw1, void* dw2, void* dw3, float* d_topk_w,
                       const moe_router_bwd* router, const moe_bwd_sync* sync,
                       void* ws, size_t ws_bytes, void* stream);

/* Router backward on its own (used by the expert-parallel path, where the
 * gate-weight gradient d_topk_w arrives from the expert owners):
 *   dlogits = softmax-Jacobian of the (renormalised) gate weights applied to
 *   d_topk_w [T,k] fp32; router->dw_gate = dlogits^T X (written);
 *   dx = dx_partial + dlogits W_g  (dx_partial, dx: [T,d] dtype; may alias). */
moe_status moe_router_backward(const moe_problem* p, const float* d_topk_w, const void* x,
                               const moe_router_bwd* router, const void* dx_partial, void* dx,
                               void* ws, size_t ws_bytes, void* stream);

/* Expert-parallel helpers (the paper's "future work"; SURVEY §8(e),
 * §8(f) NEXT-1).  P = n_ranks ranks; rank q owns the experts
 * [q*experts_per_rank, (q+1)*experts_per_rank).  A token's row travels ONCE to
 * every rank that owns at least one of its k experts (per-destination dedup),
 * carrying the k slots restricted to that rank; the receiver's expert outputs
 * for the token come back already summed over its experts (one row per
 * (token, rank) pair instead of one per (token, expert) pair).
 *
 * Local pairs never travel: a token's slots owned by its own rank (`self_rank`)
 * are computed where the token lives.  The receiver's problem has the T local
 * tokens first (their own-rank slots, moe_ep_local_slots) and the received rows
 * after them, so the local partial output of token t is row t of its output and
 * is added by moe_combine_rows as `base`.
 *
 * moe_ep_dest: dest[t*P + q] = q if some ids[t, j] is owned by rank q and
 *   q != self_rank, else -1 (self_rank = -1: no rank excluded).
 *   topk_ids [T,k] (p->T, p->k; p->E = global experts) -> dest [T, P] int32.
 *   moe_dispatch_build over dest (T tokens, "k" = E = P, sparse slots, rows =
 *   number of (token, rank) pairs or any upper bound up to T*P) then yields the
 *   send plan: counts[q] rows to rank q, expert_token_indices = the tokens to
 *   send, grouped by rank, ascending (the send order), token_index_map [T,P] =
 *   send position of (t, q) or -1, row_slot = t*P + q.
 * moe_ep_local_slots: local_ids[t*k + j] = ids[t,j] - rank*experts_per_rank if
 *   rank owns ids[t,j] else -1; local_w[t*k + j] = topk_w[t,j] there, else 0:
 *   the sparse topk_ids / topk_w of the local tokens on their own rank.
 * moe_ep_send_meta: for send row i < n_send (send_row_slot = that row_slot):
 *   send_ids[i*k + j] = ids[t,j] - q*experts_per_rank if rank q owns ids[t,j]
 *   else -1, send_w[i*k + j] = topk_w[t,j] (0 for -1): the receiver's sparse
 *   topk_ids / topk_w.
 * moe_ep_slot_grad: dg[t*k + j] = dg_local[t*k + j] if self_rank owns ids[t,j],
 *   else dg_back[send_pos[t*P + q]*k + j] with q the owner of ids[t,j]: the
 *   gate-weight gradients computed locally and returned by the owners, in
 *   (token, slot) order.  dg_back [n_send, k] fp32 (may be NULL when no slot is
 *   remote); dg_local [T, k] fp32 (ignored when self_rank = -1).
 * moe_gather_rows: dst[i, :] = src[index[i], :] for i < n (rows of `width`
 *   elements of `elem_bytes` in {2,4}; row bytes a multiple of 4); builds the
 *   all-to-all send buffer in send order.  index entries must be in [0, n_src).
 *   index = NULL: dst[i, :] = src[i, :] (n <= n_src), a copy done by a kernel:
 *   dst may be pinned host memory (UVA-mapped), which the kernel writes over
 *   PCIe without queueing behind the copy engines' bulk transfers (the EP
 *   split-size read uses it while the host pipeline streams activations).
 * moe_combine_rows: out[t, :] = base[t, :] + sum_{j<k, tim[t*k+j] >= 0}
 *   rows[tim[t*k+j], :] (base [T, d] optional, NULL = 0; fixed j order, fp32
 *   accumulation, dtype output; -1 entries skipped; rows may be NULL only if
 *   every entry is -1; d % 8 == 0): the token-side combine of returned rows
 *   through token_index_map ("gather its k expert outputs"); with the
 *   send plan (k = P) it sums a token's per-rank partial outputs. */
moe_status moe_ep_dest(const moe_problem* p, const int32_t* topk_ids, int32_t experts_per_rank,
                       int32_t n_ranks, int32_t self_rank, int32_t* dest, void* stream);
moe_status moe_ep_local_slots(const moe_problem* p, const int32_t* topk_ids, const float* topk_w,
                              int32_t experts_per_rank, int32_t rank, int32_t* local_ids, float* local_w,
                              void* stream);
moe_status moe_ep_send_meta(const moe_problem* p, const int32_t* topk_ids, const float* topk_w,
                            int32_t experts_per_rank, int32_t n_ranks, const int32_t* send_row_slot,
                            int64_t n_send, int32_t* send_ids, float* send_w, void* stream);
moe_status moe_ep_slot_grad(const moe_problem* p, const int32_t* topk_ids, int32_t experts_per_rank,
                            int32_t n_ranks, const int32_t* send_pos, const float* dg_back,
                            const float* dg_local, int32_t self_rank, float* dg, void* stream);
moe_status moe_gather_rows(const void* src, int64_t n_src, const int32_t* index, int64_t n,
                           int64_t width, int32_t elem_bytes, void* dst, void* stream);
moe_status moe_combine_rows(const moe_problem* p, const void* rows, const int32_t* token_index_map,
                            const void* base, void* out, void* stream);

/* Device-initiated expert-parallel exchange over peer memory (SURVEY §8(f)
 * NEXT-1: "no host sync in the EP step"; the paper names distribution as
 * future work).  The NCCL path above sizes its all-to-all buffers from
 * ONE device->host read of the split sizes per step.  This path has none: every
 * rank owns a "symmetric" set of receive buffers (same layout on every rank,
 * mapped into every peer's address space by the caller -- CUDA IPC over
 * NVLink/NVSwitch), sized for the worst case (P*T token rows), and the kernels
 * below move rows with plain loads/stores into / out of peer memory; ordering
 * between ranks is carried by epoch flags in peer memory, never by the host.
 *
 * Flags: flags[phase * P + s] (uint64, zero-initialised, written only by rank
 * s) = the last epoch in which rank s completed `phase` towards this rank.  A
 * signal is a release store at system scope after a system-scope fence (so
 * every write that precedes it in stream order -- including the remote row
 * stores of a push -- is visible first); a wait is an acquire-load spin on the
 * local flags of every rank, bounded by `timeout_ns`: on expiry it records
 * 1 + phase in *status (first failure wins) and returns, so a lost peer costs
 * a wrong result the caller detects through `status`, never a hung GPU.
 * Epochs must increase by one per step and be the same on every rank.
 * cmat[s * P + q] = rows rank s sends to rank q in the current step (every
 * rank's row, written by moe_ep_publish_counts into every peer).
 * The receive-side row layout is the NCCL path's: row r < T is the local token
 * r; the rows from rank s start at T + sum_{s' < s} cmat[s' * P + me].
 *
 * All pointers are device pointers except the moe_ep_peers struct itself
 * (host).  peer_* arrays are device arrays of P device pointers, entry q =
 * rank q's buffer as mapped in this process (entry `rank` = the local buffer).
 * Errors: MOE_ERR_INVALID_ARG for null/inconsistent arguments, MOE_ERR_CUDA on
 * launch failure.  Not graph-capturable across steps (the epoch is an argument). */
enum { MOE_EP_PH_ENTER = 0, MOE_EP_PH_COUNTS = 1, MOE_EP_PH_ROWS = 2, MOE_EP_PH_Y = 3, MOE_EP_PH_DY = 4,
       MOE_EP_PH_DX = 5, MOE_EP_PH_DWG = 6, MOE_EP_NPHASE = 7 };

typedef struct {
  int32_t n_ranks;             /* P >= 1 */
  int32_t rank;                /* this rank, 0 <= rank < P */
  uint64_t* const* peer_flags; /* [P] -> each rank's flags [MOE_EP_NPHASE * P] (entry rank = local) */
  int32_t* const* peer_cmat;   /* [P] -> each rank's cmat [P * P] */
  uint32_t* arrive;            /* local [MOE_EP_NPHASE] zero-initialised counters (last-CTA signal) */
  int32_t* status;             /* local int32, 0 = ok; 1 + phase of the first wait that timed out */
  int64_t timeout_ns;          /* per wait; <= 0: 30 s */
} moe_ep_peers;

/* Signal `phase` of `epoch` to every rank (itself included) after all prior
 * work on the stream. */
moe_status moe_ep_signal(const moe_ep_peers* g, int32_t phase, uint64_t epoch, void* stream);
/* Block the stream until every rank has signalled `phase` of `epoch` here. */
moe_status moe_ep_wait(const moe_ep_peers* g, int32_t phase, uint64_t epoch, void* stream);
/* counts [P] (rows this rank sends to each rank) -> row `rank` of every rank's
 * cmat; then signals MOE_EP_PH_COUNTS. */
moe_status moe_ep_publish_counts(const moe_ep_peers* g, const int32_t* counts, uint64_t epoch, void* stream);
/* Fused gather + exchange: for every send position i < send_offs[P], with q
 * the rank whose segment [send_offs[q], send_offs[q+1]) holds i,
 *   peer_dst[q] row (dst_row0 + sum_{s<rank} cmat[s*P+q] + i - send_offs[q])
 *     = src row (index ? index[i] : i)
 * (rows of row_bytes bytes, a multiple of 4; 16-byte rows move as uint4).
 * send_offs [P+1] (the send plan's expert_offsets), index = the send order
 * (its expert_token_indices).  n_max >= send_offs[P] bounds the grid.  Reads
 * the local cmat, so it must follow moe_ep_wait(MOE_EP_PH_COUNTS).  phase >= 0:
 * the last CTA signals `phase` to every rank once all rows are stored; < 0:
 * no signal (a later push's signal covers this one). */
moe_status moe_ep_push_rows(const moe_ep_peers* g, const void* src, const int32_t* index, const int32_t* send_offs,
                            int64_t n_max, int64_t row_bytes, int64_t dst_row0, void* const* peer_dst,
                            int32_t phase, uint64_t epoch, void* stream);
/* Receiver slots after moe_ep_wait(MOE_EP_PH_ROWS): rows [T, T+U) of ids [T_cap, k]
 * hold the senders' GLOBAL expert ids; rewrite them to local ids
 * (id - rank*experts_per_rank where owned, else -1, w = 0 there) and set rows
 * [T+U, T_cap) to -1 (U = sum_s cmat[s*P+rank]), so moe_dispatch_build over the
 * T_cap rows (sparse slots, rows = any upper bound) sees exactly the received
 * (token, local expert) pairs.  token_rows (optional, device int32) receives
 * T + U, the moe_dispatch.token_rows bound of the receiver's problem. */
moe_status moe_ep_recv_prepare(const moe_ep_peers* g, int64_t T, int64_t T_cap, int32_t k, int32_t experts_per_rank,
                               int32_t* ids, float* w, int32_t* token_rows, void* stream);
/* Fused exchange + combine: out[t] = base[t] + sum_{q != rank, send_pos[t*P+q] >= 0}
 *   peer_rows[q] row (row0 + sum_{s<rank} cmat[s*P+q] + send_pos[t*P+q] - send_offs[q])
 * (q ascending, fp32 accumulation, p->dtype rows of p->d, d % 8 == 0; p->T = T
 * tokens).  send_pos = the send plan's token_index_map [T, P].  Must follow
 * moe_ep_wait on the phase that published peer_rows. */
moe_status moe_ep_pull_combine(const moe_ep_peers* g, const moe_problem* p, const void* const* peer_rows,
                               int64_t row0, const int32_t* send_offs, const int32_t* send_pos, const void* base,
                               void* out, void* stream);
/* dg[t*k+j] = dg_local[t*k+j] if this rank owns ids[t,j], else
 *   peer_dg[q][(row0 + sum_{s<rank} cmat[s*P+q] + send_pos[t*P+q] - send_offs[q]) * k + j]
 * with q the owner (p->T, p->k, p->E = global experts). */
moe_status moe_ep_pull_slot_grad(const moe_ep_peers* g, const moe_problem* p, int32_t experts_per_rank,
                                 const int32_t* topk_ids, const float* const* peer_dg, int64_t row0,
                                 const int32_t* send_offs, const int32_t* send_pos, const float* dg_local, float* dg,
                                 void* stream);
/* out[i] = sum_{q = 0..P-1} peer_src[q][i], i < n, fp32 accumulation in rank
 * order (bitwise identical on every rank), dtype elements: the all-reduce of
 * the replicated router's gradient. */
moe_status moe_ep_pull_sum(const moe_ep_peers* g, const void* const* peer_src, int64_t n, int32_t dtype, void* out,
                           void* stream);
/* Mapping the symmetric buffers (host calls, synchronous, once per layer).
 * moe_ep_ipc_handle: the CUDA IPC handle (64 bytes into handle_out) of the
 * device allocation containing `ptr` and ptr's byte offset inside it (the
 * buffer may be a sub-allocation of a caching allocator; not for VMM /
 * expandable-segment memory).  moe_ep_ipc_open: map a peer's handle into the
 * CURRENT device's address space (peer access enabled lazily over NVLink;
 * works as well for another process on the same GPU) and return base + offset
 * in *ptr_out, *base_out the mapping to pass to moe_ep_ipc_close. */
moe_status moe_ep_ipc_handle(const void* ptr, void* handle_out, int64_t* offset_out);
moe_status moe_ep_ipc_open(const void* handle, int64_t offset, void** ptr_out, void** base_out);
moe_status moe_ep_ipc_close(void* base);

/* Bench instrumentation.  While enabled, every expert-GEMM launch is
 * bracketed by two CUDA events recorded on the launch stream.
 * moe_profile_read returns, for one GEMM kind (0 FWD_UP: A,B = X W1, X W2 +
 * SwiGLU; 1 FWD_DOWN: U W3 + combine; 2 BWD_DH: dY W3^T + SwiGLU bwd;
 * 3 BWD_DX: [dA|dB][W1;W2]; 4 DW3; 5 DW12), the summed event time in ms and
 * the number of launches since the last reset (it waits for those events).
 * Not thread-safe; off by default. */
moe_status moe_profile_enable(int32_t on);
moe_status moe_profile_reset(void);
moe_status moe_profile_read(int32_t kind, double* total_ms, int64_t* launches);
/* The same for the non-GEMM steps, by name: "route", "dispatch", "zero_acc"
 * (the fp32 combine accumulators' zeroing), "combine" (Y = dtype(Y_acc)),
 * "dg_reduce", "router_bwd" (dlogits + dW_g), "finalize_dx" (dX = dtype(dX_acc
 * + dlogits W_g)).  Unknown names read 0 launches. */
moe_status moe_profile_read_named(const char* name, double* total_ms, int64_t* launches);

/* SM topology used by the expert GEMMs' tile scheduler (not a step of the
 * method; a B200 placement detail).  A B200 is two dies whose
 * L2s each cache lines of both dies' HBM, so CTAs on different dies reading
 * the same operand tile fetch it twice.  The library measures once per device
 * which die each SM is on (DRAM latency classes of cold lines, topology.cu)
 * and splits every expert's n-tiles between the dies.  die_of_sm[s] (host
 * array of max_sm entries) receives 0 or 1 for SM id s, -1 for an SM the
 * probe did not reach; n_per_die[0..1] the SM counts (n_per_die[1] == 0: no
 * split, e.g. MOEBLAZE_DIE=0 or an ambiguous measurement).  Results of every
 * call are independent of this map.  Runs the probe on first use (about a
 * millisecond, synchronous); MOE_ERR_INVALID_ARG on null pointers. */
moe_status moe_sm_topology(int32_t* die_of_sm, int32_t max_sm, int32_t* n_per_die);

/* Human-readable status. */
const char* moe_status_string(moe_status s);

/* Number of CUDA kernels this library has launched since load (monotonic;
 * used by the bench to report its own launches). */
uint64_t moe_launch_count(void);

/* Library version (major*10000 + minor*100 + patch). */
int32_t moe_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MOEBLAZE_H_ */
