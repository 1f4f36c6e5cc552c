// gemm.h — the six expert GEMMs of the MoE layer behind one call descriptor.
// bf16 runs on the tcgen05/TMEM/TMA kernels (gemm_tc.cu); fp32 storage mode
// runs on the CUDA-core kernels (gemm_simt.cu), which keep true fp32 math.
#pragma once
#include "common.cuh"

namespace moeb {

enum GemmWhich { GEMM_FWD_UP = 0, GEMM_FWD_DOWN = 1, GEMM_BWD_DH = 2, GEMM_BWD_DX = 3, GEMM_DW3 = 4, GEMM_DW12 = 5 };

struct GemmCall {
  int which;
  const void *x, *dy, *w1, *w2, *w3;
  const float* topw;
  const int32_t *offs, *eti, *row_slot;
  void *a_save, *b_save, *u;
  float* acc_out;
  float* dg_part;
  void *dw_a, *dw_b;
  int64_t T, R;
  int d, h, E;
  bool bf16;
  int act;  // MOE_ACT_*: 0 = SwiGLU (gated), 1 = SiLU, 2 = ReLU (non-gated)
  int out_mode;   // FWD_DOWN / BWD_DX epilogue target, OutMode
  void* out_tok;  // OUT_TOKN: [T, d] output in the run dtype
  bool u_weighted;  // MOE_CKPT_ABU: FWD_UP writes wU = w * U, FWD_DOWN then adds wU W3 (unit weight)
  bool dh_skip_u;   // MOE_CKPT_ABU: BWD_DH does not write wU (the saved one is read by DW3)
  int* sched;       // 4 claim counters of the tile scheduler (in the caller's ws; zeroed per launch)
  // FWD_UP / FWD_DOWN only (bf16, CTA-pair engine: tc_splits_rows()): split_half 1 = each
  // expert's rows [offs[e], row_split[e]), 2 = [row_split[e], offs[e+1]); NULL = all rows
  const int32_t* row_split;
  int split_half;
  int sm_reserve;  // SMs the launch leaves free for a concurrent exchange kernel (0 = none)
};

// Where FWD_DOWN / BWD_DX put a routed row's result v (row r, token t = eti[r]):
//   OUT_RED  acc_out[t] += v    fp32 [T,d], red.add (default combine)
//   OUT_ROWS acc_out[r]  = v    fp32 [R,d], ordered token-side sum later (NEXT-4)
//   OUT_TOK  acc_out[t]  = v    fp32 [T,d], k = 1 (one row per token)
//   OUT_TOKN out_tok[t]  = dtype(v), k = 1 with nothing left to add
enum OutMode { OUT_RED = 0, OUT_ROWS = 1, OUT_TOK = 2, OUT_TOKN = 3 };

// non-gated activation sigma and its derivative
__device__ __forceinline__ float act_fwd(int act, float a, float sg) { return act == 2 ? fmaxf(a, 0.f) : a * sg; }
__device__ __forceinline__ float act_grad(int act, float a, float sg) {
  return act == 2 ? (a > 0.f ? 1.f : 0.f) : sg * (1.f + a * (1.f - sg));
}

moe_status run_gemm(const GemmCall& c, cudaStream_t st);
bool tc_splits_rows();                   // FWD_UP / FWD_DOWN honour GemmCall.row_split
// die of every SM of the current device, measured once (topology.cu); device
// array indexed by %smid, n_sm = SMs per die (n_sm[1] == 0: no split)
const uint8_t* sm_die_map(int n_sm[2]);
int gemm_dg_parts(const GemmCall& c);  // dg partial columns per row written by BWD_DH

}  // namespace moeb
