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
};

moe_status run_gemm(const GemmCall& c, cudaStream_t st);
int gemm_dg_parts(const GemmCall& c);  // dg partial columns per row written by BWD_DH

}  // namespace moeb
