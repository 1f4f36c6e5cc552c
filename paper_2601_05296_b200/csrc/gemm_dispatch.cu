// gemm_dispatch.cu — routes each expert GEMM to its kernel family.
#include "gemm.h"

namespace moeb {

moe_status simt_gemm(const GemmCall& c, cudaStream_t st);
int simt_dg_parts(int h);
moe_status tc_gemm(const GemmCall& c, cudaStream_t st);
int tc_dg_parts(int h);

int gemm_dg_parts(const GemmCall& c) { return c.bf16 ? tc_dg_parts(c.h) : simt_dg_parts(c.h); }

moe_status run_gemm(const GemmCall& c, cudaStream_t st) {
  return c.bf16 ? tc_gemm(c, st) : simt_gemm(c, st);
}

}  // namespace moeb
