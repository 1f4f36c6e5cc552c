// gemm_dispatch.cu — routes each expert GEMM to its kernel family, and the
// optional per-launch CUDA-event instrumentation used by bench.py.
#include <string.h>

#include <vector>

#include "gemm.h"

namespace moeb {

moe_status simt_gemm(const GemmCall& c, cudaStream_t st);
int simt_dg_parts(int h);
moe_status tc_gemm(const GemmCall& c, cudaStream_t st);
int tc_dg_parts(int h, int d);

int gemm_dg_parts(const GemmCall& c) { return c.bf16 ? tc_dg_parts(c.h, c.d) : simt_dg_parts(c.h); }

namespace {
struct ProfRec { int kind; cudaEvent_t a, b; const char* name; };  // kind -1: a named scope
bool g_prof = false;
std::vector<ProfRec> g_recs;
std::vector<cudaEvent_t> g_pool;
cudaEvent_t take_event() {
  if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

moe_status run_gemm(const GemmCall& c, cudaStream_t st) {
  if (!g_prof) return c.bf16 ? tc_gemm(c, st) : simt_gemm(c, st);
  ProfRec r{c.which, take_event(), take_event(), nullptr};
  cudaEventRecord(r.a, st);
  moe_status s = c.bf16 ? tc_gemm(c, st) : simt_gemm(c, st);
  cudaEventRecord(r.b, st);
  g_recs.push_back(r);
  return s;
}

ProfScope::ProfScope(const char* n, cudaStream_t s) : name(n), st(s), a(nullptr) {
  if (!g_prof) return;
  a = take_event();
  cudaEventRecord(a, st);
}

ProfScope::~ProfScope() {
  if (!a) return;
  ProfRec r{-1, a, take_event(), name};
  cudaEventRecord(r.b, st);
  g_recs.push_back(r);
}

}  // namespace moeb

using namespace moeb;

extern "C" {

moe_status moe_profile_enable(int32_t on) {
  g_prof = on != 0;
  return MOE_OK;
}

moe_status moe_profile_reset(void) {
  for (auto& r : g_recs) {
    cudaEventSynchronize(r.b);
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
  return MOE_OK;
}

static moe_status sum_records(int32_t kind, const char* name, double* total_ms, int64_t* launches) {
  if (!total_ms || !launches) return MOE_ERR_INVALID_ARG;
  double t = 0;
  int64_t n = 0;
  for (auto& r : g_recs) {
    if (name ? (r.kind != -1 || strcmp(r.name, name) != 0) : r.kind != kind) continue;
    float ms = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess) return MOE_ERR_CUDA;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) return MOE_ERR_CUDA;
    t += ms;
    ++n;
  }
  *total_ms = t;
  *launches = n;
  return MOE_OK;
}

moe_status moe_profile_read(int32_t kind, double* total_ms, int64_t* launches) {
  return sum_records(kind, nullptr, total_ms, launches);
}

moe_status moe_profile_read_named(const char* name, double* total_ms, int64_t* launches) {
  if (!name) return MOE_ERR_INVALID_ARG;
  return sum_records(-1, name, total_ms, launches);
}

}  // extern "C"
