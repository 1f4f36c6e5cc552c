// ep_p2p.cu — device-initiated expert-parallel exchange over peer memory
// (no host sync in the EP step; P:345 names distribution
// as future work).  Contract and memory-ordering rules: include/moeblaze.h,
// "Device-initiated expert-parallel exchange".
//
// Every rank's receive buffers are mapped into every peer (CUDA IPC over
// NVLink / NVSwitch).  Rows move with plain 16-byte loads/stores to peer
// addresses -- the gather of the send rows is fused into the push (no send
// buffer), the combine of returned rows into the pull (no receive buffer on
// the token side).  Cross-rank ordering uses per-(phase, source) epoch flags:
// release stores at system scope after a system-scope fence, acquire-load
// spins bounded by %globaltimer so a lost peer can never hang the GPU.
#include <cuda.h>  // driver types only (cuMemGetAddressRange through the runtime entry point)

#include <string.h>

#include "common.cuh"

namespace moeb {
namespace {

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// flags[phase * P + me] = epoch on every rank (threads of one block stride over q)
__device__ __forceinline__ void signal_peers(const moe_ep_peers& g, int phase, uint64_t epoch) {
  for (int q = threadIdx.x; q < g.n_ranks; q += blockDim.x)
    st_release_sys(g.peer_flags[q] + (int64_t)phase * g.n_ranks + g.rank, epoch);
}

__global__ void ep_signal_kernel(moe_ep_peers g, int phase, uint64_t epoch) {
  __threadfence_system();  // every prior write of this stream (earlier kernels) before the flag
  signal_peers(g, phase, epoch);
}

__global__ void ep_wait_kernel(moe_ep_peers g, int phase, uint64_t epoch) {
  if (*(volatile int32_t*)g.status != 0) return;  // an earlier wait already failed: do not stack timeouts
  const uint64_t* flags = g.peer_flags[g.rank] + (int64_t)phase * g.n_ranks;
  const uint64_t limit = g.timeout_ns > 0 ? (uint64_t)g.timeout_ns : 30000000000ull;
  const uint64_t t0 = global_ns();
  for (int s = threadIdx.x; s < g.n_ranks; s += blockDim.x) {
    while (ld_acquire_sys(flags + s) < epoch) {
      if (global_ns() - t0 > limit) {
        atomicCAS(g.status, 0, 1 + phase);
        break;
      }
      __nanosleep(128);
    }
  }
}

__global__ void ep_publish_counts_kernel(moe_ep_peers g, const int32_t* __restrict__ counts, uint64_t epoch) {
  const int P = g.n_ranks;
  for (int i = threadIdx.x; i < P * P; i += blockDim.x) {
    const int q = i / P, c = i - q * P;
    g.peer_cmat[q][g.rank * P + c] = counts[c];
  }
  __threadfence_system();
  __syncthreads();
  signal_peers(g, MOE_EP_PH_COUNTS, epoch);
}

// per-block prologue shared by the push / pull kernels: s_off[q] = send_offs[q]
// (q <= P) and s_base[q] = row0 + sum_{s < me} cmat[s*P + q], the first row of
// this rank's segment in rank q's receive buffers
__device__ __forceinline__ void load_plan(const moe_ep_peers& g, const int32_t* send_offs, int64_t row0, int* s_off,
                                          int64_t* s_base) {
  const int P = g.n_ranks;
  const int32_t* cmat = g.peer_cmat[g.rank];
  for (int q = threadIdx.x; q <= P; q += blockDim.x) {
    s_off[q] = send_offs[q];
    if (q < P) {
      int64_t b = row0;
      for (int s = 0; s < g.rank; ++s) b += cmat[s * P + q];
      s_base[q] = b;
    }
  }
  __syncthreads();
}

template <typename V>
__global__ void ep_push_rows_kernel(moe_ep_peers g, const V* __restrict__ src, const int32_t* __restrict__ index,
                                    const int32_t* __restrict__ send_offs, int64_t upr, int64_t row0,
                                    void* const* __restrict__ peer_dst, int phase, uint64_t epoch) {
  extern __shared__ int64_t smem_push[];
  const int P = g.n_ranks;
  int64_t* s_base = smem_push;                                   // [P]
  V** s_dst = reinterpret_cast<V**>(smem_push + P);              // [P]
  int* s_off = reinterpret_cast<int*>(smem_push + 2 * P);        // [P + 1]
  for (int q = threadIdx.x; q < P; q += blockDim.x) s_dst[q] = reinterpret_cast<V*>(peer_dst[q]);
  load_plan(g, send_offs, row0, s_off, s_base);
  const int64_t total = (int64_t)s_off[P] * upr;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / upr, c = e - i * upr;
    const int q = find_segment(s_off, P, (int)i);
    const int64_t srow = index ? (int64_t)__ldg(index + i) : i;
    s_dst[q][(s_base[q] + i - s_off[q]) * upr + c] = src[srow * upr + c];
  }
  if (phase < 0) return;
  __threadfence_system();  // this block's remote stores before its arrival
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    last = atomicAdd(g.arrive + phase, 1u) == gridDim.x - 1;
    if (last) {
      g.arrive[phase] = 0;  // ready for the next push of this phase (stream-ordered)
      __threadfence_system();
    }
  }
  __syncthreads();
  if (last) signal_peers(g, phase, epoch);
}

__global__ void ep_recv_prepare_kernel(moe_ep_peers g, int64_t T, int64_t T_cap, int k, int epr,
                                       int32_t* __restrict__ ids, float* __restrict__ w,
                                       int32_t* __restrict__ token_rows) {
  __shared__ int64_t s_u;
  if (threadIdx.x == 0) {
    const int32_t* cmat = g.peer_cmat[g.rank];
    int64_t u = 0;
    for (int s = 0; s < g.n_ranks; ++s) u += cmat[s * g.n_ranks + g.rank];
    s_u = u;
    if (token_rows && blockIdx.x == 0) *token_rows = (int32_t)(T + u);
  }
  __syncthreads();
  const int64_t f0 = T * k, f1 = T_cap * k, fu = (T + s_u) * k;
  const int lo = g.rank * epr;
  for (int64_t f = f0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < f1; f += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = -1;
    if (f < fu) {
      const int32_t e = ids[f];
      v = (e >= lo && e < lo + epr) ? e - lo : -1;
    }
    ids[f] = v;
    if (v < 0) w[f] = 0.f;
  }
}

template <typename T>
__global__ void ep_pull_combine_kernel(moe_ep_peers g, const void* const* __restrict__ peer_rows, int64_t row0,
                                       const int32_t* __restrict__ send_offs, const int32_t* __restrict__ send_pos,
                                       const T* __restrict__ base, int64_t Tn, int d, T* __restrict__ out) {
  extern __shared__ int64_t smem_pull[];
  const int P = g.n_ranks;
  int64_t* s_base = smem_pull;
  const T** s_src = reinterpret_cast<const T**>(smem_pull + P);
  int* s_off = reinterpret_cast<int*>(smem_pull + 2 * P);
  for (int q = threadIdx.x; q < P; q += blockDim.x) s_src[q] = reinterpret_cast<const T*>(peer_rows[q]);
  load_plan(g, send_offs, row0, s_off, s_base);
  const int cpr = d / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Tn * cpr) return;
  const int64_t t = i / cpr;
  const int col = (int)(i - t * cpr) * 8;
  float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (base) load8(base + t * d + col, a);
  for (int q = 0; q < P; ++q) {
    if (q == g.rank) continue;
    const int r = send_pos[t * P + q];
    if (r < 0) continue;
    float v[8];
    load8(s_src[q] + (s_base[q] + r - s_off[q]) * d + col, v);
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] += v[c];
  }
  store8(out + t * d + col, a);
}

__global__ void ep_pull_slot_grad_kernel(moe_ep_peers g, const int32_t* __restrict__ ids, int64_t Tn, int k, int epr,
                                         const float* const* __restrict__ peer_dg, int64_t row0,
                                         const int32_t* __restrict__ send_offs, const int32_t* __restrict__ send_pos,
                                         const float* __restrict__ dg_local, float* __restrict__ dg) {
  extern __shared__ int64_t smem_sg[];
  const int P = g.n_ranks;
  int64_t* s_base = smem_sg;
  int* s_off = reinterpret_cast<int*>(smem_sg + P);
  load_plan(g, send_offs, row0, s_off, s_base);
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= Tn * k) return;
  const int64_t t = f / k;
  const int j = (int)(f - t * k);
  const int q = ids[f] / epr;
  dg[f] = q == g.rank ? dg_local[f]
                      : peer_dg[q][(s_base[q] + send_pos[t * P + q] - s_off[q]) * k + j];
}

template <typename T>
__global__ void ep_pull_sum_kernel(moe_ep_peers g, const void* const* __restrict__ peer_src, int64_t n,
                                   T* __restrict__ out) {
  const int P = g.n_ranks;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int q = 0; q < P; ++q) a += to_f32(reinterpret_cast<const T*>(peer_src[q])[i]);
    out[i] = from_f32<T>(a);
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

moe_status check_peers(const moe_ep_peers* g) {
  if (!g || g->n_ranks < 1 || g->n_ranks > 256 || g->rank < 0 || g->rank >= g->n_ranks || !g->peer_flags ||
      !g->peer_cmat || !g->arrive || !g->status)
    return MOE_ERR_INVALID_ARG;
  return MOE_OK;
}

moe_status launched() { return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA; }

}  // namespace
}  // namespace moeb

using namespace moeb;

extern "C" {

moe_status moe_ep_signal(const moe_ep_peers* g, int32_t phase, uint64_t epoch, void* stream) {
  moe_status s = check_peers(g);
  if (s != MOE_OK) return s;
  if (phase < 0 || phase >= MOE_EP_NPHASE) return MOE_ERR_INVALID_ARG;
  MOE_LAUNCH(ep_signal_kernel, 1, 32, 0, stream, *g, phase, epoch);
  return launched();
}

moe_status moe_ep_wait(const moe_ep_peers* g, int32_t phase, uint64_t epoch, void* stream) {
  moe_status s = check_peers(g);
  if (s != MOE_OK) return s;
  if (phase < 0 || phase >= MOE_EP_NPHASE) return MOE_ERR_INVALID_ARG;
  MOE_LAUNCH(ep_wait_kernel, 1, 32, 0, stream, *g, phase, epoch);
  return launched();
}

moe_status moe_ep_publish_counts(const moe_ep_peers* g, const int32_t* counts, uint64_t epoch, void* stream) {
  moe_status s = check_peers(g);
  if (s != MOE_OK) return s;
  if (!counts) return MOE_ERR_INVALID_ARG;
  MOE_LAUNCH(ep_publish_counts_kernel, 1, 256, 0, stream, *g, counts, epoch);
  return launched();
}

moe_status moe_ep_push_rows(const moe_ep_peers* g, const void* src, const int32_t* index, const int32_t* send_offs,
                            int64_t n_max, int64_t row_bytes, int64_t dst_row0, void* const* peer_dst, int32_t phase,
                            uint64_t epoch, void* stream) {
  moe_status s = check_peers(g);
  if (s != MOE_OK) return s;
  if (!send_offs || !peer_dst || n_max < 0 || row_bytes <= 0 || row_bytes % 4 || dst_row0 < 0 ||
      phase >= MOE_EP_NPHASE || (n_max > 0 && !src))
    return MOE_ERR_INVALID_ARG;
  const int P = g->n_ranks;
  const bool vec = row_bytes % 16 == 0 && ((uintptr_t)src % 16) == 0;
  const int64_t upr = vec ? row_bytes / 16 : row_bytes / 4;
  // every CTA must arrive for the last-CTA signal, so the grid is never empty
  const int64_t want = ceil_div(std::max<int64_t>(n_max * upr, 1), 256);
  const unsigned grid = (unsigned)std::min<int64_t>(want, 8 * sm_count());
  const size_t sm = (size_t)P * 16 + (size_t)(P + 1) * 4;
  if (vec)
    MOE_LAUNCH(ep_push_rows_kernel<uint4>, grid, 256, sm, stream, *g, (const uint4*)src, index, send_offs, upr,
               dst_row0, peer_dst, phase, epoch);
  else
    MOE_LAUNCH(ep_push_rows_kernel<uint32_t>, grid, 256, sm, stream, *g, (const uint32_t*)src, index, send_offs, upr,
               dst_row0, peer_dst, phase, epoch);
  return launched();
}

moe_status moe_ep_recv_prepare(const moe_ep_peers* g, int64_t T, int64_t T_cap, int32_t k, int32_t experts_per_rank,
                               int32_t* ids, float* w, int32_t* token_rows, void* stream) {
  moe_status s = check_peers(g);
  if (s != MOE_OK) return s;
  if (T < 0 || T_cap < T || T_cap >= (1ll << 31) || k < 1 || experts_per_rank < 1 || (T_cap > T && (!ids || !w)))
    return MOE_ERR_INVALID_ARG;
  if (T_cap == T && !token_rows) return MOE_OK;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div((T_cap - T) * k, 256), 4 * sm_count()));
  MOE_LAUNCH(ep_recv_prepare_kernel, grid, 256, 0, stream, *g, T, T_cap, k, experts_per_rank, ids, w, token_rows);
  return launched();
}

moe_status moe_ep_pull_combine(const moe_ep_peers* g, const moe_problem* p, const void* const* peer_rows, int64_t row0,
                               const int32_t* send_offs, const int32_t* send_pos, const void* base, void* out,
                               void* stream) {
  moe_status s = check_peers(g);
  if (s != MOE_OK) return s;
  if (!p || p->T < 0 || p->d <= 0 || p->d % 8 || (p->dtype != MOE_BF16 && p->dtype != MOE_FP32) || row0 < 0)
    return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && (!peer_rows || !send_offs || !send_pos || !out)) return MOE_ERR_INVALID_ARG;
  if ((uintptr_t)base % 16 || (uintptr_t)out % 16) return MOE_ERR_MISALIGNED;
  const int64_t n = p->T * (p->d / 8);
  if (n == 0) return MOE_OK;
  const int P = g->n_ranks;
  const size_t sm = (size_t)P * 16 + (size_t)(P + 1) * 4;
  const unsigned grid = (unsigned)ceil_div(n, 256);
  if (p->dtype == MOE_BF16)
    MOE_LAUNCH(ep_pull_combine_kernel<__nv_bfloat16>, grid, 256, sm, stream, *g, peer_rows, row0, send_offs, send_pos,
               (const __nv_bfloat16*)base, p->T, p->d, (__nv_bfloat16*)out);
  else
    MOE_LAUNCH(ep_pull_combine_kernel<float>, grid, 256, sm, stream, *g, peer_rows, row0, send_offs, send_pos,
               (const float*)base, p->T, p->d, (float*)out);
  return launched();
}

moe_status moe_ep_pull_slot_grad(const moe_ep_peers* g, const moe_problem* p, int32_t experts_per_rank,
                                 const int32_t* topk_ids, const float* const* peer_dg, int64_t row0,
                                 const int32_t* send_offs, const int32_t* send_pos, const float* dg_local, float* dg,
                                 void* stream) {
  moe_status s = check_peers(g);
  if (s != MOE_OK) return s;
  if (!p || p->T < 0 || p->k < 1 || experts_per_rank < 1 || (int64_t)experts_per_rank * g->n_ranks != p->E ||
      row0 < 0)
    return MOE_ERR_INVALID_ARG;
  if (p->T > 0 && (!topk_ids || !peer_dg || !send_offs || !send_pos || !dg_local || !dg)) return MOE_ERR_INVALID_ARG;
  const int64_t n = p->T * p->k;
  if (n == 0) return MOE_OK;
  const int P = g->n_ranks;
  const size_t sm = (size_t)P * 8 + (size_t)(P + 1) * 4;
  MOE_LAUNCH(ep_pull_slot_grad_kernel, (unsigned)ceil_div(n, 256), 256, sm, stream, *g, topk_ids, p->T, p->k,
             experts_per_rank, peer_dg, row0, send_offs, send_pos, dg_local, dg);
  return launched();
}

moe_status moe_ep_pull_sum(const moe_ep_peers* g, const void* const* peer_src, int64_t n, int32_t dtype, void* out,
                           void* stream) {
  moe_status s = check_peers(g);
  if (s != MOE_OK) return s;
  if (n < 0 || (dtype != MOE_BF16 && dtype != MOE_FP32) || (n > 0 && (!peer_src || !out))) return MOE_ERR_INVALID_ARG;
  if (n == 0) return MOE_OK;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 256), 4 * sm_count());
  if (dtype == MOE_BF16)
    MOE_LAUNCH(ep_pull_sum_kernel<__nv_bfloat16>, grid, 256, 0, stream, *g, peer_src, n, (__nv_bfloat16*)out);
  else
    MOE_LAUNCH(ep_pull_sum_kernel<float>, grid, 256, 0, stream, *g, peer_src, n, (float*)out);
  return launched();
}

moe_status moe_ep_ipc_handle(const void* ptr, void* handle_out, int64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) return MOE_ERR_INVALID_ARG;
  typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return MOE_ERR_CUDA;
    get_range = (GetRange)fn;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return MOE_ERR_CUDA;
  cudaIpcMemHandle_t h;
  MOE_CUDA_CHECK(cudaIpcGetMemHandle(&h, (void*)base));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)((CUdeviceptr)ptr - base);
  return MOE_OK;
}

moe_status moe_ep_ipc_open(const void* handle, int64_t offset, void** ptr_out, void** base_out) {
  if (!handle || offset < 0 || !ptr_out || !base_out) return MOE_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  MOE_CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *base_out = base;
  *ptr_out = (char*)base + offset;
  return MOE_OK;
}

moe_status moe_ep_ipc_close(void* base) {
  if (!base) return MOE_ERR_INVALID_ARG;
  MOE_CUDA_CHECK(cudaIpcCloseMemHandle(base));
  return MOE_OK;
}

}  // extern "C"
