// route.cu — K1: gating network + top-k.
//
// logits[t,e] = sum_c X[t,c] * Wg[e,c]  (fp32 accumulation)
// ids[t,:]    = k largest logits, descending, exact ties -> lower expert id
// topk_w[t,j] = softmax(logits[t,:])[ids[t,j]]  (optionally renormalised)
//
// HBM-bound: X is read exactly once.  A CTA owns 32 tokens; d is streamed in
// 64-column chunks through shared memory together with the matching Wg chunk
// (Wg stays L2-resident across CTAs).  Warp w computes experts e = w, w+8, ...
// for the 32 tokens (lane = token), so X reads are conflict-free (padded rows)
// and Wg reads are warp broadcasts.  Top-k: one warp per token, k rounds of a
// warp arg-max over (value, -index).
#include "common.cuh"

namespace moeb {

constexpr int RT_TOK = 32;     // tokens per CTA
constexpr int RT_DC = 64;      // d columns per chunk
constexpr int RT_THREADS = 256;
constexpr int RT_MAXE_PER_WARP = 32;  // E <= 256 over 8 warps

template <typename T>
__global__ void __launch_bounds__(RT_THREADS)
route_kernel(const T* __restrict__ x, const T* __restrict__ wg, int64_t Tn, int d, int E, int k,
             int renorm, float* __restrict__ logits, int32_t* __restrict__ ids, float* __restrict__ topw) {
  extern __shared__ float sm[];
  float* xs = sm;                                  // [RT_TOK][RT_DC+1]
  float* ws = xs + RT_TOK * (RT_DC + 1);           // [E][RT_DC+1]
  float* ls = ws + E * (RT_DC + 1);                // [RT_TOK][E+1]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * RT_TOK;
  const int ntok = (int)min64(RT_TOK, Tn - t0);
  float acc[RT_MAXE_PER_WARP];
#pragma unroll
  for (int i = 0; i < RT_MAXE_PER_WARP; ++i) acc[i] = 0.f;
  const int ne = (E - warp + 7) / 8;  // experts of this warp

  for (int c0 = 0; c0 < d; c0 += RT_DC) {
    const int dc = min(RT_DC, d - c0);
    for (int i = tid; i < RT_TOK * RT_DC; i += RT_THREADS) {
      int r = i / RT_DC, c = i % RT_DC;
      xs[r * (RT_DC + 1) + c] = (r < ntok && c < dc) ? to_f32(x[(t0 + r) * d + c0 + c]) : 0.f;
    }
    for (int i = tid; i < E * RT_DC; i += RT_THREADS) {
      int r = i / RT_DC, c = i % RT_DC;
      ws[r * (RT_DC + 1) + c] = (c < dc) ? to_f32(wg[(int64_t)r * d + c0 + c]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RT_MAXE_PER_WARP; ++i) {
      if (i < ne) {
        const float* wr = ws + (warp + 8 * i) * (RT_DC + 1);
        const float* xr = xs + lane * (RT_DC + 1);
        float a = acc[i];
#pragma unroll 16
        for (int c = 0; c < RT_DC; ++c) a = fmaf(xr[c], wr[c], a);
        acc[i] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < RT_MAXE_PER_WARP; ++i)
    if (i < ne) ls[lane * (E + 1) + warp + 8 * i] = acc[i];
  __syncthreads();

  // one warp per token: logits out, softmax, top-k
  for (int r = warp; r < ntok; r += RT_THREADS / 32) {
    const float* lr = ls + r * (E + 1);
    const int64_t t = t0 + r;
    float m = -INFINITY;
    for (int e = lane; e < E; e += 32) {
      float v = lr[e];
      logits[t * E + e] = v;
      m = fmaxf(m, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float s = 0.f;
    for (int e = lane; e < E; e += 32) s += expf(lr[e] - m);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    // k rounds of arg-max; chosen experts are excluded by a per-lane bitmask
    uint32_t taken = 0;  // bit q <-> expert lane + 32q (E <= 256 -> q < 8)
    float wsum = 0.f;
    float wsel[16];
    int isel[16];
    for (int j = 0; j < k; ++j) {
      float bv = -INFINITY;
      int be = 0x7fffffff;
      for (int q = 0, e = lane; e < E; ++q, e += 32) {
        if ((taken >> q) & 1u) continue;
        float v = lr[e];
        if (v > bv || (v == bv && e < be)) { bv = v; be = e; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oe = __shfl_xor_sync(0xffffffffu, be, o);
        if (ov > bv || (ov == bv && oe < be)) { bv = ov; be = oe; }
      }
      if ((be & 31) == lane) taken |= 1u << (be >> 5);
      float p = expf(bv - m) / s;
      wsel[j] = p;
      isel[j] = be;
      wsum += p;
    }
    if (lane == 0) {
      for (int j = 0; j < k; ++j) {
        ids[t * k + j] = isel[j];
        topw[t * k + j] = renorm ? wsel[j] / wsum : wsel[j];
      }
    }
  }
}

size_t route_smem_bytes(int E) {
  return sizeof(float) * (RT_TOK * (RT_DC + 1) + (size_t)E * (RT_DC + 1) + RT_TOK * (E + 1));
}

moe_status tc_route(const moe_problem* p, const void* x, const void* wg, float* logits, int32_t* ids, float* topw,
                    cudaStream_t st);

// bf16: tensor-core router (gemm_tc.cu, TC_ROUTE); fp32 storage mode: the CUDA-core kernel above.
moe_status launch_route(const moe_problem* p, const void* x, const void* wg, float* logits, int32_t* ids,
                        float* topw, cudaStream_t st) {
  if (p->T == 0) return MOE_OK;
  if (p->dtype == MOE_BF16) return tc_route(p, x, wg, logits, ids, topw, st);
  dim3 grid((unsigned)ceil_div(p->T, RT_TOK));
  size_t smem = route_smem_bytes(p->E);
  MOE_CUDA_CHECK(cudaFuncSetAttribute(route_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  MOE_LAUNCH(route_kernel<float>, grid, RT_THREADS, smem, st, (const float*)x, (const float*)wg, p->T, p->d,
             p->E, p->k, p->renormalize, logits, ids, topw);
  MOE_CUDA_CHECK(cudaGetLastError());
  return MOE_OK;
}

}  // namespace moeb
