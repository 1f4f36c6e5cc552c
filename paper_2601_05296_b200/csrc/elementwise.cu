// elementwise.cu — HBM-bound kernels around the expert GEMMs.
//
//  K9a dg_reduce   : d_topk_w[t,j] = sum_p partial[tim[t,j], p]  (fixed order)
//  K9b router_bwd  : dlogits = p * (dp - <p,dp>), dp = scatter of dsel (renorm-aware)
//  K9c dwg_partial / dwg_reduce : dW_g = dlogits^T X (split over tokens, fixed-order sum)
//  K10 finalize    : out = dtype(acc [+ dlogits W_g])  (Y, dX)
//  K11 gather_rows / combine_rows : expert-parallel send-buffer gather and the
//                    token-side k-way combine through token_index_map.
// The gate-weight gradient and router backward are the analytic derivative of
// P:42/P:91 (not in the paper; reading #14).
#include "common.cuh"

namespace moeb {

__global__ void dg_reduce_kernel(const float* __restrict__ part, int nparts, const int32_t* __restrict__ tim,
                                 int64_t R, float* __restrict__ dg) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= R) return;
  const float* p = part + (int64_t)tim[f] * nparts;
  float s = 0.f;
  for (int i = 0; i < nparts; ++i) s += p[i];
  dg[f] = s;
}

// one warp per token
__global__ void router_bwd_kernel(const float* __restrict__ logits, const int32_t* __restrict__ ids,
                                  const float* __restrict__ dg, int64_t T, int E, int k, int renorm,
                                  float* __restrict__ dlogits) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= T) return;
  const float* l = logits + t * E;
  float m = -INFINITY;
  for (int e = lane; e < E; e += 32) m = fmaxf(m, l[e]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
  for (int e = lane; e < E; e += 32) s += expf(l[e] - m);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float inv = 1.f / s;
  // selected probabilities and dsel (all lanes compute the same k values)
  float psum = 0.f, dgw = 0.f;
  for (int j = 0; j < k; ++j) psum += expf(l[ids[t * k + j]] - m) * inv;
  if (renorm)
    for (int j = 0; j < k; ++j) dgw += dg[t * k + j] * (expf(l[ids[t * k + j]] - m) * inv / psum);
  // <p, dp> = sum_j p_sel_j dsel_j
  float pdp = 0.f;
  for (int j = 0; j < k; ++j) {
    float ds = renorm ? (dg[t * k + j] - dgw) / psum : dg[t * k + j];
    pdp += expf(l[ids[t * k + j]] - m) * inv * ds;
  }
  for (int e = lane; e < E; e += 32) {
    float dp = 0.f;
    for (int j = 0; j < k; ++j)
      if (ids[t * k + j] == e) dp = renorm ? (dg[t * k + j] - dgw) / psum : dg[t * k + j];
    float p = expf(l[e] - m) * inv;
    dlogits[t * E + e] = p * (dp - pdp);
  }
}

// partial[c][e][col] = sum_{t in chunk c} dlogits[t,e] X[t,col].
// Block: 128 columns x ET experts x one token chunk; thread = 4 columns x
// ET/8 experts in registers; 32-token tiles of X and dlogits staged in shared
// memory (fp32) and read as float4: X is read exactly once over the grid.
constexpr int WG_COLS = 128;
constexpr int WG_TT = 32;  // tokens per shared-memory tile
template <typename T, int ET>
__global__ void __launch_bounds__(256) dwg_partial_kernel(const float* __restrict__ dlogits, const T* __restrict__ x,
                                                          int64_t Tn, int d, int E, int64_t tch,
                                                          float* __restrict__ part) {
  constexpr int EPT = ET / 8;  // experts per thread
  __shared__ __align__(16) float xs[WG_TT][WG_COLS];
  __shared__ __align__(16) float ds[WG_TT][ET];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c0 = blockIdx.x * WG_COLS;
  const int e0 = blockIdx.y * ET;
  const int64_t ta = blockIdx.z * tch, tb = min64(ta + tch, Tn);
  float acc[EPT][4];
#pragma unroll
  for (int i = 0; i < EPT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int64_t t0 = ta; t0 < tb; t0 += WG_TT) {
    const int nt = (int)min64(WG_TT, tb - t0);
    __syncthreads();
    for (int i = threadIdx.x; i < WG_TT * WG_COLS; i += 256) {
      const int r = i / WG_COLS, c = i % WG_COLS;
      xs[r][c] = (r < nt && c0 + c < d) ? to_f32(x[(t0 + r) * d + c0 + c]) : 0.f;
    }
    for (int i = threadIdx.x; i < WG_TT * ET; i += 256) {
      const int r = i / ET, e = i % ET;
      ds[r][e] = (r < nt && e0 + e < E) ? dlogits[(t0 + r) * E + e0 + e] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < WG_TT; ++r) {
      const float4 xv = *reinterpret_cast<const float4*>(&xs[r][4 * tx]);
      float dv[EPT];
      if constexpr (EPT % 4 == 0) {
#pragma unroll
        for (int q = 0; q < EPT; q += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(&ds[r][ty * EPT + q]);
          dv[q] = t4.x; dv[q + 1] = t4.y; dv[q + 2] = t4.z; dv[q + 3] = t4.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < EPT; ++q) dv[q] = ds[r][ty * EPT + q];
      }
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        acc[q][0] = fmaf(dv[q], xv.x, acc[q][0]);
        acc[q][1] = fmaf(dv[q], xv.y, acc[q][1]);
        acc[q][2] = fmaf(dv[q], xv.z, acc[q][2]);
        acc[q][3] = fmaf(dv[q], xv.w, acc[q][3]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const int e = e0 + ty * EPT + q;
    if (e >= E) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = c0 + 4 * tx + j;
      if (col < d) part[((int64_t)blockIdx.z * E + e) * d + col] = acc[q][j];
    }
  }
}

// dx[t, :] = dtype(acc[t, :] + sum_e dl[t, e] Wg[e, :]) — the router's share of
// the token gradient, fused with the fp32 -> dtype finalisation.  Block: 64
// tokens x 128 columns; thread = 8 tokens x 4 columns; experts in chunks of 32
// (W_g chunk and dl^T chunk staged in shared memory as fp32).
template <typename T, typename A>
__global__ void __launch_bounds__(256) router_dx_kernel(const A* __restrict__ acc, const float* __restrict__ dl,
                                                        const T* __restrict__ wg, int64_t Tn, int d, int E,
                                                        T* __restrict__ out) {
  __shared__ __align__(16) float ws_[32][128];
  __shared__ __align__(16) float dsT[32][64];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.y * 64;
  const int c0 = blockIdx.x * 128;
  const int col = c0 + 4 * tx;
  float a[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t t = t0 + ty * 8 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) a[i][j] = (t < Tn && col + j < d) ? to_f32(acc[t * d + col + j]) : 0.f;
  }
  for (int e0 = 0; e0 < E; e0 += 32) {
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 128; i += 256) {
      const int e = i / 128, c = i % 128;
      ws_[e][c] = (e0 + e < E && c0 + c < d) ? to_f32(wg[(int64_t)(e0 + e) * d + c0 + c]) : 0.f;
    }
    for (int i = threadIdx.x; i < 32 * 64; i += 256) {
      const int r = i / 32, e = i % 32;
      dsT[e][r] = (t0 + r < Tn && e0 + e < E) ? dl[(t0 + r) * E + e0 + e] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int e = 0; e < 32; ++e) {
      const float4 w = *reinterpret_cast<const float4*>(&ws_[e][4 * tx]);
      const float4 p0 = *reinterpret_cast<const float4*>(&dsT[e][ty * 8]);
      const float4 p1 = *reinterpret_cast<const float4*>(&dsT[e][ty * 8 + 4]);
      const float pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a[i][0] = fmaf(pv[i], w.x, a[i][0]);
        a[i][1] = fmaf(pv[i], w.y, a[i][1]);
        a[i][2] = fmaf(pv[i], w.z, a[i][2]);
        a[i][3] = fmaf(pv[i], w.w, a[i][3]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t t = t0 + ty * 8 + i;
    if (t >= Tn) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (col + j < d) out[t * d + col + j] = from_f32<T>(a[i][j]);
  }
}

template <typename T>
__global__ void dwg_reduce_kernel(const float* __restrict__ part, int nch, int64_t n, T* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int c = 0; c < nch; ++c) s += part[c * n + i];
  out[i] = from_f32<T>(s);
}

// out[t, :] = dtype(acc[t, :] + sum_e dl[t, e] Wg[e, :]); block: 16 tokens x 256 cols
template <typename T, typename A>
__global__ void __launch_bounds__(256) finalize_kernel(const A* __restrict__ acc, const float* __restrict__ dl,
                                                       const T* __restrict__ wg, int64_t Tn, int d, int E,
                                                       T* __restrict__ out) {
  extern __shared__ float sdl[];  // [16][E]
  const int col = blockIdx.x * 256 + threadIdx.x;
  const int64_t t0 = (int64_t)blockIdx.y * 16;
  const int nt = (int)min64(16, Tn - t0);
  float a[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) a[r] = (r < nt && col < d) ? to_f32(acc[(t0 + r) * d + col]) : 0.f;
  if (dl) {
    for (int i = threadIdx.x; i < 16 * E; i += 256) {
      int r = i / E, e = i % E;
      sdl[i] = r < nt ? dl[(t0 + r) * E + e] : 0.f;
    }
    __syncthreads();
    if (col < d) {
      for (int e = 0; e < E; ++e) {
        float w = to_f32(wg[(int64_t)e * d + col]);
#pragma unroll
        for (int r = 0; r < 16; ++r) a[r] = fmaf(sdl[r * E + e], w, a[r]);
      }
    }
  }
  if (col < d) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (r < nt) out[(t0 + r) * d + col] = from_f32<T>(a[r]);
  }
}

// per-row EP payload: gate weight and local expert id of every routed row
__global__ void ep_row_meta_kernel(const int32_t* __restrict__ row_slot, const int32_t* __restrict__ ids,
                                   const float* __restrict__ topw, int64_t R, int epr, float* __restrict__ row_w,
                                   int32_t* __restrict__ row_e) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int s = row_slot[r];
  row_w[r] = topw[s];
  row_e[r] = ids[s] % epr;
}

// 4-byte row gather for rows that are not a multiple of 16 bytes
__global__ void gather_rows4_kernel(const uint32_t* __restrict__ src, const int32_t* __restrict__ index, int64_t n,
                                    int64_t w_per_row, uint32_t* __restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * w_per_row) return;
  int64_t row = i / w_per_row, c = i % w_per_row;
  dst[i] = src[(int64_t)index[row] * w_per_row + c];
}

// vectorised row gather: 16-byte chunks
__global__ void gather_rows_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ index, int64_t n,
                                   int64_t vec_per_row, uint4* __restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = n * vec_per_row;
  if (i >= total) return;
  int64_t row = i / vec_per_row, c = i % vec_per_row;
  dst[i] = src[(int64_t)index[row] * vec_per_row + c];
}

template <typename T>
__global__ void combine_rows_kernel(const T* __restrict__ rows, const int32_t* __restrict__ tim, int64_t Tn, int d,
                                    int k, T* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Tn * d) return;
  int64_t t = i / d;
  int c = (int)(i % d);
  float s = 0.f;
  for (int j = 0; j < k; ++j) s += to_f32(rows[(int64_t)tim[t * k + j] * d + c]);
  out[i] = from_f32<T>(s);
}

// ----------------------------------------------------------------- launchers
moe_status launch_dg_reduce(const float* part, int nparts, const int32_t* tim, int64_t R, float* dg, cudaStream_t st) {
  if (R == 0) return MOE_OK;
  MOE_LAUNCH(dg_reduce_kernel, (unsigned)ceil_div(R, 256), 256, 0, st, part, nparts, tim, R, dg);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

static int dwg_et(int E) { return E <= 8 ? 8 : (E <= 16 ? 16 : (E <= 32 ? 32 : 64)); }

int dwg_chunks(int64_t T, int d) {
  // token chunks so that (column blocks x chunks) >= ~3 waves of 148 SMs, >= 128 tokens per chunk
  const int64_t colb = ceil_div(d, WG_COLS);
  int64_t nch = ceil_div(3 * 148, colb);
  nch = std::min<int64_t>(nch, std::max<int64_t>(1, T / 128));
  return (int)std::max<int64_t>(1, std::min<int64_t>(nch, 256));
}

template <typename T>
static void launch_dwg_partial(const float* dl, const T* x, int64_t Tn, int d, int E, int nch, int64_t tch, float* part,
                               cudaStream_t st) {
  const int et = dwg_et(E);
  dim3 grid((unsigned)ceil_div(d, WG_COLS), (unsigned)ceil_div(E, et), nch);
  if (et == 8) MOE_LAUNCH((dwg_partial_kernel<T, 8>), grid, 256, 0, st, dl, x, Tn, d, E, tch, part);
  else if (et == 16) MOE_LAUNCH((dwg_partial_kernel<T, 16>), grid, 256, 0, st, dl, x, Tn, d, E, tch, part);
  else if (et == 32) MOE_LAUNCH((dwg_partial_kernel<T, 32>), grid, 256, 0, st, dl, x, Tn, d, E, tch, part);
  else MOE_LAUNCH((dwg_partial_kernel<T, 64>), grid, 256, 0, st, dl, x, Tn, d, E, tch, part);
}

moe_status launch_router_bwd(const moe_problem* p, const float* logits, const int32_t* ids, const float* dg,
                             const void* x, float* dlogits, float* dwg_part, void* dwg, cudaStream_t st) {
  const int64_t T = p->T;
  const int E = p->E, d = p->d;
  if (T > 0) {
    MOE_LAUNCH(router_bwd_kernel, (unsigned)ceil_div(T * 32, 256), 256, 0, st, logits, ids, dg, T, E, p->k,
               p->renormalize, dlogits);
  }
  const int nch = dwg_chunks(T, d);
  const int64_t tch = ceil_div(std::max<int64_t>(T, 1), nch);
  const int64_t n = (int64_t)E * d;
  if (p->dtype == MOE_BF16) {
    launch_dwg_partial<__nv_bfloat16>(dlogits, (const __nv_bfloat16*)x, T, d, E, nch, tch, dwg_part, st);
    MOE_LAUNCH(dwg_reduce_kernel<__nv_bfloat16>, (unsigned)ceil_div(n, 256), 256, 0, st, dwg_part, nch, n, (__nv_bfloat16*)dwg);
  } else {
    launch_dwg_partial<float>(dlogits, (const float*)x, T, d, E, nch, tch, dwg_part, st);
    MOE_LAUNCH(dwg_reduce_kernel<float>, (unsigned)ceil_div(n, 256), 256, 0, st, dwg_part, nch, n, (float*)dwg);
  }
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

// acc_is_dtype: the accumulator is a [T,d] tensor of the run dtype (EP path) instead of fp32
moe_status launch_finalize(const moe_problem* p, const void* acc, const float* dl, const void* wg, void* out,
                           cudaStream_t st, bool acc_is_dtype) {
  if (p->T == 0) return MOE_OK;
  typedef __nv_bfloat16 bf;
  if (dl) {
    dim3 g2((unsigned)ceil_div(p->d, 128), (unsigned)ceil_div(p->T, 64));
    if (p->dtype == MOE_BF16) {
      if (acc_is_dtype)
        MOE_LAUNCH((router_dx_kernel<bf, bf>), g2, 256, 0, st, (const bf*)acc, dl, (const bf*)wg, p->T, p->d, p->E, (bf*)out);
      else
        MOE_LAUNCH((router_dx_kernel<bf, float>), g2, 256, 0, st, (const float*)acc, dl, (const bf*)wg, p->T, p->d, p->E,
                   (bf*)out);
    } else {
      MOE_LAUNCH((router_dx_kernel<float, float>), g2, 256, 0, st, (const float*)acc, dl, (const float*)wg, p->T, p->d,
                 p->E, (float*)out);
    }
    return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
  }
  dim3 grid((unsigned)ceil_div(p->d, 256), (unsigned)ceil_div(p->T, 16));
  size_t sm = 0;
  if (p->dtype == MOE_BF16) {
    if (acc_is_dtype)
      MOE_LAUNCH((finalize_kernel<bf, bf>), grid, 256, sm, st, (const bf*)acc, dl, (const bf*)wg, p->T, p->d, p->E, (bf*)out);
    else
      MOE_LAUNCH((finalize_kernel<bf, float>), grid, 256, sm, st, (const float*)acc, dl, (const bf*)wg, p->T, p->d, p->E,
                 (bf*)out);
  } else {
    MOE_LAUNCH((finalize_kernel<float, float>), grid, 256, sm, st, (const float*)acc, dl, (const float*)wg, p->T, p->d,
               p->E, (float*)out);
  }
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

moe_status launch_ep_row_meta(const int32_t* row_slot, const int32_t* ids, const float* topw, int64_t R, int epr,
                              float* row_w, int32_t* row_e, cudaStream_t st) {
  if (R == 0) return MOE_OK;
  MOE_LAUNCH(ep_row_meta_kernel, (unsigned)ceil_div(R, 256), 256, 0, st, row_slot, ids, topw, R, epr, row_w, row_e);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

moe_status launch_gather_rows(const void* src, const int32_t* index, int64_t n, int64_t row_bytes, void* dst,
                              cudaStream_t st) {
  if (n == 0) return MOE_OK;
  if (row_bytes % 16 != 0) {
    const int64_t wpr = row_bytes / 4;
    MOE_LAUNCH(gather_rows4_kernel, (unsigned)ceil_div(n * wpr, 256), 256, 0, st, (const uint32_t*)src, index, n,
               wpr, (uint32_t*)dst);
    return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
  }
  const int64_t vpr = row_bytes / 16;
  MOE_LAUNCH(gather_rows_kernel, (unsigned)ceil_div(n * vpr, 256), 256, 0, st, (const uint4*)src, index, n, vpr,
             (uint4*)dst);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

moe_status launch_combine_rows(const moe_problem* p, const void* rows, const int32_t* tim, void* out, cudaStream_t st) {
  const int64_t n = p->T * p->d;
  if (n == 0) return MOE_OK;
  if (p->dtype == MOE_BF16)
    MOE_LAUNCH(combine_rows_kernel<__nv_bfloat16>, (unsigned)ceil_div(n, 256), 256, 0, st,
               (const __nv_bfloat16*)rows, tim, p->T, p->d, p->k, (__nv_bfloat16*)out);
  else
    MOE_LAUNCH(combine_rows_kernel<float>, (unsigned)ceil_div(n, 256), 256, 0, st, (const float*)rows, tim, p->T,
               p->d, p->k, (float*)out);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

}  // namespace moeb
