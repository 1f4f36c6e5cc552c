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

// g lanes (1 or 32, chosen by the launcher) per routed slot f: the
// slot's partials row is read contiguously by the group and tree-summed (fixed order)
__global__ void dg_reduce_kernel(const float* __restrict__ part, int nparts, const int32_t* __restrict__ tim,
                                 int64_t R, float* __restrict__ dg, int g) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t f = gt / g;
  const int sub = (int)(gt % g);
  float s = 0.f;
  if (f < R) {
    const int r = tim[f];
    if (r >= 0) {  // r < 0: empty slot (sparse slots) -> no routed row, zero gradient
      const float* p = part + (int64_t)r * nparts;
      for (int i = sub; i < nparts; i += g) s += p[i];
    }
  }
  for (int o = g >> 1; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);  // stays inside the group
  if (f < R && sub == 0) dg[f] = s;
}

// one warp per token
// dlhl != NULL (bf16 runs): also dl = hi + lo as two bf16 [T, ep8] tensors (zero
// columns E..ep8-1), the tensor-core operands of router_tc.cu
__global__ void router_bwd_kernel(const float* __restrict__ logits, const int32_t* __restrict__ ids,
                                  const float* __restrict__ dg, int64_t T, int E, int k, int renorm,
                                  float* __restrict__ dlogits, __nv_bfloat16* __restrict__ dlhl, int ep8) {
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
  // the k routed slots side by side: lane j < k holds slot j (ids, dg, p_sel), so the
  // sums over slots are warp reductions instead of k dependent load chains
  int id_j = -1;
  float p_j = 0.f, dg_j = 0.f;
  if (lane < k) {
    id_j = ids[t * k + lane];
    dg_j = dg[t * k + lane];
    p_j = id_j >= 0 ? expf(l[id_j] - m) * inv : 0.f;
  }
  auto wsum = [](float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  const float psum = wsum(p_j);
  const float dgw = renorm ? wsum(dg_j * (p_j / psum)) : 0.f;
  const float ds_j = lane < k ? (renorm ? (dg_j - dgw) / psum : dg_j) : 0.f;
  // <p, dp> = sum_j p_sel_j dsel_j
  const float pdp = wsum(p_j * ds_j);
  for (int e0 = 0; e0 < E; e0 += 32) {  // warp-uniform trip count: the shuffles see all lanes
    const int e = e0 + lane;
    float dp = 0.f;
    for (int j = 0; j < k; ++j) {
      const int idj = __shfl_sync(0xffffffffu, id_j, j);
      const float dsj = __shfl_sync(0xffffffffu, ds_j, j);
      if (idj == e) dp = dsj;
    }
    if (e >= E) continue;
    float p = expf(l[e] - m) * inv;
    const float v = p * (dp - pdp);
    dlogits[t * E + e] = v;
    if (dlhl) {
      const __nv_bfloat16 hi = __float2bfloat16_rn(v);
      dlhl[t * ep8 + e] = hi;
      dlhl[(T + t) * ep8 + e] = __float2bfloat16_rn(v - __bfloat162float(hi));
    }
  }
  if (dlhl)
    for (int e = E + lane; e < ep8; e += 32) {
      dlhl[t * ep8 + e] = __float2bfloat16_rn(0.f);
      dlhl[(T + t) * ep8 + e] = __float2bfloat16_rn(0.f);
    }
}

// partial[c][e][col] = sum_{t in chunk c} dlogits[t,e] X[t,col].
// Thread tile: 8 consecutive columns x 8 experts (64 fp32 accumulators).
// Block = 256 threads = CGR column groups x EGR expert groups (EGR =
// ceil(E/8) <= 8).  X streams through a double-buffered 16 KB shared-memory
// tile filled with 16-byte cp.async (TT = 4*EGR tokens per tile) so enough
// bytes are in flight to run at HBM speed; the chunk's dlogits rows are
// staged alongside.  X is read exactly once.  Requires d % 8 == 0.
__device__ __forceinline__ void cpa16(void* dst, const void* src, bool ok) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16u : 0u) : "memory");
}
template <typename T, int EGR>
__global__ void __launch_bounds__(256) dwg_partial_kernel(const float* __restrict__ dlogits, const T* __restrict__ x,
                                                          int64_t Tn, int d, int E, int64_t tch,
                                                          float* __restrict__ part) {
  constexpr int CGR = 256 / EGR;            // column groups (8 columns each)
  constexpr int COLS = CGR * 8;             // columns per block
  constexpr int TT = 16384 / (COLS * (int)sizeof(T)) > 0 ? 16384 / (COLS * (int)sizeof(T)) : 1;  // tokens per tile
  constexpr int VPR = COLS * (int)sizeof(T) / 16;  // 16-byte vectors per token row of the tile
  __shared__ __align__(16) uint8_t xs_raw[2][TT * COLS * sizeof(T)];
  __shared__ __align__(16) float ds[2][TT][EGR * 8];
  const int cg = threadIdx.x % CGR, eg = threadIdx.x / CGR;
  const int c0 = blockIdx.x * COLS;
  const int col = c0 + cg * 8;
  const int ebase = blockIdx.z * EGR * 8;  // expert block (E > 64 uses several)
  const int64_t ta = blockIdx.y * tch, tb = min64(ta + tch, Tn);
  const int ntiles = (int)ceil_div(tb - ta, TT);
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  auto issue = [&](int it, int buf) {
    const int64_t t0 = ta + (int64_t)it * TT;
    T* xs = reinterpret_cast<T*>(xs_raw[buf]);
    for (int v = threadIdx.x; v < TT * VPR; v += 256) {
      const int r = v / VPR, cv = v % VPR;
      const int64_t t = t0 + r;
      const int cc = cv * (16 / (int)sizeof(T));
      const bool ok = t < tb && c0 + cc < d;
      cpa16(xs + r * COLS + cc, ok ? (const void*)(x + t * d + c0 + cc) : (const void*)x, ok);
    }
    for (int v = threadIdx.x; v < TT * EGR * 8; v += 256) {
      const int r = v / (EGR * 8), e = v % (EGR * 8);
      const int64_t t = t0 + r;
      ds[buf][r][e] = (t < tb && ebase + e < E) ? dlogits[t * E + ebase + e] : 0.f;
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (ntiles > 0) issue(0, 0);
  for (int it = 0; it < ntiles; ++it) {
    const int buf = it & 1;
    if (it + 1 < ntiles) {
      issue(it + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const T* xs = reinterpret_cast<const T*>(xs_raw[buf]);
#pragma unroll
    for (int r = 0; r < TT; ++r) {
      float xv[8];
      load8(xs + r * COLS + cg * 8, xv);
      const float4 e0 = *reinterpret_cast<const float4*>(&ds[buf][r][eg * 8]);
      const float4 e1 = *reinterpret_cast<const float4*>(&ds[buf][r][eg * 8 + 4]);
      const float ev[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[q][j] = fmaf(ev[q], xv[j], acc[q][j]);
    }
    __syncthreads();
  }
  if (col < d) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = ebase + eg * 8 + q;
      if (e < E) store8(part + ((int64_t)blockIdx.y * E + e) * d + col, acc[q]);
    }
  }
}

// The token-side accumulator of 8 columns: acc[t] ([T,d], fused red.add or
// k = 1 store), or with tim != NULL the ordered combine of NEXT-4: acc holds
// one fp32 row per routed row ([R,d], expert-sorted) and token t sums its k
// rows in slot order j = 0..k-1 (fixed order -> bitwise reproducible).
template <typename A>
__device__ __forceinline__ void load_acc8(const A* acc, const int32_t* tim, int k, int64_t t, int d, int col, float* a) {
  if (!tim) {
    load8(acc + t * d + col, a);
    return;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 0.f;
  for (int j = 0; j < k; ++j) {
    const int r = tim[t * k + j];
    if (r < 0) continue;  // empty slot
    float v[8];
    load8(acc + (int64_t)r * d + col, v);
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] += v[q];
  }
}

// dx[t, :] = dtype(acc[t, :] + sum_e dl[t, e] Wg[e, :]) — the router's share of
// the token gradient fused with the fp32 -> dtype finalisation.  Thread tile:
// 8 consecutive columns (one 16-byte W_g load per expert, L1/L2-resident) x 8
// tokens; block = 32 column groups (256 columns) x 8 token groups (64 tokens);
// a warp shares its token group, so the dlogits reads are smem broadcasts.
template <typename T, typename A>
__global__ void __launch_bounds__(256) router_dx_kernel(const A* __restrict__ acc, const int32_t* __restrict__ tim,
                                                        int k, const float* __restrict__ dl,
                                                        const T* __restrict__ wg, int64_t Tn, int d, int E,
                                                        T* __restrict__ out) {
  __shared__ __align__(16) float wsm[32][256];  // W_g chunk: 32 experts x 256 columns (fp32)
  __shared__ float dsm[32][64 + 1];             // dlogits chunk: 32 experts x 64 tokens
  const int cg = threadIdx.x & 31, tg = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.y * 64;
  const int c0 = blockIdx.x * 256;
  const int col = c0 + cg * 8;
  float a[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t t = t0 + tg * 8 + i;
    if (t < Tn && col < d) load_acc8(acc, tim, k, t, d, col, a[i]);
    else
#pragma unroll
      for (int j = 0; j < 8; ++j) a[i][j] = 0.f;
  }
  for (int e0 = 0; e0 < E; e0 += 32) {
    __syncthreads();
    for (int v = threadIdx.x; v < 32 * 32; v += 256) {  // 32 experts x 32 vectors of 8 columns
      const int e = v / 32, cv = v % 32;
      float w[8];
      if (e0 + e < E && c0 + cv * 8 < d) load8(wg + (int64_t)(e0 + e) * d + c0 + cv * 8, w);
      else
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = 0.f;
      store8(&wsm[e][cv * 8], w);
    }
    for (int v = threadIdx.x; v < 64 * 32; v += 256) {
      const int r = v / 32, e = v % 32;
      dsm[e][r] = (t0 + r < Tn && e0 + e < E) ? dl[(t0 + r) * E + e0 + e] : 0.f;
    }
    __syncthreads();
    const int ne = min(32, E - e0);
#pragma unroll 4
    for (int e = 0; e < ne; ++e) {
      float w[8];
      load8(&wsm[e][cg * 8], w);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float p = dsm[e][tg * 8 + i];
#pragma unroll
        for (int j = 0; j < 8; ++j) a[i][j] = fmaf(p, w[j], a[i][j]);
      }
    }
  }
  if (col >= d) return;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t t = t0 + tg * 8 + i;
    if (t < Tn) store8(out + t * d + col, a[i]);
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
__global__ void __launch_bounds__(256) finalize_kernel(const A* __restrict__ acc, const int32_t* __restrict__ tim,
                                                       int k, const float* __restrict__ dl,
                                                       const T* __restrict__ wg, int64_t Tn, int d, int E,
                                                       T* __restrict__ out) {
  extern __shared__ float sdl[];  // [16][E]
  const int col = blockIdx.x * 256 + threadIdx.x;
  const int64_t t0 = (int64_t)blockIdx.y * 16;
  const int nt = (int)min64(16, Tn - t0);
  float a[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    a[r] = 0.f;
    if (r < nt && col < d) {
      if (!tim) a[r] = to_f32(acc[(t0 + r) * d + col]);
      else
        for (int j = 0; j < k; ++j) {
          const int rr = tim[(t0 + r) * k + j];
          if (rr >= 0) a[r] += to_f32(acc[(int64_t)rr * d + col]);
        }
    }
  }
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

// ---- expert-parallel plan (NEXT-1: one row per (token, destination rank))
// dest[t, q] = q if rank q owns one of the token's experts, else -1; the column of rank
// `self` (>= 0) stays -1: those pairs are computed where the token lives (no exchange)
__global__ void ep_dest_kernel(const int32_t* __restrict__ ids, int64_t T, int k, int epr, int P, int self,
                               int32_t* __restrict__ dest) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  uint32_t mask[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // P <= 256 ranks
  for (int j = 0; j < k; ++j) {
    const int q = ids[t * k + j] / epr;
    mask[q >> 5] |= 1u << (q & 31);
  }
  for (int q = 0; q < P; ++q) dest[t * P + q] = (q != self && ((mask[q >> 5] >> (q & 31)) & 1u)) ? q : -1;
}

// the local rank's own slots of every local token: ids - rank*epr where owned, else -1
__global__ void ep_local_slots_kernel(const int32_t* __restrict__ ids, const float* __restrict__ topw, int64_t n,
                                      int epr, int rank, int32_t* __restrict__ lids, float* __restrict__ lw) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  const int e = ids[f];
  const bool mine = e / epr == rank;
  lids[f] = mine ? e - rank * epr : -1;
  lw[f] = mine ? topw[f] : 0.f;
}

// send row i (row_slot = t*P + q): the token's slots restricted to rank q, local expert ids
__global__ void ep_send_meta_kernel(const int32_t* __restrict__ ids, const float* __restrict__ topw, int k, int epr,
                                    int P, const int32_t* __restrict__ row_slot, int64_t n,
                                    int32_t* __restrict__ send_ids, float* __restrict__ send_w) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // f = i*k + j
  if (f >= n * k) return;
  const int64_t i = f / k;
  const int j = (int)(f - i * k);
  const int rs = row_slot[i];
  const int64_t t = rs / P;
  const int q = rs - (int)(t * P);
  const int e = ids[t * k + j];
  const bool mine = e / epr == q;
  send_ids[f] = mine ? e - q * epr : -1;
  send_w[f] = mine ? topw[t * k + j] : 0.f;
}

// dg[t, j] = dg_back[send_pos[t, owner(ids[t,j])], j], or dg_local[t, j] when the owner is
// `self` (computed here, on the receiver's first T token rows)
__global__ void ep_slot_grad_kernel(const int32_t* __restrict__ ids, int64_t T, int k, int epr, int P,
                                    const int32_t* __restrict__ send_pos, const float* __restrict__ dg_back,
                                    const float* __restrict__ dg_local, int self, float* __restrict__ dg) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= T * k) return;
  const int64_t t = f / k;
  const int j = (int)(f - t * k);
  const int q = ids[f] / epr;
  dg[f] = q == self ? dg_local[f] : dg_back[(int64_t)send_pos[t * P + q] * k + j];
}

// 4-byte row gather for rows that are not a multiple of 16 bytes
__global__ void gather_rows4_kernel(const uint32_t* __restrict__ src, const int32_t* __restrict__ index, int64_t n,
                                    int64_t w_per_row, uint32_t* __restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * w_per_row) return;
  int64_t row = i / w_per_row, c = i % w_per_row;
  dst[i] = src[(index ? (int64_t)index[row] : row) * w_per_row + c];
}

// vectorised row gather: 16-byte chunks
__global__ void gather_rows_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ index, int64_t n,
                                   int64_t vec_per_row, uint4* __restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = n * vec_per_row;
  if (i >= total) return;
  int64_t row = i / vec_per_row, c = i % vec_per_row;
  dst[i] = src[(index ? (int64_t)index[row] : row) * vec_per_row + c];
}

// out[t, 8c .. 8c+7] = sum_j rows[tim[t,j], ...] (fixed j order, -1 skipped); d % 8 == 0
// base (optional, [T, d]): added first (the locally computed partial of the token)
template <typename T>
__global__ void combine_rows_kernel(const T* __restrict__ rows, const int32_t* __restrict__ tim, const T* __restrict__ base,
                                    int64_t Tn, int d, int k, T* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int cpr = d / 8;
  if (i >= Tn * cpr) return;
  const int64_t t = i / cpr;
  const int col = (int)(i - t * cpr) * 8;
  float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (base) load8(base + t * d + col, a);
  for (int j = 0; j < k; ++j) {
    const int r = tim[t * k + j];
    if (r < 0) continue;
    float v[8];
    load8(rows + (int64_t)r * d + col, v);
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] += v[q];
  }
  store8(out + t * d + col, a);
}

// ----------------------------------------------------------------- launchers
moe_status launch_dg_reduce(const float* part, int nparts, const int32_t* tim, int64_t R, float* dg, cudaStream_t st) {
  if (R == 0) return MOE_OK;
  // a warp per slot only for long rows (Mixtral-like h: 112 partials, 16.4 -> 9.4 us);
  // short rows keep a thread per slot (DeepSeek-like, 11 partials: 7.6 us vs 12.4 at g = 16)
  const int g = nparts >= 32 ? 32 : 1;
  MOE_LAUNCH(dg_reduce_kernel, (unsigned)ceil_div(R * g, 256), 256, 0, st, part, nparts, tim, R, dg, g);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

static int dwg_egr(int E) {
  const int g = (int)ceil_div(E, 8);
  return g <= 1 ? 1 : (g <= 2 ? 2 : (g <= 4 ? 4 : 8));
}

int router_dwg_tc_splits(int64_t T, int d);
int router_ep8(int E);
moe_status launch_router_dwg_tc(const __nv_bfloat16* dlhl, const void* x, int64_t T, int d, int E, float* part,
                                cudaStream_t st);
moe_status launch_router_dx_tc(bool load, const void* acc, bool acc_is_dtype, const int32_t* tim, int k,
                               const __nv_bfloat16* dlhl, const void* wg, int64_t T, int d, int E, void* out,
                               cudaStream_t st);

// token chunks of the dW_g partial sums: bf16 runs use the tensor-core split
// (router_tc.cu); fp32 runs the CUDA-core kernel below
int dwg_chunks(const moe_problem* p) {
  const int64_t T = p->T;
  const int d = p->d, E = p->E;
  if (p->dtype == MOE_BF16) return router_dwg_tc_splits(T, d);
  // column blocks x token chunks >= ~3 waves of 148 SMs, >= 64 tokens per chunk
  const int64_t colb = ceil_div(d, 8 * (256 / dwg_egr(E)));
  int64_t nch = ceil_div(3 * 148, colb);
  nch = std::min<int64_t>(nch, std::max<int64_t>(1, T / 64));
  return (int)std::max<int64_t>(1, std::min<int64_t>(nch, 256));
}

template <typename T>
static void launch_dwg_partial(const float* dl, const T* x, int64_t Tn, int d, int E, int nch, int64_t tch, float* part,
                               cudaStream_t st) {
  const int egr = dwg_egr(E);
  const int cols_per_block = 8 * (256 / egr);
  dim3 grid((unsigned)ceil_div(d, cols_per_block), nch, (unsigned)ceil_div(E, egr * 8));
  if (egr == 1) MOE_LAUNCH((dwg_partial_kernel<T, 1>), grid, 256, 0, st, dl, x, Tn, d, E, tch, part);
  else if (egr == 2) MOE_LAUNCH((dwg_partial_kernel<T, 2>), grid, 256, 0, st, dl, x, Tn, d, E, tch, part);
  else if (egr == 4) MOE_LAUNCH((dwg_partial_kernel<T, 4>), grid, 256, 0, st, dl, x, Tn, d, E, tch, part);
  else MOE_LAUNCH((dwg_partial_kernel<T, 8>), grid, 256, 0, st, dl, x, Tn, d, E, tch, part);
}

// dlhl: bf16 runs, [2, T, router_ep8(E)] hi / lo split of dlogits (written here)
moe_status launch_router_bwd(const moe_problem* p, const float* logits, const int32_t* ids, const float* dg,
                             const void* x, float* dlogits, __nv_bfloat16* dlhl, float* dwg_part, void* dwg,
                             cudaStream_t st) {
  const int64_t T = p->T;
  const int E = p->E, d = p->d;
  const bool bf = p->dtype == MOE_BF16;
  if (T > 0) {
    MOE_LAUNCH(router_bwd_kernel, (unsigned)ceil_div(T * 32, 256), 256, 0, st, logits, ids, dg, T, E, p->k,
               p->renormalize, dlogits, bf ? dlhl : nullptr, router_ep8(E));
  }
  const int nch = dwg_chunks(p);
  const int64_t tch = ceil_div(std::max<int64_t>(T, 1), nch);
  const int64_t n = (int64_t)E * d;
  if (p->dtype == MOE_BF16) {
    moe_status s = launch_router_dwg_tc(dlhl, x, T, d, E, dwg_part, st);  // tensor cores, split-T partials
    if (s != MOE_OK) return s;
    MOE_LAUNCH(dwg_reduce_kernel<__nv_bfloat16>, (unsigned)ceil_div(n, 256), 256, 0, st, dwg_part, nch, n, (__nv_bfloat16*)dwg);
  } else {
    launch_dwg_partial<float>(dlogits, (const float*)x, T, d, E, nch, tch, dwg_part, st);
    MOE_LAUNCH(dwg_reduce_kernel<float>, (unsigned)ceil_div(n, 256), 256, 0, st, dwg_part, nch, n, (float*)dwg);
  }
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

// out = dtype(acc [+ dlogits W_g]).  acc_is_dtype: the accumulator is a [T,d]
// tensor of the run dtype (EP path) instead of fp32; tim != NULL: acc is the
// [R,d] fp32 row-result buffer, summed per token in slot order (NEXT-4).
// bf16 with the router term: tensor cores (router_tc.cu) from the hi/lo split dlhl.
// out[i] = bf16(acc[i]) over n8 groups of 8 (two 16-byte loads, one 16-byte store per thread
// per step, grid-stride: the HBM-bound Y finalize)
__global__ void __launch_bounds__(256) convert_f32_bf16_kernel(const float4* __restrict__ acc, int64_t n8,
                                                                uint4* __restrict__ out,
                                                                const int32_t* __restrict__ t_rows, int d8,
                                                                int64_t row0) {
  // rows past the device bound are unused (acc / out start at token row row0)
  if (t_rows) n8 = min64(n8, max((int64_t)0, (int64_t)__ldg(t_rows) - row0) * d8);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = __ldcs(acc + 2 * i), b = __ldcs(acc + 2 * i + 1);
    uint4 o;
    __nv_bfloat162 h;
    h = __floats2bfloat162_rn(a.x, a.y); o.x = *reinterpret_cast<uint32_t*>(&h);
    h = __floats2bfloat162_rn(a.z, a.w); o.y = *reinterpret_cast<uint32_t*>(&h);
    h = __floats2bfloat162_rn(b.x, b.y); o.z = *reinterpret_cast<uint32_t*>(&h);
    h = __floats2bfloat162_rn(b.z, b.w); o.w = *reinterpret_cast<uint32_t*>(&h);
    out[i] = o;
  }
}

// acc[t, :] = 0 for t < *t_rows (the fp32 combine accumulator; the rows past the
// device-side bound are never referenced)
__global__ void zero_rows_kernel(float4* __restrict__ acc, int64_t n4, const int32_t* __restrict__ t_rows, int d4) {
  const int64_t n = t_rows ? min64(n4, (int64_t)__ldg(t_rows) * d4) : n4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

static int sm_count_cached() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  return nsm;
}

#ifndef ZERO_KERNEL
#define ZERO_KERNEL 0  // 1: the library's zeroing kernel also without a device row bound (A/B vs cudaMemsetAsync)
#endif
moe_status launch_zero_acc(float* acc, int64_t T, int d, const int32_t* t_rows, cudaStream_t st) {
  if (T == 0) return MOE_OK;
  if ((!t_rows && !ZERO_KERNEL) || d % 4) {
    MOE_CUDA_CHECK(cudaMemsetAsync(acc, 0, (size_t)T * d * 4, st));
    return MOE_OK;
  }
  const int64_t n4 = T * (int64_t)d / 4;
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n4, 256), (int64_t)sm_count_cached() * 8);
  MOE_LAUNCH(zero_rows_kernel, blocks, 256, 0, st, (float4*)acc, n4, t_rows, d / 4);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

moe_status launch_finalize(const moe_problem* p, const void* acc, const float* dl, const __nv_bfloat16* dlhl,
                           const void* wg, void* out, cudaStream_t st, bool acc_is_dtype, const int32_t* tim,
                           const int32_t* t_rows, int64_t row0) {
  if (p->T == 0) return MOE_OK;
  typedef __nv_bfloat16 bf;
  if (dl && p->dtype == MOE_BF16)
    return launch_router_dx_tc(true, acc, acc_is_dtype, tim, p->k, dlhl, wg, p->T, p->d, p->E, out, st);
  if (dl) {  // fp32 storage: CUDA-core FMA (true fp32)
    dim3 g2((unsigned)ceil_div(p->d, 256), (unsigned)ceil_div(p->T, 64));
    MOE_LAUNCH((router_dx_kernel<float, float>), g2, 256, 0, st, (const float*)acc, tim, p->k, dl, (const float*)wg,
               p->T, p->d, p->E, (float*)out);
    return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
  }
  if (p->dtype == MOE_BF16 && !acc_is_dtype && !tim && p->d % 8 == 0) {
    // the plain Y conversion (fp32 accumulator -> bf16): 8 columns per thread per step
    const int64_t n8 = p->T * (int64_t)p->d / 8;
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n8, 256), (int64_t)sm_count_cached() * 8);
    MOE_LAUNCH(convert_f32_bf16_kernel, blocks, 256, 0, st, (const float4*)acc, n8, (uint4*)out, t_rows, p->d / 8,
               row0);
    return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
  }
  dim3 grid((unsigned)ceil_div(p->d, 256), (unsigned)ceil_div(p->T, 16));
  size_t sm = 0;
  if (p->dtype == MOE_BF16) {
    if (acc_is_dtype)
      MOE_LAUNCH((finalize_kernel<bf, bf>), grid, 256, sm, st, (const bf*)acc, tim, p->k, dl, (const bf*)wg, p->T, p->d, p->E, (bf*)out);
    else
      MOE_LAUNCH((finalize_kernel<bf, float>), grid, 256, sm, st, (const float*)acc, tim, p->k, dl, (const bf*)wg, p->T, p->d, p->E,
                 (bf*)out);
  } else {
    MOE_LAUNCH((finalize_kernel<float, float>), grid, 256, sm, st, (const float*)acc, tim, p->k, dl, (const float*)wg, p->T, p->d,
               p->E, (float*)out);
  }
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

moe_status launch_ep_dest(const int32_t* ids, int64_t T, int k, int epr, int P, int self, int32_t* dest,
                          cudaStream_t st) {
  if (T == 0) return MOE_OK;
  MOE_LAUNCH(ep_dest_kernel, (unsigned)ceil_div(T, 256), 256, 0, st, ids, T, k, epr, P, self, dest);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

moe_status launch_ep_local_slots(const int32_t* ids, const float* topw, int64_t n, int epr, int rank, int32_t* lids,
                                 float* lw, cudaStream_t st) {
  if (n == 0) return MOE_OK;
  MOE_LAUNCH(ep_local_slots_kernel, (unsigned)ceil_div(n, 256), 256, 0, st, ids, topw, n, epr, rank, lids, lw);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

moe_status launch_ep_send_meta(const int32_t* ids, const float* topw, int k, int epr, int P, const int32_t* row_slot,
                               int64_t n, int32_t* send_ids, float* send_w, cudaStream_t st) {
  if (n == 0) return MOE_OK;
  MOE_LAUNCH(ep_send_meta_kernel, (unsigned)ceil_div(n * k, 256), 256, 0, st, ids, topw, k, epr, P, row_slot, n,
             send_ids, send_w);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

moe_status launch_ep_slot_grad(const int32_t* ids, int64_t T, int k, int epr, int P, const int32_t* send_pos,
                               const float* dg_back, const float* dg_local, int self, float* dg, cudaStream_t st) {
  if (T == 0) return MOE_OK;
  MOE_LAUNCH(ep_slot_grad_kernel, (unsigned)ceil_div(T * k, 256), 256, 0, st, ids, T, k, epr, P, send_pos, dg_back,
             dg_local, self, dg);
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

moe_status launch_combine_rows(const moe_problem* p, const void* rows, const int32_t* tim, const void* base, void* out,
                               cudaStream_t st) {
  const int64_t n = p->T * (p->d / 8);
  if (n == 0) return MOE_OK;
  if (p->dtype == MOE_BF16)
    MOE_LAUNCH(combine_rows_kernel<__nv_bfloat16>, (unsigned)ceil_div(n, 256), 256, 0, st,
               (const __nv_bfloat16*)rows, tim, (const __nv_bfloat16*)base, p->T, p->d, p->k, (__nv_bfloat16*)out);
  else
    MOE_LAUNCH(combine_rows_kernel<float>, (unsigned)ceil_div(n, 256), 256, 0, st, (const float*)rows, tim,
               (const float*)base, p->T, p->d, p->k, (float*)out);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

}  // namespace moeb
