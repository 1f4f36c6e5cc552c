// gemm_simt.cu — K0: CUDA-core (FMA) variants of the six expert GEMMs.
//
// Used for the MOE_FP32 storage mode, where the contract is true fp32
// arithmetic (tcgen05 has no fp32-input kind; TF32 would miss the 1e-4 gate).
// Same index logic as the tcgen05 path: rows are never copied; A operands are
// gathered through expert_token_indices, results reduced back by index.
//
// Row-kind GEMMs (M = routed rows of one expert segment, device offsets):
//   FWD_UP   : A_r, B_r = X[eti[r]] W1_e, X[eti[r]] W2_e ; U_r = SiLU(A_r) B_r     (Alg.1 l.9)
//   FWD_DOWN : Yacc[eti[r]] += w_r * U_r W3_e                                    (Alg.1 l.10)
//   BWD_DH   : dH_r = dY[eti[r]] W3_e^T ; SwiGLU bwd epilogue (dA, dB in place,
//              wU = w_r U_r, dg partials)                                        (Alg.1 l.20-28)
//   BWD_DX   : dXacc[eti[r]] += [dA_r | dB_r] [W1_e ; W2_e]^T  (K = 2h)          (Alg.1 l.30)
// Weight-grad GEMMs (K = rows of one expert):
//   DW3      : dW3_e = sum_r dY[eti[r]]^T (w_r U_r)                              (Alg.1 l.18)
//   DW12     : [dW1_e ; dW2_e] = sum_r [dA_r | dB_r]^T X[eti[r]]                 (Alg.1 l.29)
#include "gemm.h"

namespace moeb {

enum RowsMode { FWD_UP = 0, FWD_DOWN = 1, BWD_DH = 2, BWD_DX = 3 };
enum WgradMode { DW3 = 0, DW12 = 1 };

constexpr int SB = 64, SK = 16, ST = 256;

template <typename T>
struct SimtArgs {
  const T* x; const T* dy; const T* w1; const T* w2; const T* w3;
  const float* topw; const int32_t* offs; const int32_t* eti; const int32_t* row_slot;
  T* a_save; T* b_save; T* u;            // [R, h]
  float* acc_out;                        // Yacc or dXacc [T, d]
  float* dg_part;                        // [R, nparts]
  T* dw_a; T* dw_b;                      // DW3: dw3 ; DW12: dw1, dw2
  int64_t R; int d, h, E;
  int act;                               // 0 SwiGLU (gated); 1 SiLU, 2 ReLU (non-gated)
  int out_mode;                          // FWD_DOWN / BWD_DX target (gemm.h OutMode)
  T* out_tok;                            // OUT_TOKN destination [T, d]
  int u_weighted;                        // MOE_CKPT_ABU: u holds w * U (FWD_UP writes it, FWD_DOWN adds it unscaled)
  int dh_skip_u;                         // MOE_CKPT_ABU: BWD_DH leaves u (the saved wU) untouched
};

template <typename T>
__device__ __forceinline__ void simt_out(const SimtArgs<T>& g, int64_t r, int64_t t, int n, float v) {
  switch (g.out_mode) {
    case OUT_RED: atomicAdd(&g.acc_out[t * g.d + n], v); break;
    case OUT_ROWS: g.acc_out[r * g.d + n] = v; break;
    case OUT_TOK: g.acc_out[t * g.d + n] = v; break;
    default: g.out_tok[t * g.d + n] = from_f32<T>(v); break;
  }
}

template <typename T, int MODE>
__global__ void __launch_bounds__(ST) simt_rows_kernel(SimtArgs<T> g) {
  __shared__ float As[SK][SB + 4];
  __shared__ float Bs[2][SK][SB + 4];
  __shared__ int tstart[257];
  __shared__ float red[SB][17];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int E = g.E;
  if (tid == 0) {
    int s = 0;
    for (int e = 0; e < E; ++e) { tstart[e] = s; s += (int)ceil_div(g.offs[e + 1] - g.offs[e], SB); }
    tstart[E] = s;
  }
  __syncthreads();
  const int mt = blockIdx.x;
  if (mt >= tstart[E]) return;
  const int e = find_segment(tstart, E, mt);
  const int seg0 = g.offs[e], seg1 = g.offs[e + 1];
  const int r0 = seg0 + (mt - tstart[e]) * SB;
  const bool gated = g.act == 0;
  const int N = (MODE == FWD_UP || MODE == BWD_DH) ? g.h : g.d;
  const int K = (MODE == FWD_UP || MODE == BWD_DH) ? g.d : (MODE == FWD_DOWN ? g.h : (gated ? 2 : 1) * g.h);
  const int n0 = blockIdx.y * SB;
  const int64_t hd = (int64_t)g.h * g.d;
  float acc[2][4][4];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[q][i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += SK) {
    for (int i = tid; i < SB * SK; i += ST) {
      int rr = i / SK, kk = i % SK;
      int r = r0 + rr, kg = k0 + kk;
      float v = 0.f;
      if (r < seg1 && kg < K) {
        if (MODE == FWD_UP) v = to_f32(g.x[(int64_t)g.eti[r] * g.d + kg]);
        else if (MODE == BWD_DH) v = to_f32(g.dy[(int64_t)g.eti[r] * g.d + kg]);
        else if (MODE == FWD_DOWN) v = to_f32(g.u[(int64_t)r * g.h + kg]);
        else v = kg < g.h ? to_f32(g.a_save[(int64_t)r * g.h + kg]) : to_f32(g.b_save[(int64_t)r * g.h + kg - g.h]);
      }
      As[kk][rr] = v;
    }
    for (int i = tid; i < SB * SK; i += ST) {
      int kk = i / SB, nn = i % SB;
      int kg = k0 + kk, n = n0 + nn;
      float v0 = 0.f, v1 = 0.f;
      if (kg < K && n < N) {
        if (MODE == FWD_UP) {
          v0 = to_f32(g.w1[e * hd + (int64_t)n * g.d + kg]);
          v1 = gated ? to_f32(g.w2[e * hd + (int64_t)n * g.d + kg]) : 0.f;
        } else if (MODE == FWD_DOWN) {
          v0 = to_f32(g.w3[e * hd + (int64_t)n * g.h + kg]);
        } else if (MODE == BWD_DH) {
          v0 = to_f32(g.w3[e * hd + (int64_t)kg * g.h + n]);
        } else {
          v0 = kg < g.h ? to_f32(g.w1[e * hd + (int64_t)kg * g.d + n]) : to_f32(g.w2[e * hd + (int64_t)(kg - g.h) * g.d + n]);
        }
      }
      Bs[0][kk][nn] = v0;
      if (MODE == FWD_UP) Bs[1][kk][nn] = v1;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK; ++kk) {
      float a[4], b0[4], b1[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) { b0[j] = Bs[0][kk][tx * 4 + j]; if (MODE == FWD_UP) b1[j] = Bs[1][kk][tx * 4 + j]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[0][i][j] = fmaf(a[i], b0[j], acc[0][i][j]);
          if (MODE == FWD_UP) acc[1][i][j] = fmaf(a[i], b1[j], acc[1][i][j]);
        }
    }
    __syncthreads();
  }
  // epilogue
  float rowsum[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty * 4 + i;
    const bool rv = r < seg1;
    const int slot = rv ? g.row_slot[r] : 0;
    const float w = rv ? ((MODE == FWD_DOWN && g.u_weighted) ? 1.f : g.topw[slot]) : 0.f;
    const float uw = (MODE == FWD_UP && g.u_weighted) ? w : 1.f;  // scale of the stored U
    const int64_t t = rv ? g.eti[r] : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (!rv || n >= N) continue;
      if (MODE == FWD_UP) {
        float a = acc[0][i][j], b = acc[1][i][j];
        int64_t o = (int64_t)r * g.h + n;
        g.a_save[o] = from_f32<T>(a);
        if (gated) {
          g.b_save[o] = from_f32<T>(b);
          g.u[o] = from_f32<T>(uw * (a * sigmoidf_(a) * b));
        } else {
          g.u[o] = from_f32<T>(uw * act_fwd(g.act, a, sigmoidf_(a)));
        }
      } else if (MODE == FWD_DOWN) {
        simt_out(g, r, t, n, w * acc[0][i][j]);
      } else if (MODE == BWD_DH) {
        int64_t o = (int64_t)r * g.h + n;
        const float a = to_f32(g.a_save[o]), dH = acc[0][i][j], s = sigmoidf_(a), dU = w * dH;
        if (gated) {
          const float b = to_f32(g.b_save[o]), S = a * s, U = S * b;
          rowsum[i] += dH * U;
          g.a_save[o] = from_f32<T>(dU * b * s * (1.f + a * (1.f - s)));
          g.b_save[o] = from_f32<T>(dU * S);
          if (!g.dh_skip_u) g.u[o] = from_f32<T>(w * U);
        } else {
          const float U = act_fwd(g.act, a, s);
          rowsum[i] += dH * U;
          g.a_save[o] = from_f32<T>(dU * act_grad(g.act, a, s));
          if (!g.dh_skip_u) g.u[o] = from_f32<T>(w * U);
        }
      } else {
        simt_out(g, r, t, n, acc[0][i][j]);
      }
    }
  }
  if (MODE == BWD_DH) {
#pragma unroll
    for (int i = 0; i < 4; ++i) red[ty * 4 + i][tx] = rowsum[i];
    __syncthreads();
    if (tid < SB) {
      const int r = r0 + tid;
      if (r < seg1) {
        float s = 0.f;
        for (int q = 0; q < 16; ++q) s += red[tid][q];
        const int nparts = (int)ceil_div(g.h, SB);
        g.dg_part[(int64_t)r * nparts + blockIdx.y] = s;
      }
    }
  }
}

template <typename T, int MODE>
__global__ void __launch_bounds__(ST) simt_wgrad_kernel(SimtArgs<T> g) {
  __shared__ float As[SK][SB + 4];
  __shared__ float Bs[SK][SB + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int e = blockIdx.z;
  const int M = MODE == DW3 ? g.d : (g.act == 0 ? 2 : 1) * g.h;
  const int N = MODE == DW3 ? g.h : g.d;
  const int m0 = blockIdx.y * SB, n0 = blockIdx.x * SB;
  const int seg0 = g.offs[e], seg1 = g.offs[e + 1];
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = seg0; k0 < seg1; k0 += SK) {
    for (int i = tid; i < SB * SK; i += ST) {
      int kk = i / SB, mm = i % SB;
      int r = k0 + kk, m = m0 + mm;
      float v = 0.f;
      if (r < seg1 && m < M) {
        if (MODE == DW3) v = to_f32(g.dy[(int64_t)g.eti[r] * g.d + m]);
        else v = m < g.h ? to_f32(g.a_save[(int64_t)r * g.h + m]) : to_f32(g.b_save[(int64_t)r * g.h + m - g.h]);
      }
      As[kk][mm] = v;
      int n = n0 + mm;
      float u = 0.f;
      if (r < seg1 && n < N) {
        if (MODE == DW3) u = to_f32(g.u[(int64_t)r * g.h + n]);
        else u = to_f32(g.x[(int64_t)g.eti[r] * g.d + n]);
      }
      Bs[kk][mm] = u;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int64_t hd = (int64_t)g.h * g.d;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      if (MODE == DW3) g.dw_a[e * hd + (int64_t)m * g.h + n] = from_f32<T>(acc[i][j]);
      else if (m < g.h) g.dw_a[e * hd + (int64_t)m * g.d + n] = from_f32<T>(acc[i][j]);
      else g.dw_b[e * hd + (int64_t)(m - g.h) * g.d + n] = from_f32<T>(acc[i][j]);
    }
  }
}

int simt_dg_parts(int h) { return (int)ceil_div(h, SB); }

template <typename T>
static moe_status simt_launch_all(int which, const SimtArgs<T>& g, cudaStream_t st) {
  const unsigned mtiles = (unsigned)(ceil_div(g.R, SB) + g.E);
  switch (which) {
    case 0: MOE_LAUNCH((simt_rows_kernel<T, FWD_UP>), dim3(mtiles, ceil_div(g.h, SB)), ST, 0, st, g); break;
    case 1: MOE_LAUNCH((simt_rows_kernel<T, FWD_DOWN>), dim3(mtiles, ceil_div(g.d, SB)), ST, 0, st, g); break;
    case 2: MOE_LAUNCH((simt_rows_kernel<T, BWD_DH>), dim3(mtiles, ceil_div(g.h, SB)), ST, 0, st, g); break;
    case 3: MOE_LAUNCH((simt_rows_kernel<T, BWD_DX>), dim3(mtiles, ceil_div(g.d, SB)), ST, 0, st, g); break;
    case 4: MOE_LAUNCH((simt_wgrad_kernel<T, DW3>), dim3(ceil_div(g.h, SB), ceil_div(g.d, SB), g.E), ST, 0, st, g); break;
    case 5: MOE_LAUNCH((simt_wgrad_kernel<T, DW12>), dim3(ceil_div(g.d, SB), ceil_div((g.act == 0 ? 2 : 1) * g.h, SB), g.E), ST, 0, st, g); break;
  }
  MOE_CUDA_CHECK(cudaGetLastError());
  return MOE_OK;
}

moe_status simt_gemm(const GemmCall& c, cudaStream_t st) {
  if (c.bf16) {
    using T = __nv_bfloat16;
    SimtArgs<T> g{(const T*)c.x, (const T*)c.dy, (const T*)c.w1, (const T*)c.w2, (const T*)c.w3, c.topw, c.offs, c.eti,
                  c.row_slot, (T*)c.a_save, (T*)c.b_save, (T*)c.u, c.acc_out, c.dg_part, (T*)c.dw_a, (T*)c.dw_b,
                  c.R, c.d, c.h, c.E, c.act, c.out_mode, (T*)c.out_tok, c.u_weighted, c.dh_skip_u};
    return simt_launch_all<T>(c.which, g, st);
  }
  using T = float;
  SimtArgs<T> g{(const T*)c.x, (const T*)c.dy, (const T*)c.w1, (const T*)c.w2, (const T*)c.w3, c.topw, c.offs, c.eti,
                c.row_slot, (T*)c.a_save, (T*)c.b_save, (T*)c.u, c.acc_out, c.dg_part, (T*)c.dw_a, (T*)c.dw_b,
                c.R, c.d, c.h, c.E, c.act, c.out_mode, (T*)c.out_tok, c.u_weighted, c.dh_skip_u};
  return simt_launch_all<T>(c.which, g, st);
}

}  // namespace moeb
