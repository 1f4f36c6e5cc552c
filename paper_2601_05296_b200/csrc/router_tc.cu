// router_tc.cu — the router backward's two contractions on sm_100a tensor
// cores (bf16 runs; fp32 storage keeps the CUDA-core kernels of
// elementwise.cu).  Not in the paper: the analytic derivative of P:42/P:91
// through the softmax (reading #14), K9/K10 of SURVEY §8(a) row a9.
//
//   RDX: dx[t, :] = bf16(acc[t, :] + dl[t, :] W_g), the finalisation of dX fused
//        with the router term (acc: the fp32 accumulator the dX GEMM red.added
//        into, the EP partial dX in bf16, or the ordered-combine rows through tim).
//        M = 128 tokens, N = 256 columns of d, K = E (64-wide chunks, zero-padded).
//        (LOAD = false stores dl W_g alone, fp32: kept for measurement; adding
//        the router term first would make the k = 2 red.add order-dependent.)
//   DWG: part[s][e][c] = sum_{t in split s} dl[t, e] X[t, c], then the
//        fixed-order dwg_reduce sums the splits (deterministic).
//        M = 128 columns of d (A = X^T, MN-major), N = E padded to 64, K = tokens
//
// dl (dlogits, fp32) enters the bf16 MMA as the split dl = hi + lo
// (hi = bf16(dl), lo = bf16(dl - hi), exact to ~2^-17 relative), written by the
// router-backward kernel as two [T, Ep8] bf16 tensors (Ep8 = E rounded up to 8,
// zero columns): two MMAs per K16 step into one fp32 TMEM accumulator, so the
// products carry ~fp32 accuracy (X and W_g are bf16 already).  Every operand
// arrives by TMA; one elected thread issues the MMAs.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ptx.cuh"

namespace moeb {

template <typename A>
__device__ __forceinline__ float4 ld_acc4(const A* p);
template <>
__device__ __forceinline__ float4 ld_acc4<float>(const float* p) { return *reinterpret_cast<const float4*>(p); }
template <>
__device__ __forceinline__ float4 ld_acc4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 a = ptx::unpack_bf16(u.x), b = ptx::unpack_bf16(u.y);
  return make_float4(a.x, a.y, b.x, b.y);
}

// ---------------------------------------------------------------- RDX
// 256 threads: warp w reads TMEM lane quadrant w & 3, column half w >> 2.  Two CTAs per SM
// (<= 128 registers, 2 x 99 KB smem, 2 x 256 TMEM columns) keep twice the accumulator rows in flight.
// smem: [A_hi 16 KB][A_lo 16 KB][B 32 KB: 4 MN-major panels of 64 cols x 64 e][staging 8 x 4 KB][barriers]
constexpr int RDX_THREADS = 256;
constexpr int RDX_SMEM = 16384 * 2 + 32768 + 8 * 4096 + 64 + 1024;

#ifndef RDX_L2PF
#define RDX_L2PF 1  // router dX / finalise: L2 prefetch of the tile's accumulator rows before its MMA
                    // (ncu 61.5 -> 57.3 us DeepSeek-like, in-step 80 -> 73 / 87 -> 80 us; profiles/variants_r02aw_rdx_l2pf.txt)
#endif
template <bool LOAD, typename A>
__global__ void __launch_bounds__(RDX_THREADS, 2)
router_dx_tc_kernel(const __grid_constant__ CUtensorMap mDh, const __grid_constant__ CUtensorMap mDl,
                    const __grid_constant__ CUtensorMap mWg, const A* __restrict__ acc, const int32_t* __restrict__ tim,
                    int k, int64_t Tn, int d, int E, void* __restrict__ out_) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sAh = smem;
  uint8_t* sAl = smem + 16384;
  uint8_t* sB = smem + 32768;
  uint8_t* stg_all = smem + 65536;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 65536 + 8 * 4096);  // [0] tma, [1] mma
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, half = warp >> 2;
  // persistent: the CTA walks tiles (128 tokens x 256 columns) ti = blockIdx.x + i * gridDim.x,
  // columns fastest; barriers, TMEM and the tensor-map prefetch are set up once per CTA (the
  // per-CTA setup of 1 024 short CTAs was half the kernel's time)
  const int ntn = (int)ceil_div(d, 256);
  const int64_t ntiles = ceil_div(Tn, 128) * ntn;
  int64_t t0 = 0;
  int n0 = 0;
  // the epilogue's accumulator rows (the kernel's bulk traffic) do not depend on the MMA:
  // chunk c of this warp (32 tokens x 32 columns, row-coalesced) is loaded into registers
  // one chunk ahead, the first before the tile's MMA is even issued
  auto load_chunk = [&](int c, float4 (&a)[8]) {
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int rr = it * 4 + (lane >> 3), q = lane & 7;
      const int64_t t = t0 + quad * 32 + rr;
      const int64_t col = n0 + c + 4 * q;
      a[it] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (LOAD && t < Tn && n0 + c < d) {
        if (!tim) {
          a[it] = ld_acc4<A>(acc + t * d + col);
        } else {  // ordered combine (NEXT-4): the token's routed rows in slot order, -1 skipped
          for (int j = 0; j < k; ++j) {
            const int r = tim[t * k + j];
            if (r < 0) continue;
            const float4 b = ld_acc4<A>(acc + (int64_t)r * d + col);
            a[it].x += b.x; a[it].y += b.y; a[it].z += b.z; a[it].w += b.w;
          }
        }
      }
    }
  };
  if (tid == 0) {
    ptx::tma_prefetch(&mDh);
    ptx::tma_prefetch(&mDl);
    ptx::tma_prefetch(&mWg);
    ptx::mbar_init(&bars[0], 1);
    ptx::mbar_init(&bars[1], 2);  // two commits per K chunk (hi, lo)
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(tmem_holder, 256);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  constexpr uint32_t IDESC = ptx::umma_idesc_bf16(128, 256, 0, 1);
  const int nkc = (int)ceil_div(E, 64);
  uint32_t gk = 0;  // K chunks issued by this CTA so far (barrier phases)
  uint8_t* stg = stg_all + warp * 4096;
  const uint32_t tb = tmem + ((uint32_t)(quad * 32) << 16);
  float4 a_cur[8];
#pragma unroll 1
  for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x, gk += nkc) {
    t0 = (ti / ntn) * 128;
    n0 = (int)(ti - (ti / ntn) * ntn) * 256;
    // this warp's whole accumulator region (32 rows x 128 columns: 128 lines) of tile tt to L2,
    // so the epilogue's one-chunk-ahead register loads hit L2, not HBM
    auto prefetch_tile = [&](int64_t tt) {
      if constexpr (RDX_L2PF && LOAD) {
        if (tim || tt >= ntiles) return;
        const int64_t pt0 = (tt / ntn) * 128;
        const int pn0 = (int)(tt - (tt / ntn) * ntn) * 256;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int L = lane + 32 * i, row = L >> 2, seg = L & 3;
          const int64_t t = pt0 + quad * 32 + row;
          const int64_t col = pn0 + half * 128 + seg * 32;
          if (t < Tn && col < d) ptx::prefetch_l2(acc + t * d + col);
        }
      }
    };
    prefetch_tile(ti);  // before the tile's MMA (a whole epilogue ahead, for the next tile, measured slower)
    load_chunk(half * 128, a_cur);
    if (warp == 0) {
      for (int kc = 0; kc < nkc; ++kc) {
        const uint32_t g = gk + kc;
        const int e0 = kc * 64;
        if (kc > 0) ptx::mbar_wait(&bars[1], (g - 1) & 1);  // previous chunk's MMAs done: smem free
        if (lane == 0) {
          ptx::mbar_arrive_expect_tx(&bars[0], 65536);
          ptx::tma_load_2d(sAh, &mDh, &bars[0], e0, (int)t0);
          ptx::tma_load_2d(sAl, &mDl, &bars[0], e0, (int)t0);
#pragma unroll
          for (int p = 0; p < 4; ++p) ptx::tma_load_2d(sB + p * 8192, &mWg, &bars[0], n0 + 64 * p, e0);
        }
        __syncwarp();
        ptx::mbar_wait(&bars[0], g & 1);
        ptx::tc_fence_after();
        const uint32_t bl = (ptx::smem_u32(sB) >> 4) | ((8192u >> 4) << 16);
        ptx::umma_kblock<1, 2, 128>(tmem, (ptx::smem_u32(sAh) >> 4) | (1u << 16), bl, IDESC, kc > 0,
                                    ptx::smem_u32(&bars[1]), 0);
        ptx::umma_kblock<1, 2, 128>(tmem, (ptx::smem_u32(sAl) >> 4) | (1u << 16), bl, IDESC, 1u,
                                    ptx::smem_u32(&bars[1]), 0);
      }
      // (only warp 0 tracks the chunk phases: a late waiter on a parity that repeats
      // every two chunks could pass on an earlier chunk's completion)
      ptx::mbar_wait(&bars[1], (gk + nkc - 1) & 1);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    // epilogue: 32 tokens x 128 columns per warp in 32-column chunks, staged through a
    // swizzled fp32 tile so the global accesses are row-coalesced
#pragma unroll 1
    for (int c = half * 128; c < half * 128 + 128; c += 32) {
      if (n0 + c >= d) break;
      uint32_t v[32];
      ptx::tmem_ld32(tb + c, v);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(stg + lane * 128 + ((q ^ (lane & 7)) << 4)) =
            make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                        __uint_as_float(v[4 * q + 3]));
      __syncwarp();
      float4 a[8];
#pragma unroll
      for (int it = 0; it < 8; ++it) a[it] = a_cur[it];
      if (c + 32 < half * 128 + 128) load_chunk(c + 32, a_cur);  // next chunk in flight
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int rr = it * 4 + (lane >> 3), q = lane & 7;
        const int64_t t = t0 + quad * 32 + rr;
        if (t < Tn) {
          const float4 f = *reinterpret_cast<const float4*>(stg + rr * 128 + ((q ^ (rr & 7)) << 4));
          const int64_t o = t * d + n0 + c + 4 * q;
          if constexpr (LOAD) {
            *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out_) + o) = make_uint2(
                ptx::pack_bf16(a[it].x + f.x, a[it].y + f.y), ptx::pack_bf16(a[it].z + f.z, a[it].w + f.w));
          } else {
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(out_) + o) = f;
          }
        }
      }
      __syncwarp();
    }
    // every warp's TMEM reads are complete before the next tile's MMAs overwrite the accumulator
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  }
  if (warp == 0) ptx::tmem_dealloc(tmem, 256);
}

// ---------------------------------------------------------------- DWG
// Stage: A = X[t .. t+63, c0 .. c0+127] as two MN-major 64-column panels (16 KB);
// B_hi, B_lo = dl_hi / dl_lo [t .. t+63, 0 .. NB) as NB/64 MN-major panels each.
// Warp 0: TMA producer; warp 1: MMA issuer; all four warps: epilogue.
template <int NB>
struct DwgCfg {
  static constexpr int STAGE = 16384 + 2 * NB * 128;
  static constexpr int STAGES = (200 * 1024) / STAGE > 6 ? 6 : (200 * 1024) / STAGE;
  static constexpr int TMEM_COLS = NB <= 64 ? 64 : (NB <= 128 ? 128 : 256);
  static constexpr int SMEM = STAGES * STAGE + 256 + 1024;
};

template <int NB>
__global__ void __launch_bounds__(128, 1)
router_dwg_tc_kernel(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mDh,
                     const __grid_constant__ CUtensorMap mDl, int64_t Tn, int d, int E, int64_t tch,
                     float* __restrict__ part) {
  using C = DwgCfg<NB>;
  constexpr int S = C::STAGES;
  constexpr int NP = NB / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::STAGE);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c0 = blockIdx.x * 128;
  const int64_t ta = (int64_t)blockIdx.y * tch, tbnd = min64(ta + tch, Tn);
  const int nk = tbnd > ta ? (int)ceil_div(tbnd - ta, 64) : 0;
  if (tid == 0) {
    ptx::tma_prefetch(&mX);
    ptx::tma_prefetch(&mDh);
    ptx::tma_prefetch(&mDl);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 2);  // hi + lo commits
    }
    ptx::mbar_init(done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(tmem_holder, C::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  constexpr uint32_t IDESC = ptx::umma_idesc_bf16(128, NB, 1, 1);
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % S;
        if (kb >= S) ptx::mbar_wait(&empty[s], ((kb / S) - 1) & 1);
        uint8_t* sA = smem + s * C::STAGE;
        uint8_t* sBh = sA + 16384;
        uint8_t* sBl = sBh + NB * 128;
        const int tk = (int)(ta + (int64_t)kb * 64);
        ptx::mbar_arrive_expect_tx(&full[s], C::STAGE);
        ptx::tma_load_2d(sA, &mX, &full[s], c0, tk);
        ptx::tma_load_2d(sA + 8192, &mX, &full[s], c0 + 64, tk);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          ptx::tma_load_2d(sBh + p * 8192, &mDh, &full[s], 64 * p, tk);
          ptx::tma_load_2d(sBl + p * 8192, &mDl, &full[s], 64 * p, tk);
        }
      }
    }
  } else if (warp == 1) {
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % S;
      ptx::mbar_wait(&full[s], (kb / S) & 1);
      uint8_t* sA = smem + s * C::STAGE;
      const int64_t tk = ta + (int64_t)kb * 64;
      if (tk + 64 > tbnd && tbnd < Tn) {
        // the split's last block straddles into the next split: zero the dl rows of
        // tokens >= tbnd in smem (MN-major panels: k-row r of panel p at p*8192 +
        // r*128, whole 128-byte rows, so the swizzle does not matter)
        const int r0 = (int)(tbnd - tk), nr = 64 - r0;
        for (int i = lane; i < nr * 2 * NP * 8; i += 32) {
          const int ch = i & 7, rest = i >> 3;
          const int r = r0 + rest % nr, pp = rest / nr;  // pp: panel (hi panels, then lo panels)
          *reinterpret_cast<uint4*>(sA + 16384 + pp * 8192 + r * 128 + ch * 16) = make_uint4(0, 0, 0, 0);
        }
        ptx::fence_proxy_async();
        __syncwarp();
      }
      ptx::tc_fence_after();
      const uint32_t al = (ptx::smem_u32(sA) >> 4) | ((8192u >> 4) << 16);
      const uint32_t bh = (ptx::smem_u32(sA + 16384) >> 4) | ((8192u >> 4) << 16);
      const uint32_t bl = (ptx::smem_u32(sA + 16384 + NB * 128) >> 4) | ((8192u >> 4) << 16);
      ptx::umma_kblock<1, 128, 128>(tmem, al, bh, IDESC, kb > 0, ptx::smem_u32(&empty[s]), 0);
      ptx::umma_kblock<1, 128, 128>(tmem, al, bl, IDESC, 1u, ptx::smem_u32(&empty[s]), 0);
    }
    if (nk > 0) {
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
              ptx::smem_u32(done))
          : "memory");
    } else if (lane == 0) {
      ptx::mbar_arrive(done);
    }
  }
  ptx::mbar_wait(done, 0);
  ptx::tc_fence_after();
  // epilogue: thread (warp w, lane l) owns column c0 + 32w + l; its accumulator
  // columns are the experts -> part[split][e][col] (coalesced across the warp)
  const int col = c0 + warp * 32 + lane;
  float* dst = part + (int64_t)blockIdx.y * E * d + col;
  const uint32_t tb = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
  for (int e0 = 0; e0 < E; e0 += 32) {
    uint32_t v[32];
    if (nk > 0) {
      ptx::tmem_ld32(tb + e0, v);
      ptx::tmem_wait_ld();
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0u;
    }
    if (col < d) {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (e0 + i < E) dst[(int64_t)(e0 + i) * d] = __uint_as_float(v[i]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ----------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 rt_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// bf16 row-major [rows, cols] (row pitch `pitch` elements), box 64 cols x box_rows, 128B swizzle, OOB zero fill
static bool rt_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t pitch, uint32_t box_rows) {
  auto fn = rt_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int rt_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = 0;
    if (n <= 0) n = 148;
  }
  return n;
}

int router_ep8(int E) { return (int)ceil_div(E, 8) * 8; }

// token splits of the DWG contraction: one CTA per SM over (d/128) column tiles,
// at least 4 k-blocks (256 tokens) per split, at most 256 splits
int router_dwg_tc_splits(int64_t T, int d) {
  const int64_t mt = ceil_div(d, 128);
  int64_t s = std::max<int64_t>(1, rt_sms() / mt);
  s = std::min<int64_t>(s, std::max<int64_t>(1, T / 256));
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, 256));
}

template <int NB>
static moe_status launch_dwg_nb(const CUtensorMap& mx, const CUtensorMap& mh, const CUtensorMap& ml, int64_t T, int d,
                                int E, int splits, int64_t tch, float* part, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(router_dwg_tc_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             DwgCfg<NB>::SMEM) != cudaSuccess)
      return MOE_ERR_CUDA;
    attr = true;
  }
  dim3 grid((unsigned)ceil_div(d, 128), (unsigned)splits);
  router_dwg_tc_kernel<NB><<<grid, 128, DwgCfg<NB>::SMEM, st>>>(mx, mh, ml, T, d, E, tch, part);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

// dlhl: dl_hi [T, Ep8] then dl_lo [T, Ep8] (bf16); part: [splits][E][d] fp32
moe_status launch_router_dwg_tc(const __nv_bfloat16* dlhl, const void* x, int64_t T, int d, int E, float* part,
                                cudaStream_t st) {
  const int ep8 = router_ep8(E);
  const uint64_t rows = (uint64_t)std::max<int64_t>(T, 1);
  CUtensorMap mx, mh, ml;
  if (!rt_map(&mx, x, rows, d, d, 64) || !rt_map(&mh, dlhl, rows, ep8, ep8, 64) ||
      !rt_map(&ml, dlhl + (size_t)T * ep8, rows, ep8, ep8, 64))
    return MOE_ERR_CUDA;
  const int splits = router_dwg_tc_splits(T, d);
  const int64_t tch = ceil_div(std::max<int64_t>(T, 1), splits);
  if (E <= 64) return launch_dwg_nb<64>(mx, mh, ml, T, d, E, splits, tch, part, st);
  if (E <= 128) return launch_dwg_nb<128>(mx, mh, ml, T, d, E, splits, tch, part, st);
  if (E <= 192) return launch_dwg_nb<192>(mx, mh, ml, T, d, E, splits, tch, part, st);
  return launch_dwg_nb<256>(mx, mh, ml, T, d, E, splits, tch, part, st);
}

// load = false: out = fp32 [T, d] := dl W_g (acc unused).  load = true: out = bf16
// [T, d] := bf16(acc + dl W_g), acc [T, d] fp32 (or bf16 when acc_is_dtype), or with
// tim the [R, d] row-result buffer summed per token in slot order (NEXT-4).
moe_status launch_router_dx_tc(bool load, const void* acc, bool acc_is_dtype, const int32_t* tim, int k,
                               const __nv_bfloat16* dlhl, const void* wg, int64_t T, int d, int E, void* out,
                               cudaStream_t st) {
  if (T == 0) return MOE_OK;
  const int ep8 = router_ep8(E);
  CUtensorMap mh, ml, mw;
  if (!rt_map(&mh, dlhl, T, ep8, ep8, 128) || !rt_map(&ml, dlhl + (size_t)T * ep8, T, ep8, ep8, 128) ||
      !rt_map(&mw, wg, E, d, d, 64))
    return MOE_ERR_CUDA;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(router_dx_tc_kernel<true, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             RDX_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(router_dx_tc_kernel<true, __nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             RDX_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(router_dx_tc_kernel<false, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             RDX_SMEM) != cudaSuccess)
      return MOE_ERR_CUDA;
    attr = true;
  }
  // persistent: two CTAs per SM (the kernel's occupancy), each walking its share of the tiles
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  const int64_t ntiles = ceil_div(T, 128) * ceil_div(d, 256);
  const dim3 grid((unsigned)std::min<int64_t>(ntiles, 2LL * n_sm));
  if (!load)
    router_dx_tc_kernel<false, float><<<grid, RDX_THREADS, RDX_SMEM, st>>>(mh, ml, mw, nullptr, nullptr, k, T, d, E,
                                                                          out);
  else if (acc_is_dtype)
    router_dx_tc_kernel<true, __nv_bfloat16><<<grid, RDX_THREADS, RDX_SMEM, st>>>(
        mh, ml, mw, (const __nv_bfloat16*)acc, tim, k, T, d, E, out);
  else
    router_dx_tc_kernel<true, float><<<grid, RDX_THREADS, RDX_SMEM, st>>>(mh, ml, mw, (const float*)acc, tim, k, T,
                                                                         d, E, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

}  // namespace moeb
