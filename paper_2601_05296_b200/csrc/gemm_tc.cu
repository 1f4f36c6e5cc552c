// gemm_tc.cu — the six expert GEMMs of the MoE layer on sm_100a tensor cores.
//
// One persistent, warp-specialised kernel template (tcgen05.mma kind::f16,
// bf16 operands, fp32 accumulators in TMEM, operands staged by TMA):
//   warp 0      TMA producer: tile loads + row-GATHER loads (tile::gather4)
//               straight from the unpermuted X / dY through
//               expert_token_indices — no routed-token buffer
//   warp 1      MMA issuer (one thread): 4 x tcgen05.mma (M128 N256 K16) per
//               64-wide K block, tcgen05.commit frees the smem stage
//   warp 2      TMEM allocator (512 columns = 2 accumulator stages x 256)
//   warps 4-7   epilogue: tcgen05.ld one row per thread, fused epilogue
// Tile = 128 rows x 256 columns; smem ring of 4 stages x (16 KB A + 32 KB B),
// 128B-swizzled, K-major or MN-major UMMA descriptors as the operand's
// global layout dictates (no transposes are ever materialised).
//
// Kinds ("rows" = the routed rows of one expert segment, read from device
// expert_token_offsets: no host sync):
//   FWD_UP   M=rows N=2x128 K=d  A=gather X (K-major)     B=[W1;W2] stacked   epi: A,B saved, U=SiLU(A)B   Alg.1 l.9
//   FWD_DOWN M=rows N=256   K=h  A=U rows (K-major)       B=W3 (K-major)      epi: red.add w*O -> Yacc      Alg.1 l.10
//   BWD_DH   M=rows N=256   K=d  A=gather dY (K-major)    B=W3 (MN-major)     epi: SwiGLU bwd, dA/dB in place,
//                                                                               wU, gate-grad partials   Alg.1 l.20-28
//   BWD_DX   M=rows N=256   K=2h A=dA|dB rows (K-major)   B=W1|W2 (MN-major)  epi: red.add -> dXacc        Alg.1 l.30
//   DW3      M=d    N=256   K=rows A=gather dY (MN-major) B=wU rows (MN)      epi: store dW3_e             Alg.1 l.18
//   DW12     M=2h   N=256   K=rows A=dA|dB rows (MN)      B=gather X (MN)     epi: store dW1_e, dW2_e      Alg.1 l.29
// Rows past a segment end gather the out-of-bounds row T, which TMA fills with
// zeros: this zero-pads the K tail of the weight-gradient GEMMs in shared
// memory only (no padded buffer exists in HBM).
#include <cudaTypedefs.h>
#include <cstdlib>

#include "gemm.h"
#include "ptx.cuh"

namespace moeb {

enum TcKind { TC_FWD_UP = 0, TC_FWD_DOWN = 1, TC_BWD_DH = 2, TC_BWD_DX = 3, TC_DW3 = 4, TC_DW12 = 5, TC_ROUTE = 6 };

constexpr int TBM = 128, TBN = 256, TBK = 64;
constexpr int TSTAGES = 4;
constexpr int TA_BYTES = TBM * TBK * 2;   // 16 KB
constexpr int TB_BYTES = TBN * TBK * 2;   // 32 KB
constexpr int TSTAGE_BYTES = TA_BYTES + TB_BYTES;
constexpr int TC_THREADS = 384;   // 12 warps: 0 TMA, 1 MMA, 2 TMEM, 4-7 epilogue, 8-11 cp.async gathers
constexpr int GATHER_THREADS = 128;
constexpr int TC_SMEM = TSTAGES * TSTAGE_BYTES + 1024 /*align*/ + 1024 /*barriers*/ + 2 * 260 * 4;

struct TcParams {
  const __nv_bfloat16* x;   // gathered operand sources for the cp.async path
  const __nv_bfloat16* dy;
  const int32_t* offs;
  const int32_t* eti;
  const int32_t* row_slot;
  const float* topw;
  __nv_bfloat16* a_save;
  __nv_bfloat16* b_save;
  __nv_bfloat16* u;
  float* acc_out;
  float* dg_part;
  __nv_bfloat16* out0;
  __nv_bfloat16* out1;
  int T, d, h, E;
  int n_tiles, m_tiles;
  int dg_parts;
  // TC_ROUTE (K1): logits = X Wg^T on tensor cores, softmax + top-k in the epilogue
  float* logits;
  int32_t* ids;
  float* route_w;
  int k, renorm, route_n;
  uint32_t route_idesc;
};

template <int KIND>
struct KindTraits {
  static constexpr bool wgrad = (KIND == TC_DW3 || KIND == TC_DW12);
  static constexpr bool a_mn = wgrad;                                     // A operand MN-major?
  static constexpr bool b_mn = (KIND == TC_BWD_DH || KIND == TC_BWD_DX || wgrad);
  static constexpr int NT = (KIND == TC_FWD_UP) ? 128 : 256;             // output columns per tile
  static constexpr bool gather_a = (KIND == TC_FWD_UP || KIND == TC_BWD_DH || KIND == TC_DW3);
  static constexpr bool gather_b = (KIND == TC_DW12);
  // bytes per stage delivered by TMA tile loads (the rest comes from row gathers)
  __host__ __device__ static constexpr uint32_t tile_bytes(bool cpa) {
    return cpa ? ((gather_a ? 0u : (uint32_t)TA_BYTES) + (gather_b ? 0u : (uint32_t)TB_BYTES))
               : (uint32_t)TSTAGE_BYTES;
  }
  static constexpr uint32_t IDESC = ptx::umma_idesc_bf16(TBM, TBN, a_mn ? 1 : 0, b_mn ? 1 : 0);
};

struct TileInfo {
  int e, m0, n0, n_tile, seg0, seg1, nk;
};

template <int KIND>
__device__ __forceinline__ bool decode_tile(int tile, const TcParams& P, const int* s_offs, const int* s_tstart,
                                            TileInfo& t) {
  using K = KindTraits<KIND>;
  if constexpr (KIND == TC_ROUTE) {
    if (tile * TBM >= P.T) return false;
    t.e = 0;
    t.seg0 = 0;
    t.seg1 = P.T;
    t.m0 = tile * TBM;
    t.n0 = 0;
    t.n_tile = 0;
    t.nk = P.d / TBK;
  } else if constexpr (K::wgrad) {
    const int per_e = P.m_tiles * P.n_tiles;
    if (tile >= P.E * per_e) return false;
    t.e = tile / per_e;
    const int rem = tile - t.e * per_e;
    const int mt = rem / P.n_tiles;
    t.n_tile = rem - mt * P.n_tiles;
    t.m0 = mt * TBM;
    t.n0 = t.n_tile * TBN;
    t.seg0 = s_offs[t.e];
    t.seg1 = s_offs[t.e + 1];
    t.nk = (t.seg1 - t.seg0 + TBK - 1) / TBK;
  } else {
    if (tile >= s_tstart[P.E]) return false;
    t.e = find_segment(s_tstart, P.E, tile);
    t.seg0 = s_offs[t.e];
    t.seg1 = s_offs[t.e + 1];
    const int mt_e = (t.seg1 - t.seg0 + TBM - 1) / TBM;
    const int local = tile - s_tstart[t.e];
    t.n_tile = local / mt_e;
    t.m0 = t.seg0 + (local - t.n_tile * mt_e) * TBM;
    t.n0 = t.n_tile * K::NT;
    const int Kdim = (KIND == TC_FWD_UP || KIND == TC_BWD_DH) ? P.d : (KIND == TC_FWD_DOWN ? P.h : 2 * P.h);
    t.nk = Kdim / TBK;
  }
  return true;
}

__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float* v) {
  uint4* p = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 q;
    q.x = ptx::pack_bf16(v[8 * i + 0], v[8 * i + 1]);
    q.y = ptx::pack_bf16(v[8 * i + 2], v[8 * i + 3]);
    q.z = ptx::pack_bf16(v[8 * i + 4], v[8 * i + 5]);
    q.w = ptx::pack_bf16(v[8 * i + 6], v[8 * i + 7]);
    p[i] = q;
  }
}
__device__ __forceinline__ void load_bf16x32(const __nv_bfloat16* src, float* v) {
  const uint4* p = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 q = p[i];
    float2 f;
    f = ptx::unpack_bf16(q.x); v[8 * i + 0] = f.x; v[8 * i + 1] = f.y;
    f = ptx::unpack_bf16(q.y); v[8 * i + 2] = f.x; v[8 * i + 3] = f.y;
    f = ptx::unpack_bf16(q.z); v[8 * i + 4] = f.x; v[8 * i + 5] = f.y;
    f = ptx::unpack_bf16(q.w); v[8 * i + 6] = f.x; v[8 * i + 7] = f.y;
  }
}

template <int KIND, bool CPA>
__global__ void __launch_bounds__(TC_THREADS, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
               const __grid_constant__ CUtensorMap mB0, const __grid_constant__ CUtensorMap mB1, const TcParams P) {
  using K = KindTraits<KIND>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TSTAGES * TSTAGE_BYTES);
  uint64_t* empty = full + TSTAGES;
  uint64_t* tfull = empty + TSTAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_offs = reinterpret_cast<int*>(smem + TSTAGES * TSTAGE_BYTES + 1024);
  int* s_tstart = s_offs + 260;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = P.E;

  if constexpr (KIND != TC_ROUTE)
    for (int i = threadIdx.x; i <= E; i += TC_THREADS) s_offs[i] = P.offs[i];
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&mA0);
    ptx::tma_prefetch(&mA1);
    ptx::tma_prefetch(&mB0);
    ptx::tma_prefetch(&mB1);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      ptx::mbar_init(&full[s], 1 + ((CPA && (K::gather_a || K::gather_b)) ? GATHER_THREADS : 0));
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 4);
    }
    ptx::fence_mbar_init();
    ptx::fence_proxy_async();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_holder, 512);
  __syncthreads();
  if (!K::wgrad && KIND != TC_ROUTE && threadIdx.x == 0) {
    int s = 0;
    for (int e = 0; e < E; ++e) {
      s_tstart[e] = s;
      s += ((s_offs[e + 1] - s_offs[e] + TBM - 1) / TBM) * P.n_tiles;
    }
    s_tstart[E] = s;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int oob = P.T;  // gather row index past the end: TMA zero-fills it

  if (warp == 0) {
    // ============================ TMA producer ============================
    int stage = 0;
    uint32_t phase = 0;
    TileInfo t;
    for (int tile = blockIdx.x; decode_tile<KIND>(tile, P, s_offs, s_tstart, t); tile += gridDim.x) {
      int gi0 = 0, gi1 = 0, gi2 = 0, gi3 = 0;
      if constexpr (!CPA && (KIND == TC_FWD_UP || KIND == TC_BWD_DH)) {
        const int r = t.m0 + 4 * lane;
        gi0 = r + 0 < t.seg1 ? P.eti[r + 0] : oob;
        gi1 = r + 1 < t.seg1 ? P.eti[r + 1] : oob;
        gi2 = r + 2 < t.seg1 ? P.eti[r + 2] : oob;
        gi3 = r + 3 < t.seg1 ? P.eti[r + 3] : oob;
      }
      for (int kb = 0; kb < t.nk; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sA = smem + stage * TSTAGE_BYTES;
        uint8_t* sB = sA + TA_BYTES;
        uint64_t* bar = &full[stage];
        if (lane == 0)
          ptx::mbar_arrive_expect_tx(bar, KIND == TC_ROUTE ? (uint32_t)(TA_BYTES + P.route_n * 128)
                                                           : K::tile_bytes(CPA));
        __syncwarp();
        const int k0 = kb * TBK;
        if constexpr (KIND == TC_ROUTE) {
          if (lane == 0) ptx::tma_load_2d(sA, &mA0, bar, k0, t.m0);
          if (lane == 1) ptx::tma_load_2d(sB, &mB0, bar, k0, 0);
        } else if constexpr (KIND == TC_FWD_UP) {
          if (!CPA) ptx::tma_gather4(sA + 512 * lane, &mA0, bar, k0, gi0, gi1, gi2, gi3);
          if (lane == 0) ptx::tma_load_2d(sB, &mB0, bar, k0, t.e * P.h + t.n0);
          if (lane == 1) ptx::tma_load_2d(sB + TB_BYTES / 2, &mB1, bar, k0, t.e * P.h + t.n0);
        } else if constexpr (KIND == TC_FWD_DOWN) {
          if (lane == 0) ptx::tma_load_2d(sA, &mA0, bar, k0, t.m0);
          if (lane == 1) ptx::tma_load_2d(sB, &mB0, bar, k0, t.e * P.d + t.n0);
        } else if constexpr (KIND == TC_BWD_DH) {
          if (!CPA) ptx::tma_gather4(sA + 512 * lane, &mA0, bar, k0, gi0, gi1, gi2, gi3);
          if (lane < 4) ptx::tma_load_2d(sB + lane * 8192, &mB0, bar, t.n0 + 64 * lane, t.e * P.d + k0);
        } else if constexpr (KIND == TC_BWD_DX) {
          const bool second = k0 >= P.h;
          const int kk = second ? k0 - P.h : k0;
          if (lane == 0) ptx::tma_load_2d(sA, second ? &mA1 : &mA0, bar, kk, t.m0);
          if (lane >= 4 && lane < 8)
            ptx::tma_load_2d(sB + (lane - 4) * 8192, second ? &mB1 : &mB0, bar, t.n0 + 64 * (lane - 4),
                             t.e * P.h + kk);
        } else if constexpr (KIND == TC_DW3) {
          if (!CPA) {
            const int g = lane & 15, p = lane >> 4;
            const int r = t.seg0 + k0 + 4 * g;
            const int i0 = r + 0 < t.seg1 ? P.eti[r + 0] : oob;
            const int i1 = r + 1 < t.seg1 ? P.eti[r + 1] : oob;
            const int i2 = r + 2 < t.seg1 ? P.eti[r + 2] : oob;
            const int i3 = r + 3 < t.seg1 ? P.eti[r + 3] : oob;
            ptx::tma_gather4(sA + p * 8192 + g * 512, &mA0, bar, t.m0 + 64 * p, i0, i1, i2, i3);
          }
          if (lane < 4) ptx::tma_load_2d(sB + lane * 8192, &mB0, bar, t.n0 + 64 * lane, t.seg0 + k0);
        } else {  // TC_DW12
          if (!CPA) {
            const int g = lane & 15, ph = lane >> 4;
            const int r = t.seg0 + k0 + 4 * g;
            const int i0 = r + 0 < t.seg1 ? P.eti[r + 0] : oob;
            const int i1 = r + 1 < t.seg1 ? P.eti[r + 1] : oob;
            const int i2 = r + 2 < t.seg1 ? P.eti[r + 2] : oob;
            const int i3 = r + 3 < t.seg1 ? P.eti[r + 3] : oob;
#pragma unroll
            for (int pp = 0; pp < 2; ++pp) {
              const int p = 2 * ph + pp;
              ptx::tma_gather4(sB + p * 8192 + g * 512, &mB0, bar, t.n0 + 64 * p, i0, i1, i2, i3);
            }
          }
          const bool second = t.m0 >= P.h;
          if (lane >= 2 && lane < 4)
            ptx::tma_load_2d(sA + (lane - 2) * 8192, second ? &mA1 : &mA0, bar,
                             (second ? t.m0 - P.h : t.m0) + 64 * (lane - 2), t.seg0 + k0);
        }
        if (++stage == TSTAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 8) {
    // ======================= cp.async row gathers (CPA) =======================
    // 128 threads copy the gathered operand 16 B at a time straight into the
    // 128B-swizzled UMMA layout (chunk c of smem row q lands at q*128 +
    // ((c ^ (q & 7)) << 4)); rows outside the expert segment are zero-filled.
    if constexpr (CPA && (K::gather_a || K::gather_b)) {
      // Lane mapping: consecutive lanes copy consecutive 16-byte chunks of the
      // same gathered row, so one warp instruction covers whole 128-byte lines.
      const int gt = threadIdx.x - 256;
      int stage = 0;
      uint32_t phase = 0;
      TileInfo t;
      const __nv_bfloat16* src_base = (KIND == TC_FWD_UP || KIND == TC_DW12) ? P.x : P.dy;
      for (int tile = blockIdx.x; decode_tile<KIND>(tile, P, s_offs, s_tstart, t); tile += gridDim.x) {
        if constexpr (KIND == TC_FWD_UP || KIND == TC_BWD_DH) {
          // K-major A, 128 rows x 8 chunks: thread -> chunk c = gt&7, rows q = (gt>>3) + 16 i
          const int c = gt & 7, rb = gt >> 3;
          const __nv_bfloat16* src[8];
          uint32_t nb[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = t.m0 + rb + 16 * i;
            const int tok = r < t.seg1 ? P.eti[r] : -1;
            src[i] = src_base + (int64_t)(tok < 0 ? 0 : tok) * P.d + c * 8;
            nb[i] = tok < 0 ? 0u : 16u;
          }
          for (int kb = 0; kb < t.nk; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t sbase = ptx::smem_u32(smem + stage * TSTAGE_BYTES);
            const int k0 = kb * TBK;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int q = rb + 16 * i;
              ptx::cp_async16(sbase + q * 128 + ((c ^ (q & 7)) << 4), src[i] + k0, nb[i]);
            }
            ptx::cp_async_mbar_arrive(&full[stage]);
            if (++stage == TSTAGES) { stage = 0; phase ^= 1; }
          }
        } else {
          // MN-major: smem row q = K index (a gathered token row); DW3 copies 2
          // panels (256 B) of dY per row, DW12 4 panels (512 B) of X per row.
          constexpr int CPR = (KIND == TC_DW3) ? 16 : 32;       // 16-byte chunks per row
          constexpr int RPI = GATHER_THREADS / CPR;             // rows per pass
          constexpr int NPASS = 64 / RPI;
          const int cidx = gt % CPR, rb = gt / CPR;
          const int p = cidx >> 3, cc = cidx & 7;
          const int col = ((KIND == TC_DW3) ? t.m0 : t.n0) + 64 * p + cc * 8;
          const bool col_ok = col < P.d;
          const uint32_t dst_off = ((KIND == TC_DW3) ? 0u : (uint32_t)TA_BYTES) + p * 8192;
          for (int kb = 0; kb < t.nk; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t sbase = ptx::smem_u32(smem + stage * TSTAGE_BYTES) + dst_off;
            const int k0 = t.seg0 + kb * TBK;
#pragma unroll
            for (int i = 0; i < NPASS; ++i) {
              const int q = rb + RPI * i;
              const int r = k0 + q;
              const int tok = (r < t.seg1 && col_ok) ? P.eti[r] : -1;
              const __nv_bfloat16* sp = src_base + (int64_t)(tok < 0 ? 0 : tok) * P.d + (col_ok ? col : 0);
              ptx::cp_async16(sbase + q * 128 + ((cc ^ (q & 7)) << 4), sp, tok < 0 ? 0u : 16u);
            }
            ptx::cp_async_mbar_arrive(&full[stage]);
            if (++stage == TSTAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    int stage = 0;
    uint32_t phase = 0;
    int as = 0;
    uint32_t aphase = 0;
    TileInfo t;
    for (int tile = blockIdx.x; decode_tile<KIND>(tile, P, s_offs, s_tstart, t); tile += gridDim.x) {
      ptx::mbar_wait(&tempty[as], aphase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + as * TBN;
      for (int kb = 0; kb < t.nk; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        if (CPA) ptx::fence_proxy_async();  // cp.async (generic proxy) writes -> tcgen05 operand reads
        ptx::tc_fence_after();
        if (lane == 0) {
          const uint32_t sA = ptx::smem_u32(smem + stage * TSTAGE_BYTES);
          const uint32_t sB = sA + TA_BYTES;
#pragma unroll
          for (int ks = 0; ks < TBK / 16; ++ks) {
            const uint64_t ad = K::a_mn ? ptx::umma_desc_sw128(sA + ks * 2048, 8192, 1024)
                                        : ptx::umma_desc_sw128(sA + ks * 32, 16, 1024);
            const uint64_t bd = K::b_mn ? ptx::umma_desc_sw128(sB + ks * 2048, 8192, 1024)
                                        : ptx::umma_desc_sw128(sB + ks * 32, 16, 1024);
            ptx::umma_bf16(d_tmem, ad, bd, KIND == TC_ROUTE ? P.route_idesc : K::IDESC, (kb | ks) != 0);
          }
          ptx::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == TSTAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) {
        if (t.nk > 0) ptx::umma_commit(&tfull[as]);
        else ptx::mbar_arrive(&tfull[as]);
      }
      __syncwarp();
      if (++as == 2) { as = 0; aphase ^= 1; }
    }
  } else if (warp >= 4 && warp < 8) {
    // ============================ epilogue ============================
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    int as = 0;
    uint32_t aphase = 0;
    TileInfo t;
    for (int tile = blockIdx.x; decode_tile<KIND>(tile, P, s_offs, s_tstart, t); tile += gridDim.x) {
      ptx::mbar_wait(&tfull[as], aphase);
      ptx::tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(wq * 32) << 16) + as * TBN;
      uint32_t v[32];
      if constexpr (KIND == TC_ROUTE) {
        // one token row per thread: logits out, softmax, top-k (desc, ties -> lower id)
        const int r = t.m0 + row;
        const bool valid = r < P.T;
        const int E = P.E;
        float mx = -INFINITY;
#pragma unroll 1
        for (int c = 0; c < P.route_n; c += 32) {
          ptx::tmem_ld32(tb + c, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (c + i < E) {
              const float f = __uint_as_float(v[i]);
              mx = fmaxf(mx, f);
              if (valid) P.logits[(int64_t)r * E + c + i] = f;
            }
          }
        }
        float sum = 0.f;
#pragma unroll 1
        for (int c = 0; c < P.route_n; c += 32) {
          ptx::tmem_ld32(tb + c, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c + i < E) sum += expf(__uint_as_float(v[i]) - mx);
        }
        uint32_t taken[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        float wsum = 0.f;
        int sel_e[16];
        float sel_p[16];
#pragma unroll 1
        for (int j = 0; j < P.k; ++j) {
          float bv = -INFINITY;
          int be = 0x7fffffff;
#pragma unroll 1
          for (int c = 0; c < P.route_n; c += 32) {
            ptx::tmem_ld32(tb + c, v);
            ptx::tmem_wait_ld();
            const uint32_t tk = taken[c >> 5];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float f = __uint_as_float(v[i]);
              if (c + i < E && !((tk >> i) & 1u) && (f > bv || (f == bv && c + i < be))) {
                bv = f;
                be = c + i;
              }
            }
          }
          taken[be >> 5] |= 1u << (be & 31);
          const float pr = expf(bv - mx) / sum;
          sel_e[j] = be;
          sel_p[j] = pr;
          wsum += pr;
        }
        if (valid) {
#pragma unroll 1
          for (int j = 0; j < P.k; ++j) {
            P.ids[(int64_t)r * P.k + j] = sel_e[j];
            P.route_w[(int64_t)r * P.k + j] = P.renorm ? sel_p[j] / wsum : sel_p[j];
          }
        }
      } else if constexpr (KIND == TC_FWD_UP) {
        const int r = t.m0 + row;
        const bool valid = r < t.seg1;
        uint32_t bv[32];
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
          ptx::tmem_ld32(tb + c, v);
          ptx::tmem_ld32(tb + 128 + c, bv);
          ptx::tmem_wait_ld();
          if (valid) {
            float a[32], b[32], u[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              a[i] = __uint_as_float(v[i]);
              b[i] = __uint_as_float(bv[i]);
              u[i] = a[i] * sigmoidf_(a[i]) * b[i];
            }
            const int64_t o = (int64_t)r * P.h + t.n0 + c;
            store_bf16x32(P.a_save + o, a);
            store_bf16x32(P.b_save + o, b);
            store_bf16x32(P.u + o, u);
          }
        }
      } else if constexpr (KIND == TC_FWD_DOWN || KIND == TC_BWD_DX) {
        const int r = t.m0 + row;
        const bool valid = r < t.seg1;
        const int N = P.d;
        float w = 1.f;
        int64_t tok = 0;
        if (valid) {
          tok = P.eti[r];
          if constexpr (KIND == TC_FWD_DOWN) w = P.topw[P.row_slot[r]];
        }
#pragma unroll 1
        for (int c = 0; c < TBN; c += 32) {
          if (t.n0 + c >= N) break;
          ptx::tmem_ld32(tb + c, v);
          ptx::tmem_wait_ld();
          if (valid) {
            float* dst = P.acc_out + tok * N + t.n0 + c;
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              ptx::red_add_v4(dst + i, w * __uint_as_float(v[i]), w * __uint_as_float(v[i + 1]),
                              w * __uint_as_float(v[i + 2]), w * __uint_as_float(v[i + 3]));
          }
        }
      } else if constexpr (KIND == TC_BWD_DH) {
        const int r = t.m0 + row;
        const bool valid = r < t.seg1;
        const float w = valid ? P.topw[P.row_slot[r]] : 0.f;
        float rowsum = 0.f;
#pragma unroll 1
        for (int c = 0; c < TBN; c += 32) {
          if (t.n0 + c >= P.h) break;
          ptx::tmem_ld32(tb + c, v);
          ptx::tmem_wait_ld();
          if (valid) {
            const int64_t o = (int64_t)r * P.h + t.n0 + c;
            float a[32], b[32];
            load_bf16x32(P.a_save + o, a);
            load_bf16x32(P.b_save + o, b);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float dH = __uint_as_float(v[i]);
              const float s = sigmoidf_(a[i]);
              const float S = a[i] * s;
              const float U = S * b[i];
              rowsum = fmaf(dH, U, rowsum);
              const float dU = w * dH;
              const float dA = dU * b[i] * s * (1.f + a[i] * (1.f - s));
              const float dB = dU * S;
              a[i] = dA;
              b[i] = dB;
              v[i] = __float_as_uint(w * U);
            }
            store_bf16x32(P.a_save + o, a);
            store_bf16x32(P.b_save + o, b);
            store_bf16x32(P.u + o, reinterpret_cast<float*>(v));
          }
        }
        if (valid) P.dg_part[(int64_t)r * P.dg_parts + t.n_tile] = rowsum;
      } else {  // DW3 / DW12: store the weight-gradient tile
        const int m = t.m0 + row;
        __nv_bfloat16* dst;
        int N;
        if constexpr (KIND == TC_DW3) {
          N = P.h;
          dst = P.out0 + (int64_t)t.e * P.d * P.h + (int64_t)m * P.h;
        } else {
          N = P.d;
          dst = (m < P.h) ? P.out0 + (int64_t)t.e * P.h * P.d + (int64_t)m * P.d
                          : P.out1 + (int64_t)t.e * P.h * P.d + (int64_t)(m - P.h) * P.d;
        }
#pragma unroll 1
        for (int c = 0; c < TBN; c += 32) {
          if (t.n0 + c >= N) break;
          float f[32];
          if (t.nk > 0) {
            ptx::tmem_ld32(tb + c, v);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) f[i] = 0.f;
          }
          store_bf16x32(dst + t.n0 + c, f);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[as]);
      if (++as == 2) { as = 0; aphase ^= 1; }
    }
  }
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, 512);
  }
}

// ----------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 2D bf16 row-major [rows, cols] map with a (box_cols x box_rows) box, 128B swizzle.
static bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                     uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Row-gather engine: cp.async producer warps (default) or TMA tile::gather4
// (MOEBLAZE_GATHER=tma; kept for the measured comparison in DESIGN.md).
static bool use_cpasync() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOEBLAZE_GATHER");
    v = (e && e[0] == 't') ? 0 : 1;
  }
  return v == 1;
}

template <int KIND, bool CPA>
static moe_status launch_tc_impl(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0,
                                 const CUtensorMap& b1, const TcParams& P, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(tc_gemm_kernel<KIND, CPA>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM) !=
        cudaSuccess)
      return MOE_ERR_CUDA;
    attr = true;
  }
  MOE_LAUNCH((tc_gemm_kernel<KIND, CPA>), grid, TC_THREADS, TC_SMEM, st, a0, a1, b0, b1, P);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

template <int KIND>
static moe_status launch_tc(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0,
                            const CUtensorMap& b1, const TcParams& P, int64_t tiles_upper, cudaStream_t st) {
  if (tiles_upper <= 0) return MOE_OK;
  const int grid = (int)std::min<int64_t>(tiles_upper, num_sms());
  if (use_cpasync()) return launch_tc_impl<KIND, true>(a0, a1, b0, b1, P, grid, st);
  return launch_tc_impl<KIND, false>(a0, a1, b0, b1, P, grid, st);
}

int tc_dg_parts(int h) { return (int)ceil_div(h, TBN); }

// K1 on tensor cores (bf16): logits = X Wg^T with M = 128 tokens, N = E padded
// to a multiple of 16 (rows past E are TMA zero-fill), K = d.
moe_status tc_route(const moe_problem* p, const void* x, const void* wg, float* logits, int32_t* ids, float* topw,
                    cudaStream_t st) {
  if (p->T == 0) return MOE_OK;
  TcParams P{};
  P.T = (int)p->T; P.d = p->d; P.h = p->h; P.E = p->E;
  P.logits = logits; P.ids = ids; P.route_w = topw; P.k = p->k; P.renorm = p->renormalize;
  P.route_n = std::max(16, (int)ceil_div(p->E, 16) * 16);
  P.route_idesc = ptx::umma_idesc_bf16(TBM, P.route_n, 0, 0);
  CUtensorMap a0, b0;
  if (!make_map(&a0, x, p->T, p->d, 64, 128) || !make_map(&b0, wg, p->E, p->d, 64, P.route_n)) return MOE_ERR_CUDA;
  const int64_t tiles = ceil_div(p->T, TBM);
  const int grid = (int)std::min<int64_t>(tiles, num_sms());
  return launch_tc_impl<TC_ROUTE, false>(a0, a0, b0, b0, P, grid, st);
}

moe_status tc_gemm(const GemmCall& c, cudaStream_t st) {
  typedef __nv_bfloat16 bf;
  const int64_t T = c.T, R = c.R;
  const int d = c.d, h = c.h, E = c.E;
  TcParams P{};
  P.x = (const bf*)c.x; P.dy = (const bf*)c.dy;
  P.offs = c.offs; P.eti = c.eti; P.row_slot = c.row_slot; P.topw = c.topw;
  P.a_save = (bf*)c.a_save; P.b_save = (bf*)c.b_save; P.u = (bf*)c.u;
  P.acc_out = c.acc_out; P.dg_part = c.dg_part;
  P.out0 = (bf*)c.dw_a; P.out1 = (bf*)c.dw_b;
  P.T = (int)T; P.d = d; P.h = h; P.E = E;
  P.dg_parts = tc_dg_parts(h);
  CUtensorMap a0, a1, b0, b1;
  bool ok = true;
  const int64_t mt_upper = ceil_div(R, TBM) + E;
  switch (c.which) {
    case GEMM_FWD_UP: {
      if (R == 0) return MOE_OK;
      ok &= make_map(&a0, c.x, T, d, 64, 1);
      ok &= make_map(&b0, c.w1, (uint64_t)E * h, d, 64, 128);
      ok &= make_map(&b1, c.w2, (uint64_t)E * h, d, 64, 128);
      if (!ok) return MOE_ERR_CUDA;
      P.n_tiles = h / 128;
      return launch_tc<TC_FWD_UP>(a0, a0, b0, b1, P, mt_upper * P.n_tiles, st);
    }
    case GEMM_FWD_DOWN: {
      if (R == 0) return MOE_OK;
      ok &= make_map(&a0, c.u, R, h, 64, 128);
      ok &= make_map(&b0, c.w3, (uint64_t)E * d, h, 64, 256);
      if (!ok) return MOE_ERR_CUDA;
      P.n_tiles = (int)ceil_div(d, TBN);
      return launch_tc<TC_FWD_DOWN>(a0, a0, b0, b0, P, mt_upper * P.n_tiles, st);
    }
    case GEMM_BWD_DH: {
      if (R == 0) return MOE_OK;
      ok &= make_map(&a0, c.dy, T, d, 64, 1);
      ok &= make_map(&b0, c.w3, (uint64_t)E * d, h, 64, 64);
      if (!ok) return MOE_ERR_CUDA;
      P.n_tiles = (int)ceil_div(h, TBN);
      return launch_tc<TC_BWD_DH>(a0, a0, b0, b0, P, mt_upper * P.n_tiles, st);
    }
    case GEMM_BWD_DX: {
      if (R == 0) return MOE_OK;
      ok &= make_map(&a0, c.a_save, R, h, 64, 128);
      ok &= make_map(&a1, c.b_save, R, h, 64, 128);
      ok &= make_map(&b0, c.w1, (uint64_t)E * h, d, 64, 64);
      ok &= make_map(&b1, c.w2, (uint64_t)E * h, d, 64, 64);
      if (!ok) return MOE_ERR_CUDA;
      P.n_tiles = (int)ceil_div(d, TBN);
      return launch_tc<TC_BWD_DX>(a0, a1, b0, b1, P, mt_upper * P.n_tiles, st);
    }
    case GEMM_DW3: {
      if (R == 0) {  // no rows at all: every expert's gradient is exactly zero
        MOE_CUDA_CHECK(cudaMemsetAsync(c.dw_a, 0, (size_t)E * d * h * 2, st));
        return MOE_OK;
      }
      ok &= make_map(&a0, c.dy, T, d, 64, 1);
      ok &= make_map(&b0, c.u, R, h, 64, 64);
      if (!ok) return MOE_ERR_CUDA;
      P.m_tiles = d / TBM;
      P.n_tiles = (int)ceil_div(h, TBN);
      return launch_tc<TC_DW3>(a0, a0, b0, b0, P, (int64_t)E * P.m_tiles * P.n_tiles, st);
    }
    case GEMM_DW12: {
      if (R == 0) {
        MOE_CUDA_CHECK(cudaMemsetAsync(c.dw_a, 0, (size_t)E * d * h * 2, st));
        MOE_CUDA_CHECK(cudaMemsetAsync(c.dw_b, 0, (size_t)E * d * h * 2, st));
        return MOE_OK;
      }
      ok &= make_map(&a0, c.a_save, R, h, 64, 64);
      ok &= make_map(&a1, c.b_save, R, h, 64, 64);
      ok &= make_map(&b0, c.x, T, d, 64, 1);
      if (!ok) return MOE_ERR_CUDA;
      P.m_tiles = 2 * h / TBM;
      P.n_tiles = (int)ceil_div(d, TBN);
      return launch_tc<TC_DW12>(a0, a1, b0, b0, P, (int64_t)E * P.m_tiles * P.n_tiles, st);
    }
  }
  return MOE_ERR_INVALID_ARG;
}

}  // namespace moeb
