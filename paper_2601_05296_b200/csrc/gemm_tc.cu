// gemm_tc.cu — the expert GEMMs (and the router) of the MoE layer on sm_100a
// tensor cores.
//
// One persistent, warp-specialised kernel template (tcgen05.mma kind::f16,
// bf16 operands, fp32 accumulators in TMEM):
//   warp 0      TMA producer: tile loads of the non-gathered operand
//   warp 1      MMA issuer (one thread): 4 x tcgen05.mma (K16) per 64-wide K
//               block; tcgen05.commit frees the smem stage / publishes the
//               accumulator
//   warp 2      TMEM allocator (512 columns = 2 accumulator stages x 256); in
//               the leader CTA of a pair, lane 0 then runs the die-aware dynamic
//               tile scheduler of the expert GEMMs (tiles published through a ring
//               in both CTAs' shared memory; topology.cu measures the SM -> die map)
//   warp 3      (CTA pair) relays cp.async-gather completion to the leader
//   warps 4-7   epilogue: tcgen05.ld, one accumulator row per thread
//   warps 8-11  row gathers: 16-byte cp.async straight from the unpermuted X /
//               dY through expert_token_indices into the 128B-swizzled UMMA
//               layout — no routed-token buffer exists
//   warps 12-15 (BWD_DH, TC_BWD_DH_LK) a second epilogue warp per TMEM lane
//               quarter: warps 4-7 take columns 0-127 of the tile, 12-15 columns
//               128-255
//
// CG = 2 (default for the expert GEMMs): a CTA pair (cluster of 2) computes a
// 256 x 256 tile with tcgen05.mma.cta_group::2 — each CTA stages 128 rows of A
// and 128 columns of B (32 KB per stage, 6 stages), holds its 128 rows of the
// accumulator in its own TMEM; the leader CTA issues the MMAs and commits
// multicast to both CTAs' barriers.  CG = 1: one CTA, 128 x 256 tile, 4 stages
// of 48 KB (used by the router and kept for the measured comparison).
//
// Kinds ("rows" = routed rows of one expert segment, from device offsets):
//   FWD_UP   M=rows N=2x128 K=d  A=gather X (K-major)     B=[W1;W2] stacked   epi: A,B saved, U=SiLU(A)B   Alg.1 l.9
//   FWD_DOWN M=rows N=256   K=h  A=U rows (K-major)       B=W3 (K-major)      epi: red.add w*O -> Yacc      Alg.1 l.10
//   BWD_DH   M=rows N=256   K=d  A=gather dY (K-major)    B=W3 (MN-major)     epi: SwiGLU bwd, dA/dB in place,
//                                                                               wU, gate-grad partials   Alg.1 l.20-28
//   BWD_DX   M=rows N=256   K=2h A=dA|dB rows (K-major)   B=W1|W2 (MN-major)  epi: red.add -> dXacc        Alg.1 l.30
//   DW3      M=d    N=256   K=rows A=gather dY (MN-major) B=wU rows (MN)      epi: store dW3_e             Alg.1 l.18
//   DW12     M=2h   N=256   K=rows A=dA|dB rows (MN)      B=gather X (MN)     epi: store dW1_e, dW2_e      Alg.1 l.29
//   ROUTE    M=128 tokens N=E(16-padded) K=d: logits, softmax, top-k epilogue
// Rows past a segment end are zero-filled in shared memory (cp.async src-size
// 0, or TMA out-of-bounds fill), which zero-pads the K tail of the weight-
// gradient GEMMs on chip only (no padded buffer exists in HBM).
#include <cudaTypedefs.h>

#include <climits>
#include <cstdlib>

#include "gemm.h"
#include "ptx.cuh"

namespace moeb {

enum TcKind { TC_FWD_UP = 0, TC_FWD_DOWN = 1, TC_BWD_DH = 2, TC_BWD_DX = 3, TC_DW3 = 4, TC_DW12 = 5, TC_ROUTE = 6,
              TC_BWD_DH_LK = 7, TC_ROUTE_S = 8, TC_BWD_DH_L5 = 9 };
// K1 in two smem layouts: TC_ROUTE (any E <= 256: 32 KB of W_g rows per stage, 4 stages) and
// TC_ROUTE_S (E <= 64: 8 KB per stage, 8 stages).  With T / 128 CTAs (fewer than the SMs at
// the benchmark shapes) each CTA streams its tokens' X rows, so the bytes in flight per SM
// set the pace
__host__ __device__ constexpr bool is_route(int k) { return k == TC_ROUTE || k == TC_ROUTE_S; }
// BWD_DH comes in two forms: TC_BWD_DH (4 epilogue warps, 32-column chunks, 4 stages; the
// 1-CTA engines and the cp.async epilogue) and TC_BWD_DH_LK (16-column chunks: 128
// registers, so 8 epilogue warps fit; 4 stages) -- the CTA-pair default for every d >=
// MOEB_DH_LK_MIN_D.  Its SwiGLU-backward epilogue (10 bytes per output element) was the
// bottleneck under short mainloops (K = d = 2048)
// TC_BWD_DH_L5: the same 16-column TMA epilogue on 4 warps, which leaves the shared memory for
// a 5-stage mainloop -- the better trade for long K (d >= MOEB_DH_L5_MIN_D: Mixtral-like
// BWD_DH 1.80 -> 1.70 ms), while short K (DeepSeek-like, d = 2048) needs the 8 warps to hide
// the SwiGLU-backward epilogue (0.69 vs 0.86 ms; profiles/r02c_variants.txt)
__host__ __device__ constexpr bool is_dh(int k) { return k == TC_BWD_DH || k == TC_BWD_DH_LK || k == TC_BWD_DH_L5; }
// the forward kinds that can run on one side of a per-expert row split (moe_fwd_sync)
__host__ __device__ constexpr bool splits_rows(int k) { return k == TC_FWD_UP || k == TC_FWD_DOWN; }

#ifndef MOEB_DH_STAGES
#define MOEB_DH_STAGES 5  // BWD_DH mainloop stages in the CTA-pair engine (smem shared with the epilogue ring)
#endif
#ifndef MOEB_DH_TMA
#define MOEB_DH_TMA 1     // BWD_DH epilogue I/O by TMA boxes (1) or per-lane cp.async / stores (0)
#endif
#ifndef MOEB_DH_NBUF
#define MOEB_DH_NBUF 6    // BWD_DH epilogue ring depth (A/B chunks of DH_CW columns per warp)
#endif
#ifndef MOEB_DIE_EXPERT
// die-aware schedule of the row kinds: 0 = split every expert's n-tiles between the dies
// (weights die-local, rows read by both dies); 1 = split the experts (each expert's rows and
// weights read by one die; experiment)
#define MOEB_DIE_EXPERT 0
#endif
#ifndef MOEB_WIDE_ROW
// 256 x 512 CTA-pair tiles for FWD_DOWN (bit 0) / BWD_DX (bit 1): 25 % fewer operand
// bytes per flop, single-buffered accumulator (experiment; profiles/SUMMARY_r02.md)
#define MOEB_WIDE_ROW 0
#endif
#ifndef MOEB_WIDE_WG
// weight-gradient kinds (DW3, DW12) on 256 x 512 CTA-pair tiles: two N = 256 accumulators fill
// the 512 TMEM columns (no double buffer: the short bf16-store epilogue is exposed), for 25 %
// fewer operand bytes per flop
#define MOEB_WIDE_WG 0
#endif
#ifndef MOEB_SMEM_TIGHT
#define MOEB_SMEM_TIGHT 1  // 768-byte barrier block and no alignment slack (lets 8-warp BWD_DH run 5 stages)
#endif
#ifndef MOEB_TEMPTY_RELAXED
#define MOEB_TEMPTY_RELAXED 1  // epilogue -> MMA "accumulator free" arrive without a cluster release fence
#endif
#ifndef MOEB_DH_L2PF
// BWD_DH epilogue: prefetch the next tile's A, B rows into L2.  Off: measured slower on both
// shapes (DeepSeek-like 0.69 -> 0.74 ms, Mixtral-like 1.80 -> 1.88 ms; profiles/r02c_variants.txt)
#define MOEB_DH_L2PF 0
#endif
#ifndef MOEB_DH_EPI8
#define MOEB_DH_EPI8 1    // TC_BWD_DH_LK: 8 epilogue warps (two per TMEM lane quarter, 128 columns each)
#endif
#ifndef MOEB_UP_EPI8
// FWD_UP: 8 epilogue warps (16-column chunks; 64 of the 128 A/B columns each).  Parity-green,
// off: interleaved A/B measured FWD_UP 3-7 % slower (profiles/up8_ab_r01.txt) -- its epilogue
// already hides under the mainloop, and 32-byte row segments store less efficiently
#define MOEB_UP_EPI8 0
#endif
#ifndef MOEB_BULK_RED
// FWD_DOWN / BWD_DX red.add combine (OUT_RED) by bulk reductions from shared memory (one
// cp.reduce.async.bulk of a row's 32 columns per row, issued by one lane) instead of per-lane
// red.global.add.v4
#define MOEB_BULK_RED 0
#endif
#ifndef MOEB_RED_EVICT_LAST
// FWD_DOWN / BWD_DX red.add combine with an L2 evict_last hint: a token's accumulator row is
// hit k times at scattered moments of the launch; kept resident, its read-modify-writes
// need no DRAM read
#define MOEB_RED_EVICT_LAST 0
#endif
#ifndef MOEB_RG
#define MOEB_RG 8  // row kinds: m-tiles per rasterisation group (the group's rows stay L2-resident)
#endif
#ifndef MOEB_WG_LPT
// DW3 / DW12 tiles claimed longest-K (largest expert) first.  Skewed routing put the largest
// expert's 236-k-block tiles wherever its index fell in the list; claimed late they left a
// tail with most SMs idle: DeepSeek-like skewed DW3 0.82-0.85 -> 0.56 ms, balanced and
// Mixtral-like unchanged (profiles/variants_r02al_wgrad_lpt.txt)
#define MOEB_WG_LPT 1
#endif
#ifndef MOEB_RED_EPI8
// FWD_DOWN / BWD_DX: 8 epilogue warps (128 columns each), 5 mainloop stages.  Parity-green but
// off: interleaved A/B measured both kinds 1-5 % slower (profiles/red8_ab_r01.txt).  (Since the
// row-split segment ends joined the FWD_DOWN offsets block, its one-CTA engine variants exceed
// the 227 KB shared-memory limit with this flag; it is kept as the record of round 1.)
#define MOEB_RED_EPI8 0
#endif
// 8-warp BWD_DH: 5 mainloop stages + a 3-deep epilogue ring (one chunk of A/B prefetch) in the
// tight layout; measured DeepSeek-like BWD_DH 0.681 -> 0.670 ms (mean of 4, interleaved,
// profiles/variants_r02i_dh5.txt) against 4 stages + a 4-deep ring
#ifndef MOEB_DH8_STAGES
#define MOEB_DH8_STAGES 5
#endif
#ifndef MOEB_DH8_NBUF
#define MOEB_DH8_NBUF 3
#endif
#ifndef MOEB_DH_STAGES_SK
#define MOEB_DH_STAGES_SK 4  // the same for the short-K variant (TC_BWD_DH)
#endif
#ifndef MOEB_DH_NBUF_SK
#define MOEB_DH_NBUF_SK 4
#endif
#ifndef MOEB_NTAIL
#define MOEB_NTAIL 1      // bit 0: DW3, bit 1: BWD_DH (CTA pair): a last n-tile with <= 128 valid columns runs N = 128 MMAs
#endif
#ifndef MOEB_MTAIL
// FWD_DOWN / BWD_DX (CTA pair): an m-tile with <= 128 rows runs M = 128 MMAs.  Parity-green,
// but off: interleaved same-box A/B (profiles/mtail_ab_r01.txt) measured the whole Mixtral
// step 2 % slower with it (every kind, not only the two it changes) and DeepSeek neutral
#define MOEB_MTAIL 0
#endif
#ifndef MOEB_DYN_WG
#define MOEB_DYN_WG 1     // the weight-gradient kinds (DW3, DW12) on the dynamic scheduler too
#endif
#ifndef MOEB_DYN
#define MOEB_DYN 1        // row-kind tiles from the die-aware dynamic scheduler (0: static cluster-strided order)
#endif
// timing-only experiments (never in the product build): bit masks over TcKind
#ifndef MOEB_EXP_NOEPI
#define MOEB_EXP_NOEPI 0  // kinds whose epilogue is skipped (measures the mainloop alone)
#endif
#ifndef MOEB_EXP_SAMEB
#define MOEB_EXP_SAMEB 0  // kinds whose B tiles all come from one L2-resident panel (operand-stream experiment)
#endif
#ifndef MOEB_EXP_NOB
#define MOEB_EXP_NOB 0    // kinds whose B tiles are not loaded at all (the MMAs reuse stale smem; operand-stream experiment)
#endif
#ifndef MOEB_EXP_NOMMA
#define MOEB_EXP_NOMMA 0  // kinds whose MMAs are skipped (measures loads + epilogue)
#endif
// epilogue warps: 4 (warps 4-7), or 8 for TC_BWD_DH_LK (warps 4-7 and 12-15: two warps per
// TMEM lane quarter, each with 128 of the tile's 256 columns; its 16-column chunks keep the
// kernel at 128 registers, so 16 warps fit the register file)
__host__ __device__ constexpr int n_epi(int k) {
  return ((k == TC_BWD_DH_LK && MOEB_DH_EPI8 && MOEB_DH_TMA) || ((k == TC_FWD_DOWN || k == TC_BWD_DX) && MOEB_RED_EPI8) ||
          (k == TC_FWD_UP && MOEB_UP_EPI8))
             ? 8 : 4;
}
__host__ __device__ constexpr int tc_threads(int k) { return 32 * (8 + n_epi(k)); }
constexpr int TBN = 256, TBK = 64;         // MMA N per tile, K block
// 256 x 512 pair tiles for the weight-gradient kinds (MOEB_WIDE_WG)
// and (MOEB_WIDE_ROW bits 0 / 1) for the long-K red.add kinds FWD_DOWN / BWD_DX
template <int KIND, int CG>
__host__ __device__ constexpr bool wide_tile() {
  return CG == 2 && ((MOEB_WIDE_WG && (KIND == TC_DW3 || KIND == TC_DW12)) ||
                     ((MOEB_WIDE_ROW & 1) && KIND == TC_FWD_DOWN) || ((MOEB_WIDE_ROW & 2) && KIND == TC_BWD_DX));
}
template <int KIND, int CG>
__host__ __device__ constexpr int tile_n() { return wide_tile<KIND, CG>() ? 2 * TBN : TBN; }
constexpr int TA_BYTES = 128 * TBK * 2;    // 16 KB: 128 rows of A per CTA
constexpr int TC_THREADS = 384;            // 12 warps (16 with the 8-warp BWD_DH epilogue)
constexpr int GATHER_THREADS = 128;

template <int CG, int KIND = 0>
struct CgCfg {
  static constexpr int TM = 128 * CG;                   // tile rows per CTA group
  static constexpr int B_BYTES = (KIND == TC_ROUTE_S ? 64 : tile_n<KIND, CG>() / CG) * TBK * 2;  // B per CTA per stage
  static constexpr int STAGE = TA_BYTES + B_BYTES;
  // BWD_DH shares smem between its mainloop ring and the epilogue A/B ring (tools/tune_variants.sh:
  // 4 stages + 4-deep ring beat 3 + 7 by 11 % on the Mixtral layer)
  static constexpr bool DH = is_dh(KIND);
  static constexpr bool LK = (KIND == TC_BWD_DH_LK || KIND == TC_BWD_DH_L5) && MOEB_DH_TMA;
  static constexpr int NEPI = n_epi(KIND);
  static constexpr int STAGES = DH ? (CG == 1 ? 2 : (LK ? (NEPI == 8 ? MOEB_DH8_STAGES : MOEB_DH_STAGES) : MOEB_DH_STAGES_SK))
                                   : (KIND == TC_ROUTE_S ? 8 : CG == 1 ? 4 : (wide_tile<KIND, CG>() ? 4 : (NEPI == 8 ? 5 : 6)));
  static constexpr int DH_NBUF = LK ? (NEPI == 8 ? MOEB_DH8_NBUF : MOEB_DH_NBUF) : MOEB_DH_NBUF_SK;  // BWD_DH: A/B ring per warp
  // BWD_DH epilogue chunk: 16 columns (TMA boxes of 32 rows x 32 B, 32-byte swizzle) in the
  // TMA epilogue, 32 in the cp.async one; a slot holds the A and the B chunk
  static constexpr int DH_CW = LK ? 16 : 32;
  static constexpr int DH_SLOT = 2 * 32 * DH_CW * 2;
  // epilogue staging bytes per warp (BWD_DH: the A/B ring + two wU tiles)
  static constexpr int STG_WARP = DH ? (DH_NBUF * DH_SLOT + DH_SLOT) : ((KIND == TC_FWD_UP && NEPI == 8) ? 3072 : 6144);
  // 1024-aligned: the BWD_DH tiles are TMA boxes in the 64-byte swizzle, whose pattern is
  // taken from the smem address bits
  // after the stages: barriers (768 B: stage/accumulator/scheduler barriers at +0 / +256, the
  // BWD_DH epilogue ring's at +512) and the per-expert offsets + tile starts (2 x 260 ints)
  static constexpr int OFFS_OFF = MOEB_SMEM_TIGHT ? 768 : 1024;
  // s_offs + s_mstart (2 x 260 ints); FWD_UP / FWD_DOWN also keep each segment's end (s_offs +
  // 520: the row-split launches process [offs[e], split[e]) or [split[e], offs[e+1]))
  static constexpr int OFFS_BYTES = (MOEB_SMEM_TIGHT ? 2080 : 2176) + (splits_rows(KIND) ? 1040 : 0);
  static constexpr int STG_OFF = (STAGES * STAGE + OFFS_OFF + OFFS_BYTES + 1023) / 1024 * 1024;
  // the dynamic shared memory starts 1024-aligned (after the 1 KB the driver reserves per CTA;
  // profiles/smem_probe_r02e.txt), so the tight layout carries no alignment slack (the kernel
  // traps if that ever changes)
  static constexpr int SMEM = STG_OFF + NEPI * STG_WARP + (MOEB_SMEM_TIGHT ? 0 : 1024);
};

struct TcParams {
  const __nv_bfloat16* x;   // gathered operand sources
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
  int n_tiles, m_tiles, m_tiles2;  // m_tiles at tile height 128 / 256 (weight-gradient kinds)
  int dg_parts;
  // TC_ROUTE (K1): logits = X Wg^T on tensor cores, softmax + top-k in the epilogue
  float* logits;
  int32_t* ids;
  float* route_w;
  int k, renorm, route_n;
  uint32_t route_idesc;
  int act;  // MOE_ACT_*: 0 SwiGLU (gated: stacked [W1;W2], A and B); 1 SiLU / 2 ReLU (non-gated)
  int out_mode;                  // FWD_DOWN / BWD_DX target (gemm.h OutMode)
  __nv_bfloat16* out_tok;        // OUT_TOKN destination [T, d]
  // die-aware dynamic tile scheduler (row kinds, CTA pair): every expert's n-tiles
  // [0, n_split) form die 0's tile list, [n_split, n_tiles) die 1's; sched[0..1]
  // are the lists' claim counters (zeroed before the launch), die_map[smid] the
  // SM's die (topology.cu)
  int* sched;
  const uint8_t* die_map;
  int n_split;
  int die_expert;  // MOEB_DIE_EXPERT: the dies split the experts (all n-tiles each), n_split = n_tiles;
                   // die_sm0_permille = die 0's share of the SMs
  int die_sm0_permille;
  int u_weighted;  // MOE_CKPT_ABU: FWD_UP stores w * U; FWD_DOWN then adds U W3 with unit weight
  int dh_skip_u;   // MOE_CKPT_ABU: BWD_DH writes dA, dB only (wU is saved from the forward)
  // FWD_UP / FWD_DOWN row split (moe_fwd_sync): split_half 1 = rows [offs[e], row_split[e])
  // of every expert, 2 = rows [row_split[e], offs[e+1]); 0 = all rows
  const int32_t* row_split;
  int split_half;
  int sm_reserve;  // host only: SMs the launch leaves free (moe_fwd_sync.sm_reserve)
};

template <int KIND>
struct KindTraits;
// row kinds in the CTA-pair engine take their tiles from the dynamic scheduler
template <int KIND, int CG>
__host__ __device__ constexpr bool dyn_sched() {
  return MOEB_DYN && CG == 2 && !is_route(KIND) && (MOEB_DYN_WG || (KIND != TC_DW3 && KIND != TC_DW12));
}
constexpr int SCHED_RING = 4;  // tiles published ahead by the scheduler
// N = 128 tail tiles (N = h, B = MN-major panels of 64 columns, CTA pair) when at most
// 128 of the tile's 256 output columns exist (h % 256 == 128).  Enabled for DW3; BWD_DH
// supports it but measured slower (its half-length tail mainloop turns gather-bound
// under a full-size epilogue; DeepSeek-like BWD_DH 0.79-0.81 -> 0.83-0.84 ms)
// M = 128 tail tiles: FWD_DOWN and BWD_DX (plain epilogues; A by TMA) in the CTA pair,
// when a segment's last m-tile has <= 128 rows.  With cta_group::2 and M = 128 each CTA
// holds 64 rows of A and of the accumulator; the accumulator's first 128 columns sit in
// TMEM lanes 0-63, the other 128 in lanes 64-127, both at columns 0-127 (the 2-SM
// M_MMA = 64 layout of CUTLASS's tmem_frg_2sm), so epilogue warp wq handles rows
// 32 (wq & 1) + lane and output columns 128 (wq >> 1) + [0, 128).
template <int KIND, int CG>
__host__ __device__ constexpr bool has_mtail() {
  return MOEB_MTAIL && CG == 2 && (KIND == TC_FWD_DOWN || KIND == TC_BWD_DX) && n_epi(KIND) == 4;
}
template <int KIND, int CG>
__host__ __device__ constexpr bool has_ntail() {
  return CG == 2 && ((MOEB_NTAIL & 1) && KIND == TC_DW3 && !wide_tile<KIND, CG>() || (MOEB_NTAIL & 2) && is_dh(KIND));
}

template <int KIND>
struct KindTraits {
  static constexpr bool wgrad = (KIND == TC_DW3 || KIND == TC_DW12);
  static constexpr bool a_mn = wgrad;  // A operand MN-major?
  static constexpr bool b_mn = (is_dh(KIND) || KIND == TC_BWD_DX || wgrad);
  static constexpr int NT = (KIND == TC_FWD_UP) ? 128 : 256;  // output columns per tile
  static constexpr bool gather_a = (KIND == TC_FWD_UP || is_dh(KIND) || KIND == TC_DW3);
  static constexpr bool gather_b = (KIND == TC_DW12);
  static constexpr bool gathered = gather_a || gather_b;
};

// bytes per CTA per stage delivered by TMA (the rest comes from cp.async gathers)
template <int KIND, bool CPA, int CG>
__host__ __device__ constexpr uint32_t tma_bytes_per_cta() {
  return ((CPA && KindTraits<KIND>::gather_a) ? 0u : (uint32_t)TA_BYTES) +
         ((CPA && KindTraits<KIND>::gather_b) ? 0u : (uint32_t)CgCfg<CG, KIND>::B_BYTES);
}

struct TileInfo {
  int e, m0, n0, n_tile, seg0, seg1, nk;
};

template <int KIND, int CG>
__device__ __forceinline__ bool decode_tile(int tile, const TcParams& P, const int* s_offs, const int* s_mstart,
                                            TileInfo& t) {
  using K = KindTraits<KIND>;
  constexpr int TM = CgCfg<CG>::TM;
  if (tile < 0) return false;
  if constexpr (is_route(KIND)) {
    if (tile * TM >= P.T) return false;
    t.e = 0;
    t.seg0 = 0;
    t.seg1 = P.T;
    t.m0 = tile * TM;
    t.n0 = 0;
    t.n_tile = 0;
    t.nk = P.d / TBK;
  } else if constexpr (K::wgrad) {
    // tile lists as for the row kinds: die 0 = every expert's n-tiles [0, ns), die 1 the rest
    const int ns = dyn_sched<KIND, CG>() ? P.n_split : P.n_tiles;
    int nt = ns, nlo = 0, local = tile;
    if (tile >= P.E * P.m_tiles * ns) {
      nt = P.n_tiles - ns;
      nlo = ns;
      local = tile - P.E * P.m_tiles * ns;
      if (local >= P.E * P.m_tiles * nt) return false;
    }
    const int per_e = P.m_tiles * nt;
    // experts in the order of s_mstart (longest K first, MOEB_WG_LPT) or by index
    const int pos = local / per_e;
    t.e = MOEB_WG_LPT ? s_mstart[pos] : pos;
    const int rem = local - pos * per_e;
    int mt;
    if constexpr (KIND == TC_DW3) {
      // m fastest: the concurrent tiles share the B n-tile (wU rows, h wide: the
      // larger operand) and re-read the small gathered dY from L2
      t.n_tile = nlo + rem / P.m_tiles;
      mt = rem - (rem / P.m_tiles) * P.m_tiles;
    } else {
      // n fastest: DW12's A ([dA|dB], 2h wide) is the larger operand
      mt = rem / nt;
      t.n_tile = nlo + (rem - mt * nt);
    }
    t.m0 = mt * TM;
    t.n0 = t.n_tile * tile_n<KIND, CG>();
    t.seg0 = s_offs[t.e];
    t.seg1 = s_offs[t.e + 1];
    t.nk = (t.seg1 - t.seg0 + TBK - 1) / TBK;
  } else {
    // tile lists: die 0 = every expert's n-tiles [0, ns), die 1 = [ns, n_tiles)
    // (one list, ns = n_tiles, in the static schedule); s_mstart = prefix sum
    // of the experts' m-tile counts
    const int ns = dyn_sched<KIND, CG>() ? P.n_split : P.n_tiles;
    const int Mt = s_mstart[P.E];
    int nt, nlo, local = tile;
    if (tile < Mt * ns) {
      nt = ns;
      nlo = 0;
    } else {
      nt = P.n_tiles - ns;
      nlo = ns;
      local = tile - Mt * ns;
      if (local >= Mt * nt) return false;
    }
    t.e = find_segment(s_mstart, P.E, local / nt);
    t.seg0 = s_offs[t.e];
    t.seg1 = splits_rows(KIND) ? s_offs[520 + t.e] : s_offs[t.e + 1];  // segment ends (row split)
    const int mt_e = s_mstart[t.e + 1] - s_mstart[t.e];
    local -= s_mstart[t.e] * nt;
    // grouped rasterisation: blocks of ~RG m-tiles x the list's n-tiles, m
    // fastest, so a block's rows stay L2-resident while the weight tiles stream
    // once per block.  The segment's m-tiles are split into ng = max(1, mt_e / RG)
    // groups of near-equal size (sizes differ by at most one, the larger first):
    // a remainder never forms a small group of its own, which would re-stream the
    // expert's whole weight for a handful of rows (9 m-tiles = one group of 9,
    // not 8 + 1)
    constexpr int RG = MOEB_RG;
    const int ng = max(1, mt_e / RG);
    const int gsz = mt_e / ng, extra = mt_e - gsz * ng;  // `extra` groups have gsz + 1 m-tiles
    const int big = extra * (gsz + 1) * nt;
    int sz, mstart, within;
    if (local < big) {
      sz = gsz + 1;
      const int g = local / (sz * nt);
      within = local - g * sz * nt;
      mstart = g * sz;
    } else {
      sz = gsz;
      const int l2 = local - big;
      const int g = l2 / (sz * nt);
      within = l2 - g * sz * nt;
      mstart = extra * (gsz + 1) + g * sz;
    }
    t.n_tile = nlo + within / sz;
    const int mi = mstart + (within - (within / sz) * sz);
    t.m0 = t.seg0 + mi * TM;
    t.n0 = t.n_tile * ((KIND == TC_FWD_UP && P.act == 0) ? 128 : tile_n<KIND, CG>());
    const int Kdim = (KIND == TC_FWD_UP || is_dh(KIND)) ? P.d
                     : (KIND == TC_FWD_DOWN ? P.h : (P.act == 0 ? 2 : 1) * P.h);
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

// ---------------------------------------------------------------- epilogue staging
// Each epilogue warp owns 32 accumulator rows (one per lane).  Its 32-column
// chunks go through a small swizzled shared tile so that global loads,
// stores and red.adds are issued row-coalesced (8 lanes x 16 B per 128 B line)
// instead of one 16-byte access per lane on 32 different lines.
// bf16 tile: 32 rows x 64 B, 16-byte chunk q of row i at i*64 + ((q ^ ((i>>1)&3)) << 4)
// fp32 tile: 32 rows x 128 B, chunk q (0..7) of row i at i*128 + ((q ^ (i&7)) << 4)
__device__ __forceinline__ uint32_t stg16_off(int i, int q) { return i * 64 + ((q ^ ((i >> 1) & 3)) << 4); }
// bf16 tile of 32 rows x 16 columns (32 B), the TMA 32-byte swizzle: chunk q (0..1) of row
// i at i*32 + ((q ^ ((i>>2)&1)) << 4) (conflict-free for one row per lane)
__device__ __forceinline__ uint32_t stg8_off(int i, int q) { return i * 32 + ((q ^ ((i >> 2) & 1)) << 4); }
template <int CW>
__device__ __forceinline__ uint32_t stgw_off(int i, int q) { return CW == 16 ? stg8_off(i, q) : stg16_off(i, q); }
template <int CW>
__device__ __forceinline__ void tmem_ldw(uint32_t taddr, uint32_t (&v)[CW]) {
  if constexpr (CW == 16) ptx::tmem_ld16(taddr, v);
  else ptx::tmem_ld32(taddr, v);
}
__device__ __forceinline__ void stg8_store_bf16(const uint8_t* stg, int lane, __nv_bfloat16* base, int64_t ld,
                                                int nvalid) {
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int row = it * 16 + (lane >> 1), q = lane & 1;
    if (row < nvalid)
      *reinterpret_cast<uint4*>(base + row * ld + q * 8) = *reinterpret_cast<const uint4*>(stg + stg8_off(row, q));
  }
}
__device__ __forceinline__ uint32_t stg32_off(int i, int q) { return i * 128 + ((q ^ (i & 7)) << 4); }

__device__ __forceinline__ void stg_put_bf16(uint8_t* stg, int i, const float* v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = ptx::pack_bf16(v[8 * q + 0], v[8 * q + 1]);
    u.y = ptx::pack_bf16(v[8 * q + 2], v[8 * q + 3]);
    u.z = ptx::pack_bf16(v[8 * q + 4], v[8 * q + 5]);
    u.w = ptx::pack_bf16(v[8 * q + 6], v[8 * q + 7]);
    *reinterpret_cast<uint4*>(stg + stg16_off(i, q)) = u;
  }
}
__device__ __forceinline__ void stg_get_bf16(const uint8_t* stg, int i, float* v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 u = *reinterpret_cast<const uint4*>(stg + stg16_off(i, q));
    float2 f;
    f = ptx::unpack_bf16(u.x); v[8 * q + 0] = f.x; v[8 * q + 1] = f.y;
    f = ptx::unpack_bf16(u.y); v[8 * q + 2] = f.x; v[8 * q + 3] = f.y;
    f = ptx::unpack_bf16(u.z); v[8 * q + 4] = f.x; v[8 * q + 5] = f.y;
    f = ptx::unpack_bf16(u.w); v[8 * q + 6] = f.x; v[8 * q + 7] = f.y;
  }
}
// rows [0, nvalid) of the tile <-> global rows base + row * ld (32 bf16 columns each)
__device__ __forceinline__ void stg_store_bf16(const uint8_t* stg, int lane, __nv_bfloat16* base, int64_t ld,
                                               int nvalid) {
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int row = it * 8 + (lane >> 2), q = lane & 3;
    if (row < nvalid)
      *reinterpret_cast<uint4*>(base + row * ld + q * 8) = *reinterpret_cast<const uint4*>(stg + stg16_off(row, q));
  }
}
__device__ __forceinline__ void stg_load_bf16(uint8_t* stg, int lane, const __nv_bfloat16* base, int64_t ld,
                                              int nvalid) {
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int row = it * 8 + (lane >> 2), q = lane & 3;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (row < nvalid) u = *reinterpret_cast<const uint4*>(base + row * ld + q * 8);
    *reinterpret_cast<uint4*>(stg + stg16_off(row, q)) = u;
  }
}

__device__ __forceinline__ void stg_load_bf16_async(uint8_t* stg, int lane, const __nv_bfloat16* base, int64_t ld,
                                                    int nvalid) {
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int row = it * 8 + (lane >> 2), q = lane & 3;
    const bool ok = row < nvalid;
    ptx::cp_async16(ptx::smem_u32(stg + stg16_off(row, q)), ok ? (const void*)(base + row * ld + q * 8) : (const void*)base,
                    ok ? 16u : 0u);
  }
}

template <int KIND, bool CPA, int CG>
__global__ void __launch_bounds__(tc_threads(KIND), 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
               const __grid_constant__ CUtensorMap mB0, const __grid_constant__ CUtensorMap mB1, const TcParams P) {
  using K = KindTraits<KIND>;
  using C = CgCfg<CG, KIND>;
  static_assert(CG == 1 || CPA, "the CTA-pair path uses the cp.async gather engine");
  static_assert(C::SMEM <= 232448, "dynamic shared memory over the 227 KB opt-in limit");
  constexpr int STAGES = C::STAGES;
  constexpr bool WIDE = wide_tile<KIND, CG>();
  constexpr int NB = tile_n<KIND, CG>() / CG;  // B columns (rows of the B tile) held by this CTA
  constexpr int NPANEL = NB / 64;  // 64-column MN-major panels of B in this CTA
  constexpr uint32_t IDESC = ptx::umma_idesc_bf16(128 * CG, TBN, K::a_mn ? 1 : 0, K::b_mn ? 1 : 0);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* gfull = empty + STAGES;
  uint64_t* tfull = gfull + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* ebar = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE + 512);  // BWD_DH: [4 warps][DH_NBUF] TMA loads
  // dynamic scheduler: tile ring (published by the leader into both CTAs) and its barriers
  uint64_t* sfull = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE + 256);
  uint64_t* sempty = sfull + SCHED_RING;
  int* s_ring = reinterpret_cast<int*>(sempty + SCHED_RING);
  int* s_offs = reinterpret_cast<int*>(smem + STAGES * C::STAGE + C::OFFS_OFF);
  if constexpr (MOEB_SMEM_TIGHT)
    if (smem != smem_raw) __trap();  // no alignment slack was allocated
  int* s_mstart = s_offs + 260;
  constexpr bool DYN = dyn_sched<KIND, CG>();
  // arrivals that release a ring slot: every tile-iterating warp of both CTAs
  // (TMA producer, epilogue x4, gathers x4 + relay when gathered) + the MMA warp
  constexpr int NCONS = 2 * (1 + C::NEPI + (K::gathered ? 5 : 0)) + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = P.E;
  const uint32_t crank = (CG == 2) ? ptx::cluster_ctarank() : 0u;
  const bool leader = crank == 0;
  const int rowoff = 128 * (int)crank;  // this CTA's rows within the tile (A / accumulator)
  const int coloff = NB * (int)crank;   // this CTA's columns of B within the tile
  const int cluster_id = (CG == 2) ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int n_clusters = (CG == 2) ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if constexpr (splits_rows(KIND)) {
    // segment [s_offs[e], s_offs[520 + e]) of expert e: the whole segment, or one side of
    // row_split[e] (split_half 1: the rows before it, 2: the rows from it on)
    for (int i = threadIdx.x; i < E; i += tc_threads(KIND)) {
      int lo = P.offs[i], hi = P.offs[i + 1];
      if (P.split_half) {
        const int sp = P.row_split[i];
        if (P.split_half == 1) hi = sp;
        else lo = sp;
      }
      s_offs[i] = lo;
      s_offs[520 + i] = hi;
    }
  } else if constexpr (!is_route(KIND)) {
    for (int i = threadIdx.x; i <= E; i += tc_threads(KIND)) s_offs[i] = P.offs[i];
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&mA0);
    ptx::tma_prefetch(&mA1);
    ptx::tma_prefetch(&mB0);
    ptx::tma_prefetch(&mB1);
  }
  if (warp == 1 && lane == 0) {
    const uint32_t full_count =
        CG == 1 ? 1 + ((CPA && K::gathered) ? GATHER_THREADS : 0)
                : 1 + ((CPA && K::gathered) ? 2 : 0);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], full_count);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&gfull[s], GATHER_THREADS);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], C::NEPI * CG);
    }
    if constexpr (is_dh(KIND) && CPA && MOEB_DH_TMA)
      for (int s = 0; s < C::NEPI * C::DH_NBUF; ++s) ptx::mbar_init(&ebar[s], 1);
    if constexpr (DYN)
      for (int s = 0; s < SCHED_RING; ++s) {
        ptx::mbar_init(&sfull[s], 1);
        ptx::mbar_init(&sempty[s], NCONS);
      }
    ptx::fence_mbar_init();
    ptx::fence_proxy_async();
  }
  if (warp == 2) {
    if constexpr (CG == 2) ptx::tmem_alloc_cg2(tmem_holder, 512);
    else ptx::tmem_alloc(tmem_holder, 512);
  }
  __syncthreads();
  if (!K::wgrad && !is_route(KIND) && threadIdx.x == 0) {
    int s = 0;
    for (int e = 0; e < E; ++e) {
      s_mstart[e] = s;
      s += ((splits_rows(KIND) ? s_offs[520 + e] : s_offs[e + 1]) - s_offs[e] + C::TM - 1) / C::TM;
    }
    s_mstart[E] = s;
  }
  if constexpr (K::wgrad && MOEB_WG_LPT) {
    // weight-gradient tiles have K = the expert's rows: hand out the longest ones first (LPT),
    // so a large expert claimed late cannot leave a tail with most SMs idle (skewed routing).
    // Every CTA derives the same order: rank by (rows desc, expert id asc); s_mstart is unused
    // by these kinds and holds it
    for (int e = threadIdx.x; e < E; e += tc_threads(KIND)) {
      const int ne = s_offs[e + 1] - s_offs[e];
      int rank = 0;
      for (int j = 0; j < E; ++j) {
        const int nj = s_offs[j + 1] - s_offs[j];
        rank += (nj > ne) || (nj == ne && j < e);
      }
      s_mstart[rank] = e;
    }
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();  // peer barriers initialised + TMEM allocated
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // shared::cluster addresses of the barriers other CTAs / the leader signal, translated once:
  // mapa is a variable-latency instruction, and inside the per-k-block loops its result was
  // what the producer's TMA issue and the gather relay's arrive waited on (long scoreboard)
  const uint32_t full_c0 = (CG == 2) ? ptx::mapa(ptx::smem_u32(full), 0) : 0u;     // leader's full[]
  const uint32_t sempty_c0 = (CG == 2) ? ptx::mapa(ptx::smem_u32(sempty), 0) : 0u; // leader's sempty[]
  const uint32_t tempty_c0 = (CG == 2) ? ptx::mapa(ptx::smem_u32(tempty), 0) : 0u; // leader's tempty[]

  // i-th tile of this CTA pair: static cluster-strided order, or the dynamic
  // scheduler's ring (every tile-iterating warp reads every slot once, then
  // releases it on the leader; the slot value gates the arrive, so the read has
  // completed before the scheduler may overwrite it)
  // the tile after the current one without consuming it (the ring slot is released by the
  // regular fetch later): lets the BWD_DH epilogue prefetch its next inputs into L2
  auto peek = [&](int it) -> int {
    if constexpr (DYN) {
      const int slot = it % SCHED_RING;
      const uint32_t par = (uint32_t)(it / SCHED_RING) & 1u;
      if (leader) ptx::mbar_wait(&sfull[slot], par);
      else ptx::mbar_wait_cluster(&sfull[slot], par);
      return *reinterpret_cast<volatile int*>(&s_ring[slot]);
    } else {
      return cluster_id + it * n_clusters;
    }
  };
  auto fetch = [&](int it) -> int {
    if constexpr (DYN) {
      const int slot = it % SCHED_RING;
      const uint32_t par = (uint32_t)(it / SCHED_RING) & 1u;
      if (leader) ptx::mbar_wait(&sfull[slot], par);
      else ptx::mbar_wait_cluster(&sfull[slot], par);
      const int tile = *reinterpret_cast<volatile int*>(&s_ring[slot]);
      __syncwarp();
      if (lane == 0 && tile != INT_MIN) {
        if (leader) ptx::mbar_arrive(&sempty[slot]);
        else ptx::mbar_arrive_cluster_relaxed(sempty_c0 + 8u * (uint32_t)slot);
      }
      return tile;
    } else {
      return cluster_id + it * n_clusters;
    }
  };

  if (warp == 0) {
    // ============================ TMA producer ============================
    const int oob = P.T;  // TMA gather4 row past the end: zero-filled (CG = 1, !CPA only)
    int stage = 0;
    uint32_t phase = 0;
    TileInfo t;
    for (int it = 0; decode_tile<KIND, CG>(fetch(it), P, s_offs, s_mstart, t); ++it) {
      int gi0 = 0, gi1 = 0, gi2 = 0, gi3 = 0;
      if constexpr (!CPA && (KIND == TC_FWD_UP || is_dh(KIND))) {
        const int r = t.m0 + 4 * lane;
        gi0 = r + 0 < t.seg1 ? P.eti[r + 0] : oob;
        gi1 = r + 1 < t.seg1 ? P.eti[r + 1] : oob;
        gi2 = r + 2 < t.seg1 ? P.eti[r + 2] : oob;
        gi3 = r + 3 < t.seg1 ? P.eti[r + 3] : oob;
      }
      for (int kb = 0; kb < t.nk; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sA = smem + stage * C::STAGE;
        uint8_t* sB = sA + TA_BYTES;
        uint64_t* bar = &full[stage];
        const uint32_t bar_c = full_c0 + 8u * (uint32_t)stage;  // leader's full[stage] (CTA pair)
        if (lane == 0) {
          if constexpr (is_route(KIND)) {
            ptx::mbar_arrive_expect_tx(bar, (uint32_t)(TA_BYTES + P.route_n * 128));
          } else if constexpr (CG == 1) {
            ptx::mbar_arrive_expect_tx(bar, tma_bytes_per_cta<KIND, CPA, CG>());
          } else {
            uint32_t bytes = 2 * tma_bytes_per_cta<KIND, CPA, CG>();
            if constexpr (has_ntail<KIND, CG>())
              if (P.h - t.n0 <= 128) bytes -= (uint32_t)C::B_BYTES;  // half the B columns per CTA
            if constexpr ((MOEB_EXP_NOB >> KIND) & 1) bytes -= 2 * (uint32_t)C::B_BYTES;
            if (leader) ptx::mbar_arrive_expect_tx(bar, bytes);
          }
        }
        __syncwarp();
        auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
          if constexpr (CG == 2) ptx::tma_load_2d_cg2(dst, m, bar_c, c0, c1);
          else ptx::tma_load_2d(dst, m, bar, c0, c1);
        };
        const int k0 = kb * TBK;
        // timing-only experiment: every B tile from expert 0's first panel (results garbage)
        constexpr bool SAMEB = (MOEB_EXP_SAMEB >> KIND) & 1;
        const int bk0 = SAMEB ? 0 : k0, be = SAMEB ? 0 : t.e, bn0 = SAMEB ? 0 : t.n0;
        constexpr bool NOB = (MOEB_EXP_NOB >> KIND) & 1;
        if constexpr (is_route(KIND)) {
          if (lane == 0) load(sA, &mA0, k0, t.m0);
          if (lane == 1) load(sB, &mB0, k0, 0);
        } else if constexpr (KIND == TC_FWD_UP) {
          if (!CPA) ptx::tma_gather4(sA + 512 * lane, &mA0, bar, k0, gi0, gi1, gi2, gi3);
          const bool gated = P.act == 0;
          if constexpr (CG == 1) {
            // gated: B = [W1 tile ; W2 tile] (128 + 128 rows); non-gated: 256 rows of W1
            if (lane == 0) load(sB, &mB0, k0, t.e * P.h + t.n0);
            if (lane == 1) load(sB + C::B_BYTES / 2, gated ? &mB1 : &mB0, k0, t.e * P.h + t.n0 + (gated ? 0 : 128));
          } else {
            // gated: CTA 0 holds the W1 rows, CTA 1 the W2 rows; non-gated: W1 rows n0 + 128 * rank
            if (lane == 0 && !NOB)
              load(sB, (gated && crank) ? &mB1 : &mB0, bk0, be * P.h + bn0 + (gated ? 0 : 128 * (int)crank));
          }
        } else if constexpr (KIND == TC_FWD_DOWN) {
          // M = 128 tail: this CTA's 64 rows start at m0 + 64 * rank (the box's other 64 rows are unused)
          const int arow = (has_mtail<KIND, CG>() && t.seg1 - t.m0 <= 128) ? 64 * (int)crank : rowoff;
          if (lane == 0) load(sA, &mA0, k0, t.m0 + arow);
          if (lane == 1 && !NOB) load(sB, &mB0, bk0, be * P.d + bn0 + coloff);
        } else if constexpr (is_dh(KIND)) {
          if (!CPA) ptx::tma_gather4(sA + 512 * lane, &mA0, bar, k0, gi0, gi1, gi2, gi3);
          if (has_ntail<KIND, CG>() && P.h - t.n0 <= 128) {  // N = 128: one 64-column panel per CTA
            if (lane == 0) load(sB, &mB0, t.n0 + 64 * (int)crank, t.e * P.d + k0);
          } else if (lane < NPANEL && !NOB) {
            load(sB + lane * 8192, &mB0, bn0 + coloff + 64 * lane, be * P.d + bk0);
          }
        } else if constexpr (KIND == TC_BWD_DX) {
          const bool second = k0 >= P.h;
          const int kk = second ? k0 - P.h : k0;
          const int arow = (has_mtail<KIND, CG>() && t.seg1 - t.m0 <= 128) ? 64 * (int)crank : rowoff;
          if (lane == 0) load(sA, second ? &mA1 : &mA0, kk, t.m0 + arow);
          if (lane >= 4 && lane < 4 + NPANEL)
            load(sB + (lane - 4) * 8192, second ? &mB1 : &mB0, t.n0 + coloff + 64 * (lane - 4), t.e * P.h + kk);
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
          if (has_ntail<KIND, CG>() && P.h - t.n0 <= 128) {
            if (lane == 0) load(sB, &mB0, t.n0 + 64 * (int)crank, t.seg0 + k0);
          } else if (lane < NPANEL) {
            load(sB + lane * 8192, &mB0, t.n0 + coloff + 64 * lane, t.seg0 + k0);
          }
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
          const int m = t.m0 + rowoff;
          const bool second = m >= P.h;  // (only for the gated FFN, where M = 2h)
          if (lane >= 2 && lane < 4)
            load(sA + (lane - 2) * 8192, second ? &mA1 : &mA0, (second ? m - P.h : m) + 64 * (lane - 2), t.seg0 + k0);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 8 && warp < 12) {
    // ======================= cp.async row gathers =======================
    // Consecutive lanes copy consecutive 16-byte chunks of the same gathered
    // row (one warp instruction = whole 128-byte lines) into the swizzled
    // layout: chunk c of smem row q lands at q*128 + ((c ^ (q & 7)) << 4).
    if constexpr (CPA && K::gathered) {
      const int gt = threadIdx.x - 256;
      int stage = 0;
      uint32_t phase = 0;
      TileInfo t;
      const __nv_bfloat16* src_base = (KIND == TC_FWD_UP || KIND == TC_DW12) ? P.x : P.dy;
      uint64_t* const done_bar = CG == 2 ? gfull : full;
      for (int it = 0; decode_tile<KIND, CG>(fetch(it), P, s_offs, s_mstart, t); ++it) {
        if constexpr (KIND == TC_FWD_UP || is_dh(KIND)) {
          // K-major A, this CTA's 128 rows x 8 chunks: chunk c = gt&7, rows (gt>>3) + 16 i
          const int c = gt & 7, rb = gt >> 3;
          const __nv_bfloat16* src[8];
          uint32_t nb[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = t.m0 + rowoff + rb + 16 * i;
            const int tok = r < t.seg1 ? P.eti[r] : -1;
            src[i] = src_base + (int64_t)(tok < 0 ? 0 : tok) * P.d + c * 8;
            nb[i] = tok < 0 ? 0u : 16u;
          }
          for (int kb = 0; kb < t.nk; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t sbase = ptx::smem_u32(smem + stage * C::STAGE);
            const int k0 = kb * TBK;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int q = rb + 16 * i;
              ptx::cp_async16(sbase + q * 128 + ((c ^ (q & 7)) << 4), src[i] + k0, nb[i]);
            }
            ptx::cp_async_mbar_arrive(&done_bar[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        } else {
          // MN-major: smem row q = K index (a gathered token row); this CTA copies
          // DW3: 2 panels (its 128 M columns of dY); DW12: 4 (CG 1) / 2 (CG 2)
          // panels of its N columns of X.
          constexpr int NP = (KIND == TC_DW3) ? 2 : NPANEL;
          constexpr int CPR = NP * 8;                // 16-byte chunks per row
          constexpr int RPI = GATHER_THREADS / CPR;  // rows per pass
          constexpr int NPASS = 64 / RPI;
          const int cidx = gt % CPR, rb = gt / CPR;
          const int p = cidx >> 3, cc = cidx & 7;
          const int col = ((KIND == TC_DW3) ? t.m0 + rowoff : t.n0 + coloff) + 64 * p + cc * 8;
          const bool col_ok = col < P.d;
          const uint32_t dst_off = ((KIND == TC_DW3) ? 0u : (uint32_t)TA_BYTES) + p * 8192;
          int tok_next[NPASS];
#pragma unroll
          for (int i = 0; i < NPASS; ++i) {
            const int r = t.seg0 + rb + RPI * i;
            tok_next[i] = (r < t.seg1 && col_ok) ? P.eti[r] : -1;
          }
          for (int kb = 0; kb < t.nk; ++kb) {
            int tok[NPASS];
#pragma unroll
            for (int i = 0; i < NPASS; ++i) tok[i] = tok_next[i];
            if (kb + 1 < t.nk) {  // prefetch the next k-block's row indices
#pragma unroll
              for (int i = 0; i < NPASS; ++i) {
                const int r = t.seg0 + (kb + 1) * TBK + rb + RPI * i;
                tok_next[i] = (r < t.seg1 && col_ok) ? P.eti[r] : -1;
              }
            }
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t sbase = ptx::smem_u32(smem + stage * C::STAGE) + dst_off;
#pragma unroll
            for (int i = 0; i < NPASS; ++i) {
              const int q = rb + RPI * i;
              const __nv_bfloat16* sp = src_base + (int64_t)(tok[i] < 0 ? 0 : tok[i]) * P.d + (col_ok ? col : 0);
              ptx::cp_async16(sbase + q * 128 + ((cc ^ (q & 7)) << 4), sp, tok[i] < 0 ? 0u : 16u);
            }
            ptx::cp_async_mbar_arrive(&done_bar[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 3) {
    // ============ CTA pair: relay this CTA's gather completion to the leader ============
    // The whole warp runs the loop (it stays converged for the final .aligned
    // cluster barrier); lane 0 relays.  The local barrier completes only once
    // this CTA's cp.async writes have landed, so the relay is a relaxed
    // arrive after a generic->async proxy fence: a release.cluster arrive
    // would add a GPU-scope membar per k-block (measured 2x slower).
    if constexpr (CG == 2 && K::gathered) {
      int stage = 0;
      uint32_t phase = 0;
      TileInfo t;
      for (int it = 0; decode_tile<KIND, CG>(fetch(it), P, s_offs, s_mstart, t); ++it) {
        for (int kb = 0; kb < t.nk; ++kb) {
          ptx::mbar_wait(&gfull[stage], phase);
          if (lane == 0) {
            ptx::fence_proxy_async();
            ptx::mbar_arrive_cluster_relaxed(full_c0 + 8u * (uint32_t)stage);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    if (CG == 1 || leader) {
      int stage = 0;
      uint32_t phase = 0;
      int as = 0;
      uint32_t aphase = 0;
      TileInfo t;
      const uint32_t idesc = is_route(KIND) ? P.route_idesc : IDESC;
      const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint32_t s0 = ptx::smem_u32(smem);
      const uint32_t empty0 = ptx::smem_u32(empty);
      for (int it = 0; decode_tile<KIND, CG>(fetch(it), P, s_offs, s_mstart, t); ++it) {
        if constexpr (CG == 2) ptx::mbar_wait_cluster(&tempty[as], aphase ^ 1);
        else ptx::mbar_wait(&tempty[as], aphase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tb + as * TBN;
        uint32_t tidesc = idesc;
        if constexpr (has_mtail<KIND, CG>())
          if (t.seg1 - t.m0 <= 128) tidesc = ptx::umma_idesc_bf16(128, TBN, K::a_mn ? 1 : 0, K::b_mn ? 1 : 0);
        if constexpr (has_ntail<KIND, CG>())
          if (P.h - t.n0 <= 128) tidesc = ptx::umma_idesc_bf16(128 * CG, TBN / 2, K::a_mn ? 1 : 0, K::b_mn ? 1 : 0);
        for (int kb = 0; kb < t.nk; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          if (CPA && K::gathered) ptx::fence_proxy_async();  // cp.async (generic proxy) -> tcgen05 reads
          ptx::tc_fence_after();
          // whole warp converged; elect.sync inside the asm issues from one thread
          // (the descriptors' low words: (smem >> 4) | LBO field, see ptx::umma_kblock)
          constexpr uint32_t LBO_A = K::a_mn ? (8192u >> 4) << 16 : (16u >> 4) << 16;
          constexpr uint32_t LBO_B = K::b_mn ? (8192u >> 4) << 16 : (16u >> 4) << 16;
          constexpr uint32_t STEP_A = K::a_mn ? 2048u >> 4 : 32u >> 4;
          constexpr uint32_t STEP_B = K::b_mn ? 2048u >> 4 : 32u >> 4;
          const uint32_t sA = s0 + stage * C::STAGE;
          if constexpr ((MOEB_EXP_NOMMA >> KIND) & 1) {
            if (lane == 0) {
              if constexpr (CG == 2) ptx::umma_commit_cg2(&empty[stage], 0x3);
              else ptx::umma_commit(&empty[stage]);
            }
            __syncwarp();
          } else if constexpr (WIDE) {
            // two N = 256 MMAs per K16 step into the two accumulators: B columns [0, 128) and
            // [128, 256) of each CTA's 256 (panels 0-1 and 2-3)
            ptx::umma_kblock2<STEP_A, STEP_B>(d_tmem, d_tmem + TBN, (sA >> 4) | LBO_A,
                                              ((sA + TA_BYTES) >> 4) | LBO_B, ((sA + TA_BYTES + 16384) >> 4) | LBO_B,
                                              tidesc, kb != 0, empty0 + 8 * stage, 0x3);
          } else {
            ptx::umma_kblock<CG, STEP_A, STEP_B>(d_tmem, (sA >> 4) | LBO_A, ((sA + TA_BYTES) >> 4) | LBO_B, tidesc,
                                                 kb != 0, empty0 + 8 * stage, 0x3);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) {
          if (t.nk > 0) {
            if constexpr (CG == 2) ptx::umma_commit_cg2(&tfull[as], 0x3);
            else ptx::umma_commit(&tfull[as]);
          } else {
            ptx::mbar_arrive(&tfull[as]);
            if constexpr (CG == 2) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tfull[as]), 1));
          }
        }
        __syncwarp();
        if (WIDE || ++as == 2) { as = 0; aphase ^= 1; }  // the wide tile fills TMEM: one stage
      }
    }
  } else if (warp == 2) {
    // ===================== dynamic tile scheduler (leader) =====================
    // Claims tiles from its die's list first (sched[die]), then from the other
    // die's list, and publishes each into both CTAs' rings; -1 ends the stream.
    if constexpr (DYN) {
      if (leader && lane == 0) {
        const int Mt = K::wgrad ? E * P.m_tiles : s_mstart[E];  // m-tiles over all experts
        int cnt[2] = {Mt * P.n_split, Mt * (P.n_tiles - P.n_split)};
        if (!K::wgrad && P.die_expert) {
          // die 0 takes the experts whose m-tiles start below its SM share of all m-tiles
          const int target = (int)(((int64_t)Mt * P.die_sm0_permille + 500) / 1000);
          int es = 0;
          while (es < E && s_mstart[es + 1] <= target) ++es;
          if (es < E && target - s_mstart[es] > s_mstart[es + 1] - target) ++es;  // nearer boundary
          cnt[0] = s_mstart[es] * P.n_tiles;
          cnt[1] = Mt * P.n_tiles - cnt[0];
        }
        const int my = P.die_map ? (int)P.die_map[ptx::smid() & 255] : 0;
        int src = my;
        for (int it = 0;; ++it) {
          const int slot = it % SCHED_RING;
          ptx::mbar_wait(&sempty[slot], ((uint32_t)(it / SCHED_RING) & 1u) ^ 1u);
          int tile = -1;
          while (src >= 0) {
            const int x = atomicAdd(&P.sched[src], 1);
            if (x < cnt[src]) {
              tile = (src ? cnt[0] : 0) + x;
              break;
            }
            src = (src == my) ? 1 - my : -1;  // own list exhausted: help the other die
          }
          s_ring[slot] = tile;
          ptx::st_cluster_u32(ptx::mapa(ptx::smem_u32(&s_ring[slot]), 1), (uint32_t)tile);
          ptx::mbar_arrive(&sfull[slot]);
          ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&sfull[slot]), 1));  // release: orders the ring write
          if (tile < 0) break;
        }
      }
    }
  } else if ((warp >= 4 && warp < 8) || warp >= 12) {
    // ============================ epilogue ============================
    const int wq = warp & 3;                       // TMEM lane quarter
    const int hc = warp >= 12 ? 1 : 0;             // 8-warp BWD_DH: column half of the tile
    const int ew = wq + 4 * hc;                    // epilogue warp index (staging, barriers)
    constexpr int NCW = C::NEPI == 8 ? TBN / 2 : TBN;  // columns of the tile per warp
    const int cb = hc * NCW;                       // this warp's first column within the tile
    const int row = rowoff + wq * 32 + lane;  // row of the tile owned by this thread
    uint8_t* stg = smem + C::STG_OFF + ew * C::STG_WARP;  // this warp's staging tiles
    int as = 0;
    uint32_t aphase = 0;
    uint32_t gch = 0;  // BWD_DH (TMA epilogue): this warp's running chunk count (ring slot / parity)
    constexpr int DH_PF = C::DH_NBUF - 2;  // chunks loaded ahead (slot reuse distance 2: wait_read<1>)
    // BWD_DH epilogue TMA: 32-row x DH_CW-column bf16 boxes (32-byte swizzle = the stg8_off
    // layout) of A (mA0), B (mA1) loaded and dA, dB, wU (mB1) stored by lane 0
    constexpr int CW = C::DH_CW, HALF = C::DH_SLOT / 2;
    auto dh_load = [&](uint32_t g, int col, int row0) {
      const int slot = (int)(g % C::DH_NBUF);
      uint64_t* bar = &ebar[ew * C::DH_NBUF + slot];
      uint8_t* NA = stg + slot * C::DH_SLOT;
      ptx::mbar_arrive_expect_tx(bar, P.act == 0 ? 2u * HALF : (uint32_t)HALF);
      ptx::tma_load_2d(NA, &mA0, bar, col, row0);
      if (P.act == 0) ptx::tma_load_2d(NA + HALF, &mA1, bar, col, row0);
    };
    TileInfo t;
    for (int it = 0; decode_tile<KIND, CG>(fetch(it), P, s_offs, s_mstart, t); ++it) {
      if constexpr (is_dh(KIND) && CPA && MOEB_DH_TMA) {
        // the epilogue inputs (A, B rows of this tile) do not depend on the
        // accumulator: start their TMA loads before waiting for it
        const int r0w = t.m0 + rowoff + wq * 32;
        const int nchunk = max(0, min(NCW, P.h - t.n0 - cb)) / CW;
        if (lane == 0) {
          ptx::bulk_wait_read<1>();
          for (int ci = 0; ci < DH_PF && ci < nchunk; ++ci) dh_load(gch + ci, t.n0 + cb + CW * ci, r0w);
        }
        __syncwarp();
        if constexpr (MOEB_DH_L2PF) {
          // the NEXT tile's A, B rows of this warp go to L2 now, a whole tile ahead: the
          // ring's TMA loads then hit L2 instead of paying HBM latency DH_PF chunks ahead.
          // One row per lane, plain prefetch.global.L2 (LSU, not the TMA unit, which the
          // mainloop's W3 loads and the epilogue's boxes keep busy)
          int nt = 0;
          if (lane == 0) nt = peek(it + 1);
          nt = __shfl_sync(0xffffffffu, nt, 0);
          TileInfo tn;
          if (decode_tile<KIND, CG>(nt, P, s_offs, s_mstart, tn)) {
            const int rn = tn.m0 + rowoff + wq * 32 + lane;
            const int ncol = max(0, min(NCW, P.h - tn.n0 - cb));
            if (rn < tn.seg1)
              for (int c = 0; c < ncol; c += 64) {  // 128-byte lines
                const int64_t o = (int64_t)rn * P.h + tn.n0 + cb + c;
                ptx::prefetch_l2(P.a_save + o);
                if (P.act == 0) ptx::prefetch_l2(P.b_save + o);
              }
          }
        }
      } else if constexpr (is_dh(KIND)) {
        // the epilogue inputs (A, B rows of this tile) do not depend on the
        // accumulator: start streaming the first chunks before waiting for it
        const int r0w = t.m0 + rowoff + wq * 32;
        const int nvalid = max(0, min(32, t.seg1 - r0w));
        const int nchunk = min(TBN, P.h - t.n0) / 32;
        const int64_t o0 = (int64_t)r0w * P.h + t.n0;
#pragma unroll
        for (int ci = 0; ci < C::DH_NBUF - 1; ++ci) {
          if (ci < nchunk) {
            uint8_t* NA = stg + ci * 4096;
            stg_load_bf16_async(NA, lane, P.a_save + o0 + ci * 32, P.h, nvalid);
            if (P.act == 0) stg_load_bf16_async(NA + 2048, lane, P.b_save + o0 + ci * 32, P.h, nvalid);
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        }
      }
      ptx::mbar_wait(&tfull[as], aphase);
      ptx::tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(wq * 32) << 16) + as * TBN;
      uint32_t v[32];
      if constexpr ((MOEB_EXP_NOEPI >> KIND) & 1) {
        if constexpr (is_dh(KIND) && CPA && MOEB_DH_TMA) {
          const int nchunk = max(0, min(NCW, P.h - t.n0 - cb)) / CW;
          for (int ci = 0; ci < DH_PF && ci < nchunk; ++ci, ++gch)
            ptx::mbar_wait(&ebar[ew * C::DH_NBUF + (int)(gch % C::DH_NBUF)], (gch / C::DH_NBUF) & 1);
        } else if constexpr (is_dh(KIND)) {
          asm volatile("cp.async.wait_all;" ::: "memory");
        }
      } else if constexpr (KIND == TC_ROUTE_S) {
        // E <= 64: the token's logits are read from TMEM once into registers; max,
        // softmax denominator and the top-k scans (desc, ties -> lower id) run on them
        const int r = t.m0 + row;
        const bool valid = r < P.T;
        uint32_t v1[32];
        ptx::tmem_ld32(tb, v);
        if (P.route_n > 32) ptx::tmem_ld32(tb + 32, v1);
        ptx::tmem_wait_ld();
        float lg[64];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          lg[i] = i < E ? __uint_as_float(v[i]) : -INFINITY;
          lg[32 + i] = (32 + i < E && P.route_n > 32) ? __uint_as_float(v1[i]) : -INFINITY;
        }
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < 64; ++i) mx = fmaxf(mx, lg[i]);
        if (valid) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (i < E) P.logits[(int64_t)r * E + i] = lg[i];
        }
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (i < E) sum += expf(lg[i] - mx);
        uint64_t taken = 0;
        float wsum = 0.f;
        int sel_e[16];
        float sel_p[16];
#pragma unroll 1
        for (int j = 0; j < P.k; ++j) {
          float bv = -INFINITY;
          int be = 0x7fffffff;
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            if (i < E && !((taken >> i) & 1ull) && (lg[i] > bv || (lg[i] == bv && i < be))) {
              bv = lg[i];
              be = i;
            }
          }
          taken |= 1ull << be;
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
      } else if constexpr (is_route(KIND)) {
        // one token row per thread: logits out, softmax, top-k (desc, ties -> lower id)
        const int r = t.m0 + row;
        const bool valid = r < P.T;
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
      } else if constexpr (KIND == TC_FWD_UP && C::NEPI == 8) {
        // 8 warps: this warp's 32 rows x (gated) columns hc*64 .. +63 of A (TMEM 0-127) and of
        // B (TMEM 128-255), or (non-gated) columns cb .. cb+127 of A; 16-column chunks through
        // three 32 x 16 swizzled tiles (A, B, U)
        const int r0w = t.m0 + rowoff + wq * 32;
        const int nvalid = max(0, min(32, t.seg1 - r0w));
        uint8_t* T0 = stg;
        uint8_t* T1 = stg + 1024;
        uint8_t* T2 = stg + 2048;
        const bool gated = P.act == 0;
        const int cbeg = gated ? hc * 64 : cb, cend = gated ? cbeg + 64 : cb + NCW;
        const int rr = t.m0 + row;
        const float uw = !P.u_weighted ? 1.f : (rr < t.seg1 ? P.topw[P.row_slot[rr]] : 0.f);
#pragma unroll 1
        for (int c = cbeg; c < cend; c += 16) {
          if (!gated && t.n0 + c >= P.h) break;
          uint32_t va[16], vb[16];
          ptx::tmem_ld16(tb + c, va);
          if (gated) ptx::tmem_ld16(tb + 128 + c, vb);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint32_t oa[4], ob[4], ou[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a0 = __uint_as_float(va[8 * q + 2 * e]), a1 = __uint_as_float(va[8 * q + 2 * e + 1]);
              oa[e] = ptx::pack_bf16(a0, a1);
              if (gated) {
                const float b0 = __uint_as_float(vb[8 * q + 2 * e]), b1 = __uint_as_float(vb[8 * q + 2 * e + 1]);
                ob[e] = ptx::pack_bf16(b0, b1);
                ou[e] = ptx::pack_bf16(uw * (a0 * sigmoid_fast(a0) * b0), uw * (a1 * sigmoid_fast(a1) * b1));
              } else {
                ob[e] = 0u;
                ou[e] = ptx::pack_bf16(uw * act_fwd(P.act, a0, sigmoid_fast(a0)), uw * act_fwd(P.act, a1, sigmoid_fast(a1)));
              }
            }
            *reinterpret_cast<uint4*>(T0 + stg8_off(lane, q)) = make_uint4(oa[0], oa[1], oa[2], oa[3]);
            if (gated) *reinterpret_cast<uint4*>(T1 + stg8_off(lane, q)) = make_uint4(ob[0], ob[1], ob[2], ob[3]);
            *reinterpret_cast<uint4*>(T2 + stg8_off(lane, q)) = make_uint4(ou[0], ou[1], ou[2], ou[3]);
          }
          __syncwarp();
          if (nvalid > 0) {
            // output column of A/B/U: n0 counts A columns (stacked tiles: n0 = n_tile * 128)
            const int64_t o = (int64_t)r0w * P.h + t.n0 + c;
            stg8_store_bf16(T0, lane, P.a_save + o, P.h, nvalid);
            if (gated) stg8_store_bf16(T1, lane, P.b_save + o, P.h, nvalid);
            stg8_store_bf16(T2, lane, P.u + o, P.h, nvalid);
          }
          __syncwarp();
        }
      } else if constexpr (KIND == TC_FWD_UP) {
        const int r0w = t.m0 + rowoff + wq * 32;  // first row of this warp
        const int nvalid = max(0, min(32, t.seg1 - r0w));
        uint8_t* T0 = stg;
        uint8_t* T1 = stg + 2048;
        uint8_t* T2 = stg + 4096;
        uint32_t bv[32];
        // MOE_CKPT_ABU: the stored activation is wU (the gate weight of this row folded in)
        const int rr = t.m0 + row;
        const float uw = !P.u_weighted ? 1.f : (rr < t.seg1 ? P.topw[P.row_slot[rr]] : 0.f);
        if (P.act != 0) {  // non-gated: 256 columns of A, U = sigma(A)
#pragma unroll 1
          for (int c = 0; c < TBN; c += 32) {
            if (t.n0 + c >= P.h) break;
            ptx::tmem_ld32(tb + c, v);
            ptx::tmem_wait_ld();
            float a[32], u[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              a[i] = __uint_as_float(v[i]);
              u[i] = uw * act_fwd(P.act, a[i], sigmoid_fast(a[i]));
            }
            stg_put_bf16(T0, lane, a);
            stg_put_bf16(T2, lane, u);
            __syncwarp();
            if (nvalid > 0) {
              const int64_t o = (int64_t)r0w * P.h + t.n0 + c;
              stg_store_bf16(T0, lane, P.a_save + o, P.h, nvalid);
              stg_store_bf16(T2, lane, P.u + o, P.h, nvalid);
            }
            __syncwarp();
          }
        }
#pragma unroll 1
        for (int c = 0; c < (P.act == 0 ? 128 : 0); c += 32) {
          ptx::tmem_ld32(tb + c, v);
          ptx::tmem_ld32(tb + 128 + c, bv);
          ptx::tmem_wait_ld();
          float a[32], b[32], u[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            a[i] = __uint_as_float(v[i]);
            b[i] = __uint_as_float(bv[i]);
            u[i] = uw * (a[i] * sigmoid_fast(a[i]) * b[i]);
          }
          stg_put_bf16(T0, lane, a);
          stg_put_bf16(T1, lane, b);
          stg_put_bf16(T2, lane, u);
          __syncwarp();
          if (nvalid > 0) {
            const int64_t o = (int64_t)r0w * P.h + t.n0 + c;
            stg_store_bf16(T0, lane, P.a_save + o, P.h, nvalid);
            stg_store_bf16(T1, lane, P.b_save + o, P.h, nvalid);
            stg_store_bf16(T2, lane, P.u + o, P.h, nvalid);
          }
          __syncwarp();
        }
      } else if constexpr (KIND == TC_FWD_DOWN || KIND == TC_BWD_DX) {
        // rows / columns of this warp (M = 128 tail: 32 rows x 128 columns, see has_mtail)
        static_assert(!(WIDE && has_mtail<KIND, CG>()), "wide tiles have no M = 128 tail variant");
        const bool half = has_mtail<KIND, CG>() && t.seg1 - t.m0 <= 128;
        const int r0w = t.m0 + (half ? 64 * (int)crank + 32 * (wq & 1) : rowoff + wq * 32);
        const int coff = half ? 128 * (wq >> 1) : cb;  // first output column of this warp
        const int tcol = half ? 0 : cb;                // its first TMEM column
        const int ncol = half ? 128 : (WIDE ? tile_n<KIND, CG>() : NCW);
        const int r = r0w + lane;
        const int nvalid = max(0, min(32, t.seg1 - r0w));
        const int N = P.d;
        [[maybe_unused]] const uint64_t pol = MOEB_RED_EVICT_LAST ? ptx::policy_evict_last() : 0ull;
        float w = 1.f;
        int tok = 0;
        if (r < t.seg1) {
          tok = P.eti[r];
          if constexpr (KIND == TC_FWD_DOWN) w = P.u_weighted ? 1.f : P.topw[P.row_slot[r]];
        }
#pragma unroll 1
        for (int cc = 0; cc < ncol; cc += 32) {
          // output column within the tile (wide: TMEM column cc of accumulator cc / 256 holds tile
          // column 256 r + 128 (cc / 256) + j, r = (cc % 256) / 128 the CTA whose B rows made it)
          const int c = WIDE ? 256 * ((cc & 255) >> 7) + 128 * (cc >> 8) + (cc & 127) : coff + cc;
          if (t.n0 + c >= N) {
            if constexpr (WIDE) continue;
            else break;
          }
          ptx::tmem_ld32(tb + tcol + cc, v);
          ptx::tmem_wait_ld();
          if constexpr (MOEB_BULK_RED) {
            if (P.out_mode == OUT_RED) {
              // lane = row: its 32 scaled values in row-major staging (pitch 144 B: the 16-byte
              // stores of 8 lanes per phase hit distinct banks), then one lane issues a 128-byte
              // bulk reduction per row into the token's accumulator row
              if (lane == 0) ptx::bulk_wait_read<0>();  // the previous chunk's reductions read it
              __syncwarp();
              float4* srow = reinterpret_cast<float4*>(stg + lane * 144);
#pragma unroll
              for (int q = 0; q < 8; ++q)
                srow[q] = make_float4(w * __uint_as_float(v[4 * q]), w * __uint_as_float(v[4 * q + 1]),
                                      w * __uint_as_float(v[4 * q + 2]), w * __uint_as_float(v[4 * q + 3]));
              ptx::fence_proxy_async();  // generic smem writes -> the async proxy's reads
              __syncwarp();
              const float* dst = P.acc_out + (int64_t)tok * N + t.n0 + c;
              const uint32_t s0 = ptx::smem_u32(stg);
              for (int rr = 0; rr < nvalid; ++rr) {
                const float* d_rr = reinterpret_cast<const float*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst), rr));
                if (lane == 0) ptx::bulk_red_add_f32(d_rr, s0 + 144u * (uint32_t)rr, 128u);
              }
              if (lane == 0) ptx::bulk_commit();
              __syncwarp();
              continue;
            }
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float4*>(stg + stg32_off(lane, q)) =
                make_float4(w * __uint_as_float(v[4 * q]), w * __uint_as_float(v[4 * q + 1]),
                            w * __uint_as_float(v[4 * q + 2]), w * __uint_as_float(v[4 * q + 3]));
          __syncwarp();
          if (P.out_mode == OUT_TOKN) {  // k = 1: one row per token, final dtype, 16-byte stores
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const int rr = it * 8 + (lane >> 2), q = lane & 3;
              const int tr = __shfl_sync(0xffffffffu, tok, rr);
              if (rr < nvalid) {
                const float4 f0 = *reinterpret_cast<const float4*>(stg + stg32_off(rr, 2 * q));
                const float4 f1 = *reinterpret_cast<const float4*>(stg + stg32_off(rr, 2 * q + 1));
                uint4 o;
                o.x = ptx::pack_bf16(f0.x, f0.y); o.y = ptx::pack_bf16(f0.z, f0.w);
                o.z = ptx::pack_bf16(f1.x, f1.y); o.w = ptx::pack_bf16(f1.z, f1.w);
                *reinterpret_cast<uint4*>(P.out_tok + (int64_t)tr * N + t.n0 + c + 8 * q) = o;
              }
            }
          } else {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int rr = it * 4 + (lane >> 3), q = lane & 7;
              const int tr = __shfl_sync(0xffffffffu, tok, rr);
              if (rr < nvalid) {
                const float4 f = *reinterpret_cast<const float4*>(stg + stg32_off(rr, q));
                if (P.out_mode == OUT_RED) {
                  if constexpr (MOEB_RED_EVICT_LAST)
                    ptx::red_add_v4_hint(P.acc_out + (int64_t)tr * N + t.n0 + c + 4 * q, f.x, f.y, f.z, f.w, pol);
                  else
                    ptx::red_add_v4(P.acc_out + (int64_t)tr * N + t.n0 + c + 4 * q, f.x, f.y, f.z, f.w);
                }
                else  // OUT_ROWS: expert-sorted row r0w + rr; OUT_TOK: token tr
                  *reinterpret_cast<float4*>(P.acc_out + (int64_t)(P.out_mode == OUT_ROWS ? r0w + rr : tr) * N +
                                             t.n0 + c + 4 * q) = f;
              }
            }
          }
          __syncwarp();
        }
      } else if constexpr (is_dh(KIND) && CPA && MOEB_DH_TMA) {
        // A, B chunks of CW columns arrive by TMA in a ring of DH_NBUF slots (A at +0,
        // B at +HALF of each slot; DH_PF chunks ahead, the first ones issued before
        // the accumulator was ready); dA, dB overwrite the consumed slot, wU goes to one
        // of two tiles, and lane 0 stores the three 32 x CW boxes by TMA (rows past the
        // segment belong to the next expert: a partial row group is stored by hand).
        // TC_BWD_DH_LK's 16-column chunks keep the ring small enough for a 5-stage mainloop.
        const int r = t.m0 + row;
        const bool valid = r < t.seg1;
        const int r0w = t.m0 + rowoff + wq * 32;
        const int nvalid = max(0, min(32, t.seg1 - r0w));
        const float w = valid ? P.topw[P.row_slot[r]] : 0.f;
        constexpr int NBUF = C::DH_NBUF;
        const int nchunk = max(0, min(NCW, P.h - t.n0 - cb)) / CW;
        const int64_t o0 = (int64_t)r0w * P.h + t.n0 + cb;
        float rowsum = 0.f;
        uint32_t vw[CW];
        if (nchunk > 0) tmem_ldw<CW>(tb + cb, vw);
#pragma unroll 1
        for (int ci = 0; ci < nchunk; ++ci, ++gch) {
          const int slot = (int)(gch % NBUF);
          uint8_t* TA = stg + slot * C::DH_SLOT;
          uint8_t* TB = TA + HALF;
          uint8_t* TU = stg + NBUF * C::DH_SLOT + (gch & 1) * HALF;
          if (lane == 0) {
            ptx::bulk_wait_read<1>();  // chunk gch-2's stores have read their slot and wU tile
            if (ci + DH_PF < nchunk) dh_load(gch + DH_PF, t.n0 + cb + CW * (ci + DH_PF), r0w);
          }
          __syncwarp();
          ptx::mbar_wait(&ebar[ew * NBUF + slot], (gch / NBUF) & 1);
          // accumulator chunk ci was loaded (asynchronously) one iteration ago
          ptx::tmem_wait_ld();
          uint32_t dh[CW];
#pragma unroll
          for (int i = 0; i < CW; ++i) dh[i] = vw[i];
          if (ci + 1 < nchunk) tmem_ldw<CW>(tb + cb + (ci + 1) * CW, vw);  // overlap the next TMEM read
#pragma unroll
          for (int q = 0; q < CW / 8; ++q) {
            const uint4 ua = *reinterpret_cast<const uint4*>(TA + stgw_off<CW>(lane, q));
            const uint4 ub = *reinterpret_cast<const uint4*>(TB + stgw_off<CW>(lane, q));
            const uint32_t* pa = reinterpret_cast<const uint32_t*>(&ua);
            const uint32_t* pb = reinterpret_cast<const uint32_t*>(&ub);
            uint32_t oa[4], ob[4], ou[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 a2 = ptx::unpack_bf16(pa[e]);
              const float2 b2 = ptx::unpack_bf16(pb[e]);
              float ra[2], rb[2], ru[2];
              const float av[2] = {a2.x, a2.y}, bvv[2] = {b2.x, b2.y};
#pragma unroll
              for (int z = 0; z < 2; ++z) {
                const float dH = __uint_as_float(dh[q * 8 + e * 2 + z]);
                const float a = av[z], b = bvv[z];
                const float sg = sigmoid_fast(a);
                const float dU = w * dH;
                if (P.act == 0) {
                  const float S = a * sg;
                  const float U = S * b;
                  rowsum = fmaf(dH, U, rowsum);
                  ra[z] = dU * b * sg * (1.f + a * (1.f - sg));
                  rb[z] = dU * S;
                  ru[z] = w * U;
                } else {  // non-gated: U = sigma(A), dA = dU sigma'(A)
                  const float U = act_fwd(P.act, a, sg);
                  rowsum = fmaf(dH, U, rowsum);
                  ra[z] = dU * act_grad(P.act, a, sg);
                  rb[z] = 0.f;
                  ru[z] = w * U;
                }
              }
              oa[e] = ptx::pack_bf16(ra[0], ra[1]);
              ob[e] = ptx::pack_bf16(rb[0], rb[1]);
              ou[e] = ptx::pack_bf16(ru[0], ru[1]);
            }
            *reinterpret_cast<uint4*>(TA + stgw_off<CW>(lane, q)) = make_uint4(oa[0], oa[1], oa[2], oa[3]);
            *reinterpret_cast<uint4*>(TB + stgw_off<CW>(lane, q)) = make_uint4(ob[0], ob[1], ob[2], ob[3]);
            if (!P.dh_skip_u)
              *reinterpret_cast<uint4*>(TU + stgw_off<CW>(lane, q)) = make_uint4(ou[0], ou[1], ou[2], ou[3]);
          }
          ptx::fence_proxy_async();  // generic smem writes -> visible to the TMA stores
          __syncwarp();
          if (nvalid == 32) {
            if (lane == 0) {
              const int col = t.n0 + cb + CW * ci;
              ptx::tma_store_2d(&mA0, TA, col, r0w);
              if (P.act == 0) ptx::tma_store_2d(&mA1, TB, col, r0w);
              if (!P.dh_skip_u) ptx::tma_store_2d(&mB1, TU, col, r0w);
            }
          } else if (nvalid > 0) {
            const int64_t o = o0 + ci * CW;
            if constexpr (CW == 16) {
              stg8_store_bf16(TA, lane, P.a_save + o, P.h, nvalid);
              if (P.act == 0) stg8_store_bf16(TB, lane, P.b_save + o, P.h, nvalid);
              if (!P.dh_skip_u) stg8_store_bf16(TU, lane, P.u + o, P.h, nvalid);
            } else {
              stg_store_bf16(TA, lane, P.a_save + o, P.h, nvalid);
              if (P.act == 0) stg_store_bf16(TB, lane, P.b_save + o, P.h, nvalid);
              if (!P.dh_skip_u) stg_store_bf16(TU, lane, P.u + o, P.h, nvalid);
            }
          }
          if (lane == 0) ptx::bulk_commit();  // one (possibly empty) group per chunk
          __syncwarp();
        }
        if (valid) P.dg_part[(int64_t)r * P.dg_parts + t.n_tile * (C::NEPI == 8 ? 2 : 1) + hc] = rowsum;
      } else if constexpr (is_dh(KIND)) {
        // A, B chunks of 32 columns stream through a ring of DH_NBUF cp.async
        // staging buffers (A at +0, B at +2048 of each 4 KB slot; the first
        // slots are filled before the accumulator is ready); dA and dB
        // overwrite the consumed input slot, wU goes to its own tile.  The
        // next chunk's TMEM read is issued before this chunk is processed.
        const int r = t.m0 + row;
        const bool valid = r < t.seg1;
        const int r0w = t.m0 + rowoff + wq * 32;
        const int nvalid = max(0, min(32, t.seg1 - r0w));
        const float w = valid ? P.topw[P.row_slot[r]] : 0.f;
        constexpr int NBUF = C::DH_NBUF;
        uint8_t* TU = stg + NBUF * 4096;
        const int nchunk = min(TBN, P.h - t.n0) / 32;
        const int64_t o0 = (int64_t)r0w * P.h + t.n0;
        float rowsum = 0.f;
        if (nchunk > 0) ptx::tmem_ld32(tb, v);
#pragma unroll 1
        for (int ci = 0; ci < nchunk; ++ci) {
          uint8_t* TA = stg + (ci % NBUF) * 4096;
          uint8_t* TB = TA + 2048;
          {  // keep NBUF-1 chunks in flight: one commit group per iteration (possibly empty)
            const int nx = ci + NBUF - 1;
            if (nx < nchunk) {
              uint8_t* NA = stg + (nx % NBUF) * 4096;
              stg_load_bf16_async(NA, lane, P.a_save + o0 + nx * 32, P.h, nvalid);
              if (P.act == 0) stg_load_bf16_async(NA + 2048, lane, P.b_save + o0 + nx * 32, P.h, nvalid);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group %0;" ::"n"(NBUF - 1) : "memory");
          }
          // accumulator chunk ci was loaded (asynchronously) one iteration ago
          ptx::tmem_wait_ld();
          uint32_t dh[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) dh[i] = v[i];
          if (ci + 1 < nchunk) ptx::tmem_ld32(tb + (ci + 1) * 32, v);  // overlap the next TMEM read
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 ua = *reinterpret_cast<const uint4*>(TA + stg16_off(lane, q));
            const uint4 ub = *reinterpret_cast<const uint4*>(TB + stg16_off(lane, q));
            const uint32_t* pa = reinterpret_cast<const uint32_t*>(&ua);
            const uint32_t* pb = reinterpret_cast<const uint32_t*>(&ub);
            uint32_t oa[4], ob[4], ou[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 a2 = ptx::unpack_bf16(pa[e]);
              const float2 b2 = ptx::unpack_bf16(pb[e]);
              float ra[2], rb[2], ru[2];
              const float av[2] = {a2.x, a2.y}, bvv[2] = {b2.x, b2.y};
#pragma unroll
              for (int z = 0; z < 2; ++z) {
                const float dH = __uint_as_float(dh[q * 8 + e * 2 + z]);
                const float a = av[z], b = bvv[z];
                const float sg = sigmoid_fast(a);
                const float dU = w * dH;
                if (P.act == 0) {
                  const float S = a * sg;
                  const float U = S * b;
                  rowsum = fmaf(dH, U, rowsum);
                  ra[z] = dU * b * sg * (1.f + a * (1.f - sg));
                  rb[z] = dU * S;
                  ru[z] = w * U;
                } else {  // non-gated: U = sigma(A), dA = dU sigma'(A)
                  const float U = act_fwd(P.act, a, sg);
                  rowsum = fmaf(dH, U, rowsum);
                  ra[z] = dU * act_grad(P.act, a, sg);
                  rb[z] = 0.f;
                  ru[z] = w * U;
                }
              }
              oa[e] = ptx::pack_bf16(ra[0], ra[1]);
              ob[e] = ptx::pack_bf16(rb[0], rb[1]);
              ou[e] = ptx::pack_bf16(ru[0], ru[1]);
            }
            *reinterpret_cast<uint4*>(TA + stg16_off(lane, q)) = make_uint4(oa[0], oa[1], oa[2], oa[3]);
            *reinterpret_cast<uint4*>(TB + stg16_off(lane, q)) = make_uint4(ob[0], ob[1], ob[2], ob[3]);
            *reinterpret_cast<uint4*>(TU + stg16_off(lane, q)) = make_uint4(ou[0], ou[1], ou[2], ou[3]);
          }
          __syncwarp();
          if (nvalid > 0) {
            const int64_t o = o0 + ci * 32;
            stg_store_bf16(TA, lane, P.a_save + o, P.h, nvalid);
            if (P.act == 0) stg_store_bf16(TB, lane, P.b_save + o, P.h, nvalid);
            if (!P.dh_skip_u) stg_store_bf16(TU, lane, P.u + o, P.h, nvalid);
          }
          __syncwarp();
        }
        if (valid) P.dg_part[(int64_t)r * P.dg_parts + t.n_tile] = rowsum;
      } else {  // DW3 / DW12: store the weight-gradient tile
        const int M = (KIND == TC_DW3) ? P.d : (P.act == 0 ? 2 : 1) * P.h;
        const int m0w = t.m0 + rowoff + wq * 32;
        const int nvalid = max(0, min(32, M - m0w));
        __nv_bfloat16* base;
        int N;
        if constexpr (KIND == TC_DW3) {
          N = P.h;
          base = P.out0 + (int64_t)t.e * P.d * P.h + (int64_t)m0w * P.h;
        } else {  // a warp's 32 rows lie entirely in dW1 or in dW2 (h % 128 == 0)
          N = P.d;
          base = (m0w < P.h) ? P.out0 + (int64_t)t.e * P.h * P.d + (int64_t)m0w * P.d
                             : P.out1 + (int64_t)t.e * P.h * P.d + (int64_t)(m0w - P.h) * P.d;
        }
#pragma unroll 1
        for (int c = 0; c < tile_n<KIND, CG>(); c += 32) {
          // wide tile: TMEM column c of accumulator c / 256 holds tile column 256 r + 128 (c / 256) + j,
          // r = (c % 256) / 128 the CTA whose B columns produced it, j = c % 128
          const int oc = WIDE ? 256 * ((c & 255) >> 7) + 128 * (c >> 8) + (c & 127) : c;
          if (t.n0 + oc >= N) {
            if constexpr (WIDE) continue;
            else break;
          }
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
          stg_put_bf16(stg, lane, f);
          __syncwarp();
          if (nvalid > 0) stg_store_bf16(stg, lane, base + t.n0 + oc, N, nvalid);
          __syncwarp();
        }
      }
      // the accumulator stage is free: its tcgen05.ld's have completed (tcgen05.wait::ld) and
      // the fence orders them before the arrive.  Relaxed: a release.cluster arrive compiles to
      // MEMBAR.ALL.GPU, which would make every epilogue warp wait for its own red.adds / stores
      // to drain at the end of each tile (nothing the MMA warp reads depends on them)
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) {
          if constexpr (MOEB_TEMPTY_RELAXED) ptx::mbar_arrive_cluster_relaxed(tempty_c0 + 8u * (uint32_t)as);
          else ptx::mbar_arrive_cluster(tempty_c0 + 8u * (uint32_t)as);
        } else {
          ptx::mbar_arrive(&tempty[as]);
        }
      }
      if (WIDE || ++as == 2) { as = 0; aphase ^= 1; }
    }
    if constexpr ((is_dh(KIND) && CPA && MOEB_DH_TMA) || (MOEB_BULK_RED && (KIND == TC_FWD_DOWN || KIND == TC_BWD_DX)))
      if (lane == 0) ptx::bulk_wait<0>();  // the epilogue's TMA stores / bulk reductions are complete
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();
  else __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    if constexpr (CG == 2) ptx::tmem_dealloc_cg2(tmem_base, 512);
    else ptx::tmem_dealloc(tmem_base, 512);
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

// 2D bf16 row-major [rows, cols] map with a 32-row x cw-column box (cw = 16: 32-byte
// swizzle = stg8_off; cw = 32: 64-byte swizzle = stg16_off), the BWD_DH epilogue tiles
static bool make_map_epi(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t cw) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {cw, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, cw == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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

// Engine selection (MOEBLAZE_GEMM): "pair" (default) = CTA pair + cp.async
// gathers; "cta" = one CTA per tile + cp.async gathers; "tma" = one CTA per
// tile + TMA tile::gather4.  The alternatives are kept for the measured
// comparison in DESIGN.md / profiles.
enum Engine { ENG_PAIR = 0, ENG_CTA = 1, ENG_TMA = 2 };
static Engine engine() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOEBLAZE_GEMM");
    v = ENG_PAIR;
    if (e && e[0] == 'c') v = ENG_CTA;
    if (e && e[0] == 't') v = ENG_TMA;
  }
  return (Engine)v;
}

template <int KIND, bool CPA, int CG>
static moe_status launch_tc_impl(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0,
                                 const CUtensorMap& b1, const TcParams& P, int64_t tiles, cudaStream_t st) {
  static bool attr = false;
  auto kern = tc_gemm_kernel<KIND, CPA, CG>;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CgCfg<CG, KIND>::SMEM) != cudaSuccess)
      return MOE_ERR_CUDA;
    attr = true;
  }
  if (tiles <= 0) return MOE_OK;
  // sm_reserve: SMs left free for a concurrent kernel (an exchange overlapping this GEMM)
  const int avail = std::max(CG, num_sms() - std::max(0, P.sm_reserve));
  const int groups = (int)std::min<int64_t>(tiles, avail / CG);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(groups * CG);
  cfg.blockDim = dim3(tc_threads(KIND));
  cfg.dynamicSmemBytes = CgCfg<CG, KIND>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CG;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, a0, a1, b0, b1, P) != cudaSuccess) return MOE_ERR_CUDA;
  note_launch();
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}



// tiles_for(TM): number of tiles (an upper bound for row kinds) at tile height TM
template <int KIND, typename F>
static moe_status launch_tc(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0,
                            const CUtensorMap& b1, TcParams P, F tiles_for, cudaStream_t st) {
  switch (engine()) {
    case ENG_PAIR:
      P.m_tiles = P.m_tiles2;
      if constexpr (dyn_sched<KIND, 2>()) {
        // split every expert's n-tiles between the dies in proportion to their SMs
        int n_sm[2];
        P.die_map = sm_die_map(n_sm);
        P.n_split = P.n_tiles;
        P.die_expert = 0;
        if (MOEB_DIE_EXPERT && !KindTraits<KIND>::wgrad && P.die_map && n_sm[1] > 0 && P.E >= 2) {
          P.die_expert = 1;  // one list per die over all n-tiles, split at an expert boundary
          P.die_sm0_permille = (int)((1000LL * n_sm[0]) / (n_sm[0] + n_sm[1]));
        } else if (P.die_map && n_sm[1] > 0 && P.n_tiles >= 2) {
          const int ns = (int)((2LL * P.n_tiles * n_sm[0] + (n_sm[0] + n_sm[1])) / (2LL * (n_sm[0] + n_sm[1])));
          P.n_split = std::min(std::max(ns, 1), P.n_tiles - 1);
        }
        // claim counters: the caller's 16-byte workspace slot for this launch, zeroed on the
        // launch stream (stream-ordered, so CUDA-graph replays and other streams never share them)
        if (!P.sched || cudaMemsetAsync(P.sched, 0, 4 * sizeof(int), st) != cudaSuccess) return MOE_ERR_CUDA;
      }
      return launch_tc_impl<KIND, true, 2>(a0, a1, b0, b1, P, tiles_for(256), st);
    case ENG_CTA: return launch_tc_impl<KIND, true, 1>(a0, a1, b0, b1, P, tiles_for(128), st);
    default: return launch_tc_impl<KIND, false, 1>(a0, a1, b0, b1, P, tiles_for(128), st);
  }
}

// BWD_DH variants in the CTA-pair engine (TMA epilogue, 16-column chunks): 8 epilogue warps /
// 4 stages (TC_BWD_DH_LK) below MOEB_DH_L5_MIN_D, 4 warps / 5 stages (TC_BWD_DH_L5) from it
#ifndef MOEB_DH_LK_MIN_D
#define MOEB_DH_LK_MIN_D 0
#endif
#ifndef MOEB_DH_L5_MIN_D
#define MOEB_DH_L5_MIN_D 3072
#endif
static bool dh_long_k(int d) { return MOEB_DH_TMA && engine() == ENG_PAIR && d >= MOEB_DH_LK_MIN_D; }
static bool dh_l5(int d) { return dh_long_k(d) && d >= MOEB_DH_L5_MIN_D; }
// gate-grad partial columns per routed row written by BWD_DH (one per n-tile, two with the
// 8-warp epilogue, whose column halves each write their own)
int tc_dg_parts(int h, int d) {
  const bool two = dh_long_k(d) && !dh_l5(d) && n_epi(TC_BWD_DH_LK) == 8;
  return (int)ceil_div(h, TBN) * (two ? 2 : 1);
}

// K1 on tensor cores (bf16): logits = X Wg^T with M = 128 tokens, N = E padded
// to a multiple of 16 (rows past E are TMA zero-fill), K = d.
moe_status tc_route(const moe_problem* p, const void* x, const void* wg, float* logits, int32_t* ids, float* topw,
                    cudaStream_t st) {
  if (p->T == 0) return MOE_OK;
  TcParams P{};
  P.T = (int)p->T; P.d = p->d; P.h = p->h; P.E = p->E;
  P.logits = logits; P.ids = ids; P.route_w = topw; P.k = p->k; P.renorm = p->renormalize;
  P.route_n = std::max(16, (int)ceil_div(p->E, 16) * 16);
  P.route_idesc = ptx::umma_idesc_bf16(128, P.route_n, 0, 0);
  CUtensorMap a0, b0;
  if (!make_map(&a0, x, p->T, p->d, 64, 128) || !make_map(&b0, wg, p->E, p->d, 64, P.route_n)) return MOE_ERR_CUDA;
  if (P.route_n <= 64) return launch_tc_impl<TC_ROUTE_S, false, 1>(a0, a0, b0, b0, P, ceil_div(p->T, 128), st);
  return launch_tc_impl<TC_ROUTE, false, 1>(a0, a0, b0, b0, P, ceil_div(p->T, 128), st);
}

// FWD_UP / FWD_DOWN honour GemmCall.row_split in the CTA-pair engine (the others run all rows)
bool tc_splits_rows() { return engine() == ENG_PAIR; }

moe_status tc_gemm(const GemmCall& c, cudaStream_t st) {
  typedef __nv_bfloat16 bf;
  const int64_t T = c.T, R = c.R;
  const int d = c.d, h = c.h, E = c.E;
  // K-major W3 box rows held per CTA (the wide FWD_DOWN tile: 256 per CTA of the pair)
  const uint32_t bw = engine() == ENG_PAIR ? (wide_tile<TC_FWD_DOWN, 2>() ? 256 : 128) : 256;
  TcParams P{};
  P.act = c.act;
  const bool gated = c.act == 0;
  P.x = (const bf*)c.x; P.dy = (const bf*)c.dy;
  P.offs = c.offs; P.eti = c.eti; P.row_slot = c.row_slot; P.topw = c.topw;
  P.a_save = (bf*)c.a_save; P.b_save = (bf*)c.b_save; P.u = (bf*)c.u;
  P.acc_out = c.acc_out; P.dg_part = c.dg_part;
  P.out_mode = c.out_mode; P.out_tok = (bf*)c.out_tok;
  P.out0 = (bf*)c.dw_a; P.out1 = (bf*)c.dw_b;
  P.sched = c.sched;
  P.u_weighted = c.u_weighted; P.dh_skip_u = c.dh_skip_u;
  P.T = (int)T; P.d = d; P.h = h; P.E = E;
  P.dg_parts = tc_dg_parts(h, d);
  P.row_split = c.row_split;
  P.split_half = c.row_split ? c.split_half : 0;
  P.sm_reserve = c.sm_reserve;
  CUtensorMap a0, a1, b0, b1;
  bool ok = true;
  // upper bound on row tiles of height TM over all expert segments
  auto rows_tiles = [&](int64_t n_tiles) { return [=](int TM) { return (ceil_div(R, TM) + E) * n_tiles; }; };
  switch (c.which) {
    case GEMM_FWD_UP: {
      if (R == 0) return MOE_OK;
      ok &= make_map(&a0, c.x, T, d, 64, 1);
      ok &= make_map(&b0, c.w1, (uint64_t)E * h, d, 64, 128);
      ok &= make_map(&b1, gated ? c.w2 : c.w1, (uint64_t)E * h, d, 64, 128);
      if (!ok) return MOE_ERR_CUDA;
      P.n_tiles = gated ? h / 128 : (int)ceil_div(h, TBN);
      return launch_tc<TC_FWD_UP>(a0, a0, b0, b1, P, rows_tiles(P.n_tiles), st);
    }
    case GEMM_FWD_DOWN: {
      if (R == 0) return MOE_OK;
      ok &= make_map(&a0, c.u, R, h, 64, 128);
      ok &= make_map(&b0, c.w3, (uint64_t)E * d, h, 64, bw);
      if (!ok) return MOE_ERR_CUDA;
      P.n_tiles = (int)ceil_div(d, engine() == ENG_PAIR ? tile_n<TC_FWD_DOWN, 2>() : TBN);
      return launch_tc<TC_FWD_DOWN>(a0, a0, b0, b0, P, rows_tiles(P.n_tiles), st);
    }
    case GEMM_BWD_DH: {
      if (R == 0) return MOE_OK;
      // long K (d >= 3072): the 5-stage / 16-column-epilogue variant (CTA-pair engine)
      const bool lk = dh_long_k(d);
      ok &= make_map(&b0, c.w3, (uint64_t)E * d, h, 64, 64);
      if (engine() == ENG_TMA || !MOEB_DH_TMA) {  // dY rows by TMA gather4; cp.async epilogue
        ok &= make_map(&a0, c.dy, T, d, 64, 1);
        a1 = a0;
        b1 = b0;
      } else {  // epilogue TMA boxes: A (a0), B (a1) in, dA, dB, wU (b1) out
        const uint32_t cw = lk ? 16 : 32;
        ok &= make_map_epi(&a0, c.a_save, R, h, cw);
        ok &= make_map_epi(&a1, gated ? c.b_save : c.a_save, R, h, cw);
        ok &= make_map_epi(&b1, c.u, R, h, cw);
      }
      if (!ok) return MOE_ERR_CUDA;
      P.n_tiles = (int)ceil_div(h, TBN);
      if (lk && dh_l5(d)) return launch_tc<TC_BWD_DH_L5>(a0, a1, b0, b1, P, rows_tiles(P.n_tiles), st);
      if (lk) return launch_tc<TC_BWD_DH_LK>(a0, a1, b0, b1, P, rows_tiles(P.n_tiles), st);
      return launch_tc<TC_BWD_DH>(a0, a1, b0, b1, P, rows_tiles(P.n_tiles), st);
    }
    case GEMM_BWD_DX: {
      if (R == 0) return MOE_OK;
      ok &= make_map(&a0, c.a_save, R, h, 64, 128);
      ok &= make_map(&a1, gated ? c.b_save : c.a_save, R, h, 64, 128);
      ok &= make_map(&b0, c.w1, (uint64_t)E * h, d, 64, 64);
      ok &= make_map(&b1, gated ? c.w2 : c.w1, (uint64_t)E * h, d, 64, 64);
      if (!ok) return MOE_ERR_CUDA;
      P.n_tiles = (int)ceil_div(d, engine() == ENG_PAIR ? tile_n<TC_BWD_DX, 2>() : TBN);
      return launch_tc<TC_BWD_DX>(a0, a1, b0, b1, P, rows_tiles(P.n_tiles), st);
    }
    case GEMM_DW3: {
      if (R == 0) {  // no rows at all: every expert's gradient is exactly zero
        MOE_CUDA_CHECK(cudaMemsetAsync(c.dw_a, 0, (size_t)E * d * h * 2, st));
        return MOE_OK;
      }
      ok &= make_map(&a0, c.dy, T, d, 64, 1);
      ok &= make_map(&b0, c.u, R, h, 64, 64);
      if (!ok) return MOE_ERR_CUDA;
      P.n_tiles = (int)ceil_div(h, engine() == ENG_PAIR ? tile_n<TC_DW3, 2>() : TBN);
      P.m_tiles = (int)ceil_div(d, 128);
      P.m_tiles2 = (int)ceil_div(d, 256);
      const int64_t nt = P.n_tiles;
      return launch_tc<TC_DW3>(a0, a0, b0, b0, P, [=](int TM) { return (int64_t)E * ceil_div(d, TM) * nt; }, st);
    }
    case GEMM_DW12: {
      if (R == 0) {
        MOE_CUDA_CHECK(cudaMemsetAsync(c.dw_a, 0, (size_t)E * d * h * 2, st));
        if (gated) MOE_CUDA_CHECK(cudaMemsetAsync(c.dw_b, 0, (size_t)E * d * h * 2, st));
        return MOE_OK;
      }
      const int64_t M = (gated ? 2 : 1) * (int64_t)h;  // [dW1 ; dW2] rows, or dW1 only
      ok &= make_map(&a0, c.a_save, R, h, 64, 64);
      ok &= make_map(&a1, gated ? c.b_save : c.a_save, R, h, 64, 64);
      ok &= make_map(&b0, c.x, T, d, 64, 1);
      if (!ok) return MOE_ERR_CUDA;
      P.n_tiles = (int)ceil_div(d, engine() == ENG_PAIR ? tile_n<TC_DW12, 2>() : TBN);
      P.m_tiles = (int)ceil_div(M, 128);
      P.m_tiles2 = (int)ceil_div(M, 256);
      const int64_t nt = P.n_tiles;
      return launch_tc<TC_DW12>(a0, a1, b0, b0, P, [=](int TM) { return (int64_t)E * ceil_div(M, TM) * nt; }, st);
    }
  }
  return MOE_ERR_INVALID_ARG;
}

}  // namespace moeb
