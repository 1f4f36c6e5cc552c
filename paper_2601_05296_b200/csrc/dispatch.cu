// dispatch.cu — K2: buffer-free dispatch construction (§4.2).
//
// Same outputs as the paper's 3-step build (dense map -> expert lengths ->
// location map + scatter), reached with O(T*k) traffic instead of the
// O(T*E) dense_token_map (reading #7), atomic-free and deterministic:
//
//  view ids as the flat array f = t*k + j (length R = T*k), cut into tiles of
//  DT_TILE entries.
//  launch 1 (histogram): per tile, per-warp counts via __match_any_sync (each
//    distinct expert in a 32-entry chunk is counted once, by its lowest lane),
//    summed over warps -> tile_counts[tile][e].  Optional routing validation.
//  launch 2 (scan + scatter): every CTA derives, for its tile, the global base
//    of every expert: offs[e] + sum_{tile'<tile} tile_counts[tile'][e]
//    (offs = exclusive scan of the per-expert totals, "CTA-local
//    exclusive scan ... add with the expert's pre-computed global offsets"),
//    then walks its tile in flat order in 256-entry rounds: rank inside the
//    warp (popc of lower peer lanes) + exclusive scan of the warp counts of
//    the round gives every entry's final position `pos` with no atomics.
//    tim[f] = pos (coalesced), eti[pos] = t, row_slot[pos] = f.
//  Ascending f inside an expert => ascending token id: the stable order
//  (reading #5) that the sort-based construction also produces.
#include "common.cuh"

namespace moeb {

constexpr int DT_THREADS = 256;
constexpr int DT_WARPS = DT_THREADS / 32;

int dispatch_tile_entries(int64_t R) {
  // small tiles: many CTAs walk their tiles in a few 256-entry rounds (the walk is
  // latency-bound: 4096-entry tiles gave Mixtral-like R = 16384 only 4 CTAs of 16 rounds);
  // keep the number of tiles <= 256 so the per-CTA scan over tiles stays short
  int64_t t = 512;
  while (ceil_div(R, t) > 256) t *= 2;
  return (int)t;
}

// launch 1: tile_counts[tile*E + e]; status word validation
__global__ void __launch_bounds__(DT_THREADS)
dispatch_hist_kernel(const int32_t* __restrict__ ids, int64_t R, int k, int E, int tile, int check, int sparse,
                     int32_t* __restrict__ tile_counts, int32_t* __restrict__ status) {
  extern __shared__ int32_t hs[];  // [DT_WARPS][E]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < DT_WARPS * E; i += DT_THREADS) hs[i] = 0;
  __syncthreads();
  const int64_t f0 = (int64_t)blockIdx.x * tile;
  const int64_t f1 = min64(f0 + tile, R);
  for (int64_t base = f0 + warp * 32; base < f1; base += DT_THREADS) {
    const int64_t f = base + lane;
    const bool valid = f < f1;
    int e = valid ? ids[f] : -1;
    if (check && valid && !(sparse && e == -1)) {  // sparse slots: -1 = empty slot, not an error
      bool bad = (e < 0 || e >= E);
      // per-token uniqueness: compare with the other slots of the same token
      const int64_t t = f / k;
      for (int j = 0; j < k; ++j) {
        int64_t g = t * k + j;
        if (g != f && ids[g] == e) bad = true;
      }
      if (bad) { *status = MOE_ERR_BAD_ROUTING; e = -1; }
    }
    if (e < 0 || e >= E) e = -1;
    unsigned peers = __match_any_sync(0xffffffffu, e);
    if (e >= 0 && lane == __ffs(peers) - 1) hs[warp * E + e] += __popc(peers);
  }
  __syncthreads();
  for (int e = tid; e < E; e += DT_THREADS) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < DT_WARPS; ++w) s += hs[w * E + e];
    tile_counts[(int64_t)blockIdx.x * E + e] = s;
  }
}

// launch 2: scan over tiles/experts + position computation + scatter
__global__ void __launch_bounds__(DT_THREADS)
dispatch_scatter_kernel(const int32_t* __restrict__ ids, int64_t R, int k, int E, int tile, int ntiles,
                        const int32_t* __restrict__ tile_counts, int32_t* __restrict__ counts,
                        int32_t* __restrict__ offs, int32_t* __restrict__ eti, int32_t* __restrict__ tim,
                        int32_t* __restrict__ row_slot, int64_t rows_decl, int32_t* __restrict__ status) {
  extern __shared__ int32_t ss[];
  int32_t* base = ss;                 // [E]   running global base of each expert for this tile
  int32_t* wc = base + E;             // [DT_WARPS][E] warp counts of the current round
  int32_t* tot = wc + DT_WARPS * E;   // [E]   totals (for the scan)
  int32_t* ptot = tot + E;            // [parts][E] partial totals / prefixes over slices of tiles
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int my = blockIdx.x;
  // per expert: total over all tiles and prefix over tiles < my; the tiles are split into
  // `parts` slices so all threads share the walk (E <= 256: parts * E <= DT_THREADS)
  const int parts = max(1, DT_THREADS / E);
  int32_t* ppre = ptot + parts * E;
  for (int i = tid; i < parts * E; i += DT_THREADS) {
    const int e = i % E, part = i / E;
    const int q0 = (int)((int64_t)ntiles * part / parts), q1 = (int)((int64_t)ntiles * (part + 1) / parts);
    int total = 0, pre = 0;
    for (int q = q0; q < q1; ++q) {
      int c = tile_counts[(int64_t)q * E + e];
      if (q < my) pre += c;
      total += c;
    }
    ptot[i] = total;
    ppre[i] = pre;
  }
  __syncthreads();
  for (int e = tid; e < E; e += DT_THREADS) {
    int total = 0, pre = 0;
    for (int part = 0; part < parts; ++part) {  // fixed order: integer sums, any order is exact
      total += ptot[part * E + e];
      pre += ppre[part * E + e];
    }
    tot[e] = total;
    base[e] = pre;
  }
  __syncthreads();
  // exclusive scan of totals over experts (E <= 256): warp 0, serial chunks
  if (warp == 0) {
    int carry = 0;
    for (int c0 = 0; c0 < E; c0 += 32) {
      int e = c0 + lane;
      int v = e < E ? tot[e] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
      }
      if (e < E) {
        int excl = carry + incl - v;
        if (my == 0) { counts[e] = v; offs[e] = excl; }
        base[e] += excl;
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (my == 0 && lane == 0) {
      offs[E] = carry;
      if (status && rows_decl > 0 && carry > rows_decl) *status = MOE_ERR_BAD_ROUTING;  // more rows than declared
    }
  }
  __syncthreads();
  const int64_t f0 = (int64_t)my * tile;
  const int64_t f1 = min64(f0 + tile, R);
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t rb = f0; rb < f1; rb += DT_THREADS) {
    for (int i = tid; i < DT_WARPS * E; i += DT_THREADS) wc[i] = 0;
    __syncthreads();
    const int64_t f = rb + tid;
    const bool valid = f < f1;
    int e = valid ? ids[f] : -1;
    if (e < 0 || e >= E) e = -1;
    unsigned peers = __match_any_sync(0xffffffffu, e);
    int rank = __popc(peers & lt);
    if (e >= 0 && lane == __ffs(peers) - 1) wc[warp * E + e] = __popc(peers);
    __syncthreads();
    // exclusive scan over warps per expert, add the running base, advance it
    for (int x = tid; x < E; x += DT_THREADS) {
      int run = base[x];
#pragma unroll
      for (int w = 0; w < DT_WARPS; ++w) {
        int c = wc[w * E + x];
        wc[w * E + x] = run;
        run += c;
      }
      base[x] = run;
    }
    __syncthreads();
    if (e >= 0) {
      int pos = wc[warp * E + e] + rank;
      tim[f] = pos;
      eti[pos] = (int32_t)(f / k);
      if (row_slot) row_slot[pos] = (int32_t)f;
    } else if (valid) {
      tim[f] = -1;  // empty (sparse) or invalid slot: no routed row
    }
    __syncthreads();
  }
}

moe_status launch_dispatch(const moe_problem* p, const int32_t* ids, const moe_dispatch* out, int32_t* ws_tile_counts,
                           int32_t* status, cudaStream_t st) {
  const int64_t R = p->T * p->k;
  const int E = p->E;
  if (R == 0) {
    MOE_CUDA_CHECK(cudaMemsetAsync(out->expert_counts, 0, sizeof(int32_t) * E, st));
    MOE_CUDA_CHECK(cudaMemsetAsync(out->expert_offsets, 0, sizeof(int32_t) * (E + 1), st));
    return MOE_OK;
  }
  const int tile = dispatch_tile_entries(R);
  const int ntiles = (int)ceil_div(R, tile);
  size_t sm1 = sizeof(int32_t) * DT_WARPS * E;
  MOE_LAUNCH(dispatch_hist_kernel, ntiles, DT_THREADS, sm1, st, ids, R, p->k, E, tile, p->check_routing,
             p->rows > 0 ? 1 : 0, ws_tile_counts, status);
  const int parts = std::max(1, DT_THREADS / E);
  size_t sm2 = sizeof(int32_t) * (E + DT_WARPS * E + E + 2 * parts * E);
  MOE_LAUNCH(dispatch_scatter_kernel, ntiles, DT_THREADS, sm2, st, ids, R, p->k, E, tile, ntiles, ws_tile_counts,
             out->expert_counts, out->expert_offsets, out->expert_token_indices, out->token_index_map, out->row_slot,
             p->rows, p->check_routing ? status : nullptr);
  MOE_CUDA_CHECK(cudaGetLastError());
  return MOE_OK;
}

// row_split[e] = offs[e] + #{r in segment e : eti[r] < t_ready}: lower bound of t_ready in the
// segment (eti ascending inside an expert); one thread per expert
__global__ void row_split_kernel(const int32_t* __restrict__ offs, const int32_t* __restrict__ eti, int E,
                                 int64_t t_ready, int32_t* __restrict__ split) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int lo = offs[e], hi = offs[e + 1];
  while (lo < hi) {
    const int mid = lo + ((hi - lo) >> 1);
    if ((int64_t)eti[mid] < t_ready) lo = mid + 1;
    else hi = mid;
  }
  split[e] = lo;
}

moe_status launch_row_split(const int32_t* offs, const int32_t* eti, int E, int64_t t_ready, int32_t* split,
                            cudaStream_t st) {
  MOE_LAUNCH(row_split_kernel, (unsigned)ceil_div(E, 128), 128, 0, st, offs, eti, E, t_ready, split);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

size_t dispatch_ws_bytes(const moe_problem* p) {
  const int64_t R = p->T * p->k;
  const int64_t ntiles = R ? ceil_div(R, dispatch_tile_entries(R)) : 0;
  return 256 + sizeof(int32_t) * (size_t)ntiles * p->E;  // [status word | pad][tile_counts]
}

}  // namespace moeb
