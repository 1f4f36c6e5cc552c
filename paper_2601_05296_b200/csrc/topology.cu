// topology.cu — which of the B200's two dies each SM sits on.
//
// HBM is interleaved over both dies and each die's L2 also caches lines homed
// on the other die, so two CTAs on different dies that read the same operand
// tile both pull it into their own L2 (ncu: lts__t_sectors_srcunit_ltcfabric).
// The expert GEMMs' tile scheduler (gemm_tc.cu) splits each expert's n-tiles
// between the dies so that concurrent tiles on one die share their operands.
// The SM numbering of the two dies is irregular and floorswept per chip
// (tools/die_probe.cu measured 70 + 78 SMs, interleaved), so it is measured
// here once per device:
//   1. every SM (one CTA each) walks its own slice of cold lines with
//      dependent loads and records each latency (near die ~550 cycles, far
//      ~900);
//   2. after an L2 flush, one reference CTA walks all slices the same way;
//   3. an SM is on the reference's die iff it classifies the lines of its
//      slice near/far the same way the reference does.
// The map only steers the scheduler's work split: a wrong or missing map
// (ambiguous classification, SMs not reached) puts every SM on die 0, which
// is the die-agnostic schedule — results never depend on it.
#include <mutex>
#include <vector>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemm.h"

namespace moeb {

namespace {

constexpr int NL = 64;             // probed lines per SM slice
constexpr int LINE_STRIDE = 4224;  // bytes between probed lines (4 KB + one 128 B line)
constexpr int MAX_SM = 256;

__device__ __forceinline__ unsigned smid_reg() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// latency of a chain of dependent loads over `n` lines starting at `base`
__device__ void walk(const uint8_t* base, int n, unsigned* out) {
  int dep = 0;
  for (int i = 0; i < n; ++i) {
    const int* p = reinterpret_cast<const int*>(base + (size_t)i * LINE_STRIDE) + dep;
    const long long t0 = clock64();
    int v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    dep = v & 0x40000000;  // the buffer is zero: always 0, but the next address waits for this load
    asm volatile("" ::"r"(dep) : "memory");
    const long long t1 = clock64();
    out[i] = (unsigned)(t1 - t0) + (dep ? 1u : 0u);  // dep used: the load chain is live
  }
}

// one CTA per SM (the dynamic smem request keeps a second one off the SM)
__global__ void probe_own(const uint8_t* buf, unsigned* lat, int* owner) {
  if (threadIdx.x != 0) return;
  const unsigned s = smid_reg();
  if (s >= MAX_SM) return;
  if (atomicExch(&owner[s], 1) != 0) return;  // first CTA on this SM only
  walk(buf + (size_t)s * NL * LINE_STRIDE, NL, lat + (size_t)s * NL);
}

// one CTA: 8 warps walk all slices (lane 0 each)
__global__ void probe_ref(const uint8_t* buf, int nslices, unsigned* lat) {
  if ((threadIdx.x & 31) != 0) return;
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int s = w; s < nslices; s += nw) walk(buf + (size_t)s * NL * LINE_STRIDE, NL, lat + (size_t)s * NL);
}

__global__ void flush_l2(int4* buf, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    buf[i] = make_int4((int)i, 0, 0, 0);
}

struct Topo {
  bool done = false;
  uint8_t* d_map = nullptr;  // device [MAX_SM]
  int n[2] = {0, 0};         // SMs per die
  std::vector<int> host;     // die per smid, -1 = not reached
};

std::mutex g_mu;
Topo g_topo[64];

float threshold(std::vector<unsigned> v) {
  std::sort(v.begin(), v.end());
  return 0.5f * (v[v.size() / 10] + v[v.size() * 9 / 10]);
}

void measure(Topo& tp, int nsm) {
  tp.host.assign(MAX_SM, -1);
  const char* env = getenv("MOEBLAZE_DIE");
  if (env && env[0] == '0') return;  // die-agnostic schedule (A/B switch)
  const size_t slice = (size_t)NL * LINE_STRIDE, bytes = slice * MAX_SM + 64;
  const size_t flush_n = ((size_t)384 << 20) / 16;  // 384 MB > 126 MB of L2
  uint8_t* buf = nullptr;
  int4* fl = nullptr;
  unsigned *lat_own = nullptr, *lat_ref = nullptr;
  int* owner = nullptr;
  cudaStream_t st = nullptr;
  bool ok = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaMalloc(&buf, bytes) == cudaSuccess && cudaMalloc(&fl, flush_n * 16) == cudaSuccess &&
       cudaMalloc(&lat_own, MAX_SM * NL * 4) == cudaSuccess && cudaMalloc(&lat_ref, MAX_SM * NL * 4) == cudaSuccess &&
       cudaMalloc(&owner, MAX_SM * 4) == cudaSuccess;
  const int own_smem = 160 * 1024;
  ok = ok && cudaFuncSetAttribute(probe_own, cudaFuncAttributeMaxDynamicSharedMemorySize, own_smem) == cudaSuccess;
  if (ok) {
    cudaMemsetAsync(buf, 0, bytes, st);
    cudaMemsetAsync(owner, 0, MAX_SM * 4, st);
    cudaMemsetAsync(lat_own, 0, MAX_SM * NL * 4, st);
    flush_l2<<<4 * nsm, 256, 0, st>>>(fl, flush_n);
    probe_own<<<nsm, 32, own_smem, st>>>(buf, lat_own, owner);
    flush_l2<<<4 * nsm, 256, 0, st>>>(fl, flush_n);
    probe_ref<<<1, 256, 0, st>>>(buf, MAX_SM, lat_ref);
    ok = cudaStreamSynchronize(st) == cudaSuccess;
  }
  std::vector<unsigned> own(MAX_SM * NL), ref(MAX_SM * NL);
  std::vector<int> reached(MAX_SM);
  if (ok) {
    ok = cudaMemcpy(own.data(), lat_own, own.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
         cudaMemcpy(ref.data(), lat_ref, ref.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
         cudaMemcpy(reached.data(), owner, MAX_SM * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  cudaFree(buf); cudaFree(fl); cudaFree(lat_own); cudaFree(lat_ref); cudaFree(owner);
  if (st) cudaStreamDestroy(st);
  const cudaError_t err = cudaGetLastError();  // a failed probe leaves no sticky error behind
  const bool dbg = getenv("MOEBLAZE_DIE_DEBUG") != nullptr;
  if (dbg) fprintf(stderr, "[moeblaze topology] probe ok=%d last_error=%s\n", (int)ok, cudaGetErrorString(err));
  if (!ok) return;
  const float tref = threshold(ref);
  std::vector<int> die(MAX_SM, -1);
  int n[2] = {0, 0};
  for (int s = 0; s < MAX_SM; ++s) {
    if (!reached[s]) continue;
    std::vector<unsigned> mine(own.begin() + s * NL, own.begin() + (s + 1) * NL);
    const float t = threshold(mine);
    int agree = 0;
    for (int i = 0; i < NL; ++i) agree += (mine[i] < t) == (ref[s * NL + i] < tref);
    if (dbg)
      fprintf(stderr, "[moeblaze topology] sm %d agree %d thr %.0f ref_thr %.0f lat0 %u ref0 %u\n", s, agree, t, tref,
              mine[0], ref[s * NL]);
    if (agree >= NL * 11 / 16) die[s] = 0;
    else if (agree <= NL * 5 / 16) die[s] = 1;
    else return;  // ambiguous: keep the die-agnostic schedule
    n[die[s]]++;
  }
  if (n[0] == 0 || n[1] == 0) return;
  tp.host = die;
  tp.n[0] = n[0];
  tp.n[1] = n[1];
}

}  // namespace

// Die map of the current device (measured once); d_map[smid] in {0, 1}.
// n_sm[0], n_sm[1]: SMs per die (n_sm[1] == 0: one die / no map).
const uint8_t* sm_die_map(int n_sm[2]) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  Topo& tp = g_topo[dev & 63];
  if (!tp.done) {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    measure(tp, nsm);
    std::vector<uint8_t> m(MAX_SM, 0);
    for (int s = 0; s < MAX_SM; ++s) m[s] = tp.host[s] == 1 ? 1 : 0;
    if (cudaMalloc(&tp.d_map, MAX_SM) == cudaSuccess)
      cudaMemcpy(tp.d_map, m.data(), MAX_SM, cudaMemcpyHostToDevice);
    else
      tp.d_map = nullptr;
    tp.done = true;
  }
  n_sm[0] = tp.n[0];
  n_sm[1] = tp.n[1];
  return tp.d_map;
}

const std::vector<int>& sm_die_host() {
  int n[2];
  sm_die_map(n);
  int dev = 0;
  cudaGetDevice(&dev);
  return g_topo[dev & 63].host;
}

}  // namespace moeb

extern "C" moe_status moe_sm_topology(int32_t* die_of_sm, int32_t max_sm, int32_t* n_per_die) {
  if (!die_of_sm || !n_per_die || max_sm < 0) return MOE_ERR_INVALID_ARG;
  int n[2];
  if (!moeb::sm_die_map(n)) return MOE_ERR_CUDA;
  const std::vector<int>& h = moeb::sm_die_host();
  for (int s = 0; s < max_sm; ++s) die_of_sm[s] = s < (int)h.size() ? h[s] : -1;
  n_per_die[0] = n[0];
  n_per_die[1] = n[1];
  return MOE_OK;
}
