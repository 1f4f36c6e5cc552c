// die_probe.cu — which die is each SM on?  (B200 = two dies of 74 SMs; HBM is
// interleaved over both, so every SM sees two DRAM latency classes: lines homed
// on its own die and lines homed on the other.)  For every SM in turn: flush
// L2, then one thread on that SM walks 512 cold lines with dependent loads and
// records each latency.  SMs on the same die agree on which lines are near.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o die_probe tools/die_probe.cu && ./die_probe
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void flush(int4* buf, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    buf[i] = make_int4((int)i, 1, 2, 3);
}

__global__ void probe(const int* lines, int nlines, int stride_ints, unsigned target, unsigned* lat, int* seen) {
  if (threadIdx.x != 0) return;
  const unsigned s = smid();
  atomicAdd(&seen[s], 1);
  if (s != target) return;
  int dep = 0;
  for (int i = 0; i < nlines; ++i) {
    const int* p = lines + (size_t)i * stride_ints + dep;
    long long t0 = clock64();
    int v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    dep = v & 0x40000000;  // always 0, but the next address depends on this load
    asm volatile("" ::"r"(dep) : "memory");  // the clock read below waits for the load
    long long t1 = clock64();
    lat[i] = (unsigned)(t1 - t0) + (dep ? 1u : 0u);
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t flush_n = (size_t)512 << 20 >> 4;  // 512 MB of int4
  int4* fbuf;
  cudaMalloc(&fbuf, flush_n * 16);
  const int nlines = 512, stride = 4096 + 32;  // ints: 16 KB + 128 B between probed lines
  int* lines;
  cudaMalloc(&lines, (size_t)nlines * stride * 4 + 4096);
  cudaMemset(lines, 0, (size_t)nlines * stride * 4 + 4096);
  unsigned* lat;
  int* seen;
  cudaMalloc(&lat, nlines * 4);
  cudaMalloc(&seen, 1024 * 4);
  // max smid seen: launch with many CTAs once
  cudaMemset(seen, 0, 1024 * 4);
  probe<<<4 * nsm, 32>>>(lines, 0, stride, 0xffffffffu, lat, seen);
  cudaDeviceSynchronize();
  std::vector<int> hseen(1024);
  cudaMemcpy(hseen.data(), seen, 1024 * 4, cudaMemcpyDeviceToHost);
  int maxsm = 0;
  for (int i = 0; i < 1024; ++i) if (hseen[i]) maxsm = i;
  std::vector<std::vector<unsigned>> L(maxsm + 1);
  for (int s = 0; s <= maxsm; ++s) {
    if (!hseen[s]) continue;
    std::vector<unsigned> best(nlines, 0xffffffffu);
    for (int rep = 0; rep < 3; ++rep) {
      flush<<<4 * nsm, 256>>>(fbuf, flush_n);
      cudaMemset(seen, 0, 1024 * 4);
      probe<<<4 * nsm, 32>>>(lines, nlines, stride, (unsigned)s, lat, seen);
      std::vector<unsigned> h(nlines);
      cudaMemcpy(h.data(), lat, nlines * 4, cudaMemcpyDeviceToHost);
      for (int i = 0; i < nlines; ++i) best[i] = std::min(best[i], h[i]);
    }
    L[s] = best;
  }
  // near/far classification per SM: below that SM's median latency = near
  std::vector<std::vector<int>> bits(maxsm + 1);
  for (int s = 0; s <= maxsm; ++s) {
    if (L[s].empty()) continue;
    std::vector<unsigned> c = L[s];
    std::nth_element(c.begin(), c.begin() + nlines / 2, c.end());
    const unsigned med = c[nlines / 2];
    bits[s].resize(nlines);
    for (int i = 0; i < nlines; ++i) bits[s][i] = L[s][i] < med;
  }
  int ref = -1;
  for (int s = 0; s <= maxsm; ++s) if (!bits[s].empty()) { ref = s; break; }
  printf("nsm %d maxsmid %d\n", nsm, maxsm);
  printf("smid die agree lat_min lat_med lat_max\n");
  int count[2] = {0, 0};
  for (int s = 0; s <= maxsm; ++s) {
    if (bits[s].empty()) continue;
    int agree = 0;
    for (int i = 0; i < nlines; ++i) agree += bits[s][i] == bits[ref][i];
    const int die = agree > nlines / 2 ? 0 : 1;
    count[die]++;
    std::vector<unsigned> c = L[s];
    std::sort(c.begin(), c.end());
    printf("%d %d %d %u %u %u\n", s, die, agree, c[0], c[nlines / 2], c[nlines - 1]);
  }
  printf("die0 %d die1 %d\n", count[0], count[1]);
  return 0;
}
