// L2 -> SM read throughput of this B200: every CTA streams an L2-resident buffer
// (16-byte loads, all SMs, grid = SMs x 4), timed with CUDA events.  The expert GEMMs
// pull their operands from L2 at 64 B per SM-cycle at full tensor rate (256 x 256 pair
// tiles, BK = 64): this is the ceiling that number runs into.
#include <cstdio>
#include <cstdint>
__global__ void l2_read(const uint4* __restrict__ p, size_t n16, int iters, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
      uint4 v;
      asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (size_t mb : {8, 24, 48, 96}) {
    size_t bytes = mb << 20, n16 = bytes / 16;
    uint4 *p, *sink;
    cudaMalloc(&p, bytes);
    cudaMalloc(&sink, 16);
    cudaMemset(p, 1, bytes);
    int iters = (int)(4096 / mb);
    l2_read<<<sms * 4, 512>>>(p, n16, 2, sink);  // warm: lines resident in L2
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    l2_read<<<sms * 4, 512>>>(p, n16, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("buffer %3zu MB: %.2f TB/s L2->SM reads (%d passes, %.3f ms) %s\n", mb,
           (double)bytes * iters / (ms * 1e-3) / 1e12, iters, ms, cudaGetErrorString(cudaGetLastError()));
    cudaFree(p);
    cudaFree(sink);
  }
  return 0;
}
