// Where does dynamic shared memory start?  (alignment of the extern __shared__ base for a
// cluster launch with a large dynamic allocation, as the expert GEMMs use)
#include <cstdio>
__global__ void __cluster_dims__(2, 1, 1) probe(unsigned* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned)__cvta_generic_to_shared(sm);
}
int main() {
  unsigned* d;
  cudaMalloc(&d, 64 * 4);
  for (int bytes : {1024, 100000, 200000, 230000}) {
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    probe<<<4, 128, bytes>>>(d);
    unsigned h[4];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("dyn smem %d: base offsets %u %u %u %u (mod 1024: %u)  err=%s\n", bytes, h[0], h[1], h[2], h[3], h[0] % 1024,
           cudaGetErrorString(cudaGetLastError()));
  }
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  printf("max dyn smem per block (opt-in): %d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrReservedSharedMemoryPerBlock, 0);
  printf("reserved smem per block: %d\n", v);
  return 0;
}
