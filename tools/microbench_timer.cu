// %globaltimer resolution on the GPU: one thread reads it back to back and records the
// distinct increments it sees (with clock64 alongside).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbt tools/microbench_timer.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long* out, int n) {
  unsigned long long prev, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  long long c0 = clock64();
  int m = 0;
  for (int i = 0; i < 2000000 && m < n; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) {
      out[2 * m] = t - prev;
      out[2 * m + 1] = clock64() - c0;
      prev = t;
      ++m;
    }
  }
}
int main() {
  unsigned long long* d; const int n = 64;
  cudaMalloc(&d, 2 * n * 8); cudaMemset(d, 0, 2 * n * 8);
  k<<<1, 1>>>(d, n); cudaDeviceSynchronize();
  unsigned long long h[2 * n]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("globaltimer increments (ns) and clock64 at each change:\n");
  for (int i = 0; i < n; ++i) printf("%llu@%llu ", h[2 * i], h[2 * i + 1]);
  printf("\n");
  return 0;
}
