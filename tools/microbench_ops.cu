// Microbenchmark: cycle cost of small-CTA building blocks on sm_100a (256 threads).
#include <cuda_runtime.h>
#include <stdio.h>
#include <math.h>
__device__ double sink_d; __device__ float sink_f;
__global__ void k(const double* gd, unsigned long long* out) {
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  long long t[16]; int i = 0;
  double x = gd[tid] + 1.0;
  __syncthreads();
  t[i++] = clock64();
  for (int r = 0; r < 10; ++r) __syncthreads();
  t[i++] = clock64();                                   // 10 syncthreads
  double v = x;
  for (int r = 0; r < 10; ++r) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads(); if (lane == 0) red[w] = v; __syncthreads();
    double s = 0; for (int j = 0; j < 8; ++j) s += red[j]; v = s * 1e-3; __syncthreads();
  }
  t[i++] = clock64();                                   // 10 block reductions (double)
  double e = x;
  for (int r = 0; r < 10; ++r) e = exp(e * 1e-3);
  t[i++] = clock64();                                   // 10 dependent exp(double)
  double l = x;
  for (int r = 0; r < 10; ++r) l = log(l + 2.0);
  t[i++] = clock64();                                   // 10 dependent log(double)
  float ef = (float)x;
  for (int r = 0; r < 10; ++r) ef = expf(ef * 1e-3f);
  t[i++] = clock64();                                   // 10 dependent expf
  double dv = x;
  for (int r = 0; r < 10; ++r) dv = 1.0 / (dv + 3.0);
  t[i++] = clock64();                                   // 10 dependent double divisions
  double ld = 0;
  for (int r = 0; r < 10; ++r) ld += __ldcg(gd + ((tid + r * 977 + (int)ld) & 4095));
  t[i++] = clock64();                                   // 10 dependent L2 loads
  sink_d = v + e + l + dv + ld; sink_f = ef;
  if (tid == 0) for (int j = 0; j < i; ++j) out[j] = t[j];
}
int main() {
  double* gd; cudaMalloc(&gd, 4096 * 8); cudaMemset(gd, 0, 4096 * 8);
  unsigned long long* o; cudaMalloc(&o, 16 * 8);
  k<<<1, 256>>>(gd, o); k<<<1, 256>>>(gd, o); cudaDeviceSynchronize();
  unsigned long long h[16]; cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[] = {"10x __syncthreads", "10x block reduce (double)", "10x exp(double)", "10x log(double)",
                      "10x expf", "10x double div", "10x dependent L2 load"};
  for (int j = 0; j < 7; ++j) printf("%-28s %8llu cycles\n", nm[j], h[j + 1] - h[j]);
}
