// Throughput of the fp64 ops the S1 scoring issues on sm_100a: F2F.F64.F32 conversions and
// DFMA, per SM per clock (one CTA per SM, 16 warps, independent chains).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbfp64 tools/microbench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_cvt(const float* in, double* out, long long* cyc, int iters) {
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = in[threadIdx.x + i];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc[i] += (double)f[i];  // F2F + DADD
      f[i] = __int_as_float(__float_as_int(f[i]) ^ 1);
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_dfma(const float* in, double* out, long long* cyc, int iters) {
  double a[8], b = in[threadIdx.x] + 1.0;
  for (int i = 0; i < 8; ++i) a[i] = in[threadIdx.x + i];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, 0.5);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_ffma(const float* in, double* out, long long* cyc, int iters) {
  float a[8], b = in[threadIdx.x] + 1.0f;
  for (int i = 0; i < 8; ++i) a[i] = in[threadIdx.x + i];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, 0.5f);
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* in; double* out; long long* cyc;
  cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, sms * 1024 * 8); cudaMalloc(&cyc, sms * 8);
  const int iters = 4096;
  for (int threads : {128, 512, 1024}) {
    long long c;
    k_cvt<<<sms, threads>>>(in, out, cyc, iters); cudaDeviceSynchronize();
    k_cvt<<<sms, threads>>>(in, out, cyc, iters); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d  F2F.F64.F32+DADD: %.2f ops/clk/SM\n", threads, (double)threads * 8 * iters / c);
    k_dfma<<<sms, threads>>>(in, out, cyc, iters); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d  DFMA:             %.2f ops/clk/SM\n", threads, (double)threads * 8 * iters / c);
    k_ffma<<<sms, threads>>>(in, out, cyc, iters); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d  FFMA:             %.2f ops/clk/SM\n", threads, (double)threads * 8 * iters / c);
  }
  return 0;
}
