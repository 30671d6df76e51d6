// Latency of the hand-off primitives on sm_100a (one thread, dependent chains, clock64):
//   ld.global.cg, ld.relaxed.gpu, ld.acquire.gpu, fence.acq_rel.gpu (idle and after
//   outstanding stores), atom.add.acq_rel.gpu, red.release.gpu
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbs tools/microbench_sync.cu && /tmp/mbs
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int ld_cg(const int* p) { int r; asm volatile("ld.global.cg.b32 %0, [%1];" : "=r"(r) : "l"(p) : "memory"); return r; }
__device__ __forceinline__ int ld_rlx(const int* p) { int r; asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(p) : "memory"); return r; }
__device__ __forceinline__ int ld_acq(const int* p) { int r; asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(p) : "memory"); return r; }

__global__ void k(int* buf, long long* out) {
  if (threadIdx.x != 0) return;
  const int N = 32;
  int idx = 0;
  long long t0, t1;
  // chains: buf[i] = i + 1 (pointer chase within 32 ints spread over lines)
  t0 = clock64(); for (int i = 0; i < N; ++i) idx = ld_cg(buf + idx * 32); t1 = clock64(); out[0] = (t1 - t0) / N;
  idx = 0; t0 = clock64(); for (int i = 0; i < N; ++i) idx = ld_rlx(buf + idx * 32); t1 = clock64(); out[1] = (t1 - t0) / N;
  idx = 0; t0 = clock64(); for (int i = 0; i < N; ++i) idx = ld_acq(buf + idx * 32); t1 = clock64(); out[2] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) asm volatile("fence.acq_rel.gpu;" ::: "memory"); t1 = clock64(); out[3] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { buf[4096 + i * 32] = i; asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
  t1 = clock64(); out[4] = (t1 - t0) / N;
  int r = 0;
  t0 = clock64(); for (int i = 0; i < N; ++i) { asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(r) : "l"(buf + 8192 + (r & 0))); } t1 = clock64(); out[5] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(buf + 8192 + 32) : "memory"); t1 = clock64(); out[6] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) { asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], 1;" : "=r"(r) : "l"(buf + 8192 + 64 + (r & 0))); } t1 = clock64(); out[7] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) __threadfence(); t1 = clock64(); out[8] = (t1 - t0) / N;
  out[9] = idx + r;
}

int main() {
  int* buf; long long* out;
  cudaMalloc(&buf, 1 << 20); cudaMalloc(&out, 16 * 8);
  int h[32 * 33];
  for (int i = 0; i < 32; ++i) h[i * 32] = (i + 1) % 32;
  cudaMemcpy(buf, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    k<<<1, 32>>>(buf, out);
    long long o[16]; cudaMemcpy(o, out, 16 * 8, cudaMemcpyDeviceToHost);
    printf("cycles: ld.cg %lld  ld.relaxed.gpu %lld  ld.acquire.gpu %lld  fence.acq_rel(idle) %lld  st+fence %lld  "
           "atom.acq_rel %lld  red.release %lld  atom.relaxed %lld  threadfence %lld\n",
           o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7], o[8]);
  }
  return 0;
}
