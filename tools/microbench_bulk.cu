// Microbenchmark: global->shared gather throughput on B200 for the access patterns the
// decode path uses (contiguous runs of 256-byte K rows at random offsets).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_bulk.cu && /tmp/mb
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
          smem_u32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void bulk_cl(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

__device__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
  return x;
}

// mode 0: bulk (.shared::cta) runs of RUN rows; mode 1: bulk .shared::cluster; mode 2: LDG.128 -> STS
template <int MODE>
__global__ void gather(const uint8_t* __restrict__ src, size_t nrows, int run, int chunks, int stages,
                       unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[8];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int chunk_bytes = 64 * 256;
  unsigned long long t0 = clock64();
  float acc = 0.f;
  for (int c = 0; c < chunks + stages; ++c) {
    if (c < chunks) {
      const int st = c % stages;
      uint8_t* dst = sm + st * chunk_bytes;
      if (MODE < 2) {
        if (tid == 0) {
          expect(&bar[st], chunk_bytes);
          for (int r0 = 0; r0 < 64; r0 += run) {
            const size_t row = (size_t)(hash(blockIdx.x * 100003u + c * 977u + r0) % (uint32_t)(nrows - 64));
            if (MODE == 0) bulk(dst + r0 * 256, src + row * 256, run * 256, &bar[st]);
            else bulk_cl(dst + r0 * 256, src + row * 256, run * 256, &bar[st]);
          }
        }
      } else {
        for (int i = tid; i < 64 * 16; i += blockDim.x) {
          const int r0 = (i >> 4) / run * run, rr = (i >> 4) % run;
          const size_t row = (size_t)(hash(blockIdx.x * 100003u + c * 977u + r0) % (uint32_t)(nrows - 64)) + rr;
          *reinterpret_cast<uint4*>(dst + (i >> 4) * 256 + (i & 15) * 16) =
              *reinterpret_cast<const uint4*>(src + row * 256 + (i & 15) * 16);
        }
      }
    }
    const int cc = c - (stages - 1);
    if (cc >= 0 && cc < chunks) {
      const int st = cc % stages;
      if (MODE < 2) wait(&bar[st], (cc / stages) & 1);
      __syncthreads();
      acc += reinterpret_cast<float*>(sm + st * chunk_bytes)[tid];
      __syncthreads();
    }
  }
  unsigned long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[0] = 0;
}

int main() {
  const size_t bytes = (size_t)512 << 20;
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8 * 4);
  const size_t nrows = bytes / 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode) {
    for (int run : {1, 8, 64}) {
      for (int stages : {2, 4}) {
        const int chunks = 64;
        const int smem = stages * 64 * 256;
        void (*k)(const uint8_t*, size_t, int, int, int, unsigned long long*) =
            mode == 0 ? gather<0> : mode == 1 ? gather<1> : gather<2>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k<<<148, 256, smem>>>(src, nrows, run, chunks, stages, out);
        cudaEventRecord(a);
        k<<<148, 256, smem>>>(src, nrows, run, chunks, stages, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double gb = 148.0 * chunks * 64 * 256 / 1e9;
        printf("mode %d (%s) run %2d stages %d: %8.1f us  %7.1f GB/s  (%s)\n", mode,
               mode == 0 ? "bulk cta" : mode == 1 ? "bulk cluster" : "ldg->sts", run, stages, ms * 1e3,
               gb / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
