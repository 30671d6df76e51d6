// tail.cu -- multi-step generation.
//
// P:112 (§1): Tactic "performs full attention on newly generated tokens" and "updates
// the clustering every ... 2048 ... tokens".  Tokens generated after the index build are
// appended to a per-unit dense tail (rows n .. n + tail_len - 1 of the unit, stored in
// [units][tail_cap][128] buffers with the same 16-byte-chunk row swizzle as the index
// layout, so the attention kernel streams them as one more run after the unit's work
// list).  Re-clustering (B1-B5 over clustered + tail tokens) is the caller's policy
// (paper_2502_12216_b200.tactic.DecodeSession).
//
// assign_kernel: SPEC assign_token: the nearest centroid of a new key,
// argmin_j |k - c_j|^2 (squared Euclidean, reading 4), ties to the lowest id (reading 7),
// float64 distances from the bf16 key and the float32 centroids.
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace tactic {

// rows [tail_len, tail_len + t) of every unit's tail; one warp per row, 16-byte chunks
__global__ void tail_append_kernel(const __nv_bfloat16* __restrict__ k_new, const __nv_bfloat16* __restrict__ v_new,
                                   int t, int n, int tail_len, int tail_cap, __nv_bfloat16* __restrict__ Kt,
                                   __nv_bfloat16* __restrict__ Vt) {
  const int u = blockIdx.y;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int c = threadIdx.x & 15, half = (threadIdx.x >> 4) & 1;
  if (i >= t) return;
  const int r = tail_len + i;  // tail position; layout row n + r (its swizzle phase)
  const uint4* src = reinterpret_cast<const uint4*>((half ? v_new : k_new) + ((size_t)u * t + i) * 128);
  uint4* dst = reinterpret_cast<uint4*>((half ? Vt : Kt) + ((size_t)u * tail_cap + r) * 128);
  dst[swz_chunk(c, n + r)] = src[c];
}

cudaError_t launch_tail_append(const __nv_bfloat16* k_new, const __nv_bfloat16* v_new, int t, tactic_index_s* x,
                               cudaStream_t s) {
  const int rows_per_cta = 8;
  dim3 grid((t + rows_per_cta - 1) / rows_per_cta, x->units);
  tail_append_kernel<<<grid, 32 * rows_per_cta, 0, s>>>(k_new, v_new, t, x->n, x->tail_len, x->tail_cap, x->Kt,
                                                      x->Vt);
  return cudaGetLastError();
}

// one CTA per (unit, new key): the key in fp64 smem, each thread scans clusters j = tid,
// tid + 256, ... with direct (k - c)^2 sums, then a (distance, id) block argmin
__global__ void __launch_bounds__(256) assign_kernel(const __nv_bfloat16* __restrict__ k, int t,
                                                     const float* __restrict__ cent, int C,
                                                     int* __restrict__ assign) {
  __shared__ double kd[128];
  __shared__ double bd[8];
  __shared__ int bj[8];
  const int u = blockIdx.y, i = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 128) kd[tid] = (double)__bfloat162float(k[((size_t)u * t + i) * 128 + tid]);
  __syncthreads();
  double best = INFINITY;
  int bestj = 0x7fffffff;
  for (int j = tid; j < C; j += blockDim.x) {
    const float4* c4 = reinterpret_cast<const float4*>(cent + ((size_t)u * C + j) * 128);
    double d = 0.0;
#pragma unroll 8
    for (int e = 0; e < 32; ++e) {
      const float4 c = __ldg(c4 + e);
      const double d0 = kd[4 * e] - (double)c.x, d1 = kd[4 * e + 1] - (double)c.y;
      const double d2 = kd[4 * e + 2] - (double)c.z, d3 = kd[4 * e + 3] - (double)c.w;
      d = fma(d0, d0, d);
      d = fma(d1, d1, d);
      d = fma(d2, d2, d);
      d = fma(d3, d3, d);
    }
    if (d < best) {  // j ascending per thread: strict < keeps the lowest id
      best = d;
      bestj = j;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oj = __shfl_xor_sync(0xffffffffu, bestj, o);
    if (ob < best || (ob == best && oj < bestj)) {
      best = ob;
      bestj = oj;
    }
  }
  if (lane == 0) {
    bd[warp] = best;
    bj[warp] = bestj;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (bd[w] < best || (bd[w] == best && bj[w] < bestj)) {
        best = bd[w];
        bestj = bj[w];
      }
    assign[(size_t)u * t + i] = bestj;
  }
}

cudaError_t launch_assign(const __nv_bfloat16* k, int t, const tactic_index_s* x, int* assign, cudaStream_t s) {
  dim3 grid(t, x->units);
  assign_kernel<<<grid, 256, 0, s>>>(k, t, x->cent, x->C, assign);
  return cudaGetLastError();
}

__global__ void unit_prefix_fill_kernel(long long* up, int units, long long per_unit) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v <= units) up[v] = (long long)v * per_unit;
}

cudaError_t launch_unit_prefix_fill(long long* up, int units, long long per_unit, cudaStream_t s) {
  unit_prefix_fill_kernel<<<(units + 256) / 256, 256, 0, s>>>(up, units, per_unit);
  return cudaGetLastError();
}

}  // namespace tactic
