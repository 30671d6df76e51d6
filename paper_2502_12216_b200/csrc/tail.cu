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

// Per-head loading ablation (the GQA union loads each KV
// token once, "up to 1.65x faster than per-head loading").  One CTA per (unit, head):
// the head's own selected clusters order[0..J) (non-empty), in rank order, as a work
// list (rows, token prefix) for the attention kernel run with G = 1 per (unit, head).
__global__ void __launch_bounds__(256) head_lists_kernel(const int* __restrict__ order, const int* __restrict__ J,
                                                         const int* __restrict__ offsets, int C, int G,
                                                         int* __restrict__ hl, int* __restrict__ hp) {
  __shared__ unsigned long long ws[8];
  const int ug = blockIdx.x, u = ug / G, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Jg = J[ug];
  const int* ord = order + (size_t)ug * C;
  const int* off = offsets + (size_t)u * (C + 1);
  int* rl = hl + (size_t)ug * C;
  int* rp = hp + (size_t)ug * (C + 1);
  int seg_carry = 0, tok_carry = 0;
  for (int r0 = 0; r0 < Jg; r0 += 256) {
    const int r = r0 + tid;
    int o0 = 0, sz = 0;
    if (r < Jg) {
      const int cid = ord[r];
      o0 = off[cid];
      sz = off[cid + 1] - o0;
    }
    // packed (tokens << 20 | segments) block scan of this chunk of 256 ranks
    const unsigned long long v = sz > 0 ? (((unsigned long long)sz << 20) | 1ull) : 0ull;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    unsigned long long wb = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      wb += w < warp ? ws[w] : 0ull;
      tot += ws[w];
    }
    const unsigned long long ex = wb + incl - v;
    if (sz > 0) {
      const int seg = seg_carry + (int)(ex & 0xFFFFFull);
      rl[seg] = o0;
      rp[seg] = tok_carry + (int)(ex >> 20);
    }
    seg_carry += (int)(tot & 0xFFFFFull);
    tok_carry += (int)(tot >> 20);
    __syncthreads();  // ws reuse
  }
  for (int k = seg_carry + tid; k <= C; k += blockDim.x) {
    rp[k] = tok_carry;
    if (k < C) rl[k] = 0;
  }
}

cudaError_t launch_head_lists(const tactic_index_s* x, cudaStream_t s) {
  head_lists_kernel<<<x->units * x->G, 256, 0, s>>>(x->order, x->J, x->offsets, x->C, x->G, x->head_list,
                                                    x->head_prefix);
  return cudaGetLastError();
}

}  // namespace tactic
