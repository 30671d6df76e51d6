// kmeans.cu -- index build B1-B6 (§4.2; max 10 iterations P:402).
//
//  B1 init        c_j = K[init_j] (init from the caller or the SplitMix64 sampler).
//  B2 assign      a(i) = argmin_j |k_i - c_j|^2 = argmin_j (|c_j|^2 - 2 k_i.c_j), ties ->
//                 lowest j.  tcgen05 tensor-core GEMM: 128 keys (bf16, exact) x 128
//                 centroids per tile, centroids split as c ~ hi + lo (two bf16 MMAs into
//                 one fp32 TMEM accumulator), operands in SWIZZLE_128B K-major smem,
//                 centroid tiles streamed by 1-D bulk copies of a pre-swizzled image,
//                 double-buffered TMEM accumulators, argmin fused into the epilogue
//                 (the n x C distance matrix never exists).
//  B3 update      per-block histograms -> per-cluster scan -> stable scatter (cluster
//                 major, ascending token id) -> warp-per-cluster segmented sum in fp64 in
//                 member order (deterministic) -> float32 means (empty: keep), hi/lo
//                 split, |c|^2 of the split value, new tile image.
//  B4 converge    changed-assignment count; a unit stops once an iteration t >= 2
//                 leaves its assignment unchanged (device flag, later launches no-op).
//  B5 relayout    K/V rows gathered into cluster-contiguous, chunk-swizzled layout.
//  B6 finalize    p >= 1 work list (every non-empty cluster), iterations used.
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace tactic {

constexpr int KM_BLK = 1024;         // tokens per histogram / scatter block
constexpr int TC_STAGE = 65536;      // one centroid tile image: hi 32 KB | lo 32 KB
constexpr int TC_A = 32768;          // 128 keys x 128 dims bf16
constexpr int TC_KA = 2;             // A tiles (128 keys each) per CTA: every centroid tile
                                     // streamed from L2 feeds 256 keys (halves B traffic)
constexpr int TC_HALF = 32768;       // the hi or the lo half of a tile image
constexpr int TC_BST = 3;            // centroid half-tile stages
constexpr size_t TC_SMEM = 1024 + 2 * TC_KA * (size_t)TC_A + TC_BST * (size_t)TC_HALF + 256;

__device__ __forceinline__ const __nv_bfloat16* krow(const __nv_bfloat16* K, long long sb, long long sh,
                                                     long long sn, int Hkv, int u, int i) {
  const int b = u / Hkv, h = u % Hkv;
  return K + (long long)b * sb + (long long)h * sh + (long long)i * sn;
}

// Store centroid j of unit u (lane holds dims 4*lane .. 4*lane+3): float32 value, the
// (hi, lo) bf16 split in the pre-swizzled tile image, and |hi + lo|^2.
__device__ void store_centroid(const KmArgs& a, int u, int j, float4 c) {
  const int lane = threadIdx.x & 31;
  *reinterpret_cast<float4*>(a.cent + ((size_t)u * a.C + j) * 128 + lane * 4) = c;
  const float cv[4] = {c.x, c.y, c.z, c.w};
  __nv_bfloat16 hi[4], lo[4];
  float nrm = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    hi[i] = __float2bfloat16_rn(cv[i]);
    lo[i] = __float2bfloat16_rn(cv[i] - __bfloat162float(hi[i]));
    const float v = __bfloat162float(hi[i]) + __bfloat162float(lo[i]);
    nrm = fmaf(v, v, nrm);
  }
  nrm = warp_sum(nrm);
  if (lane == 0) a.cnorm[(size_t)u * a.Cpad + j] = nrm;
  const int t = j >> 7, rr = j & 127;
  const int c16 = lane >> 1;             // 16-byte chunk of the 128 dims (0..15)
  const int cb = c16 >> 3, cc = c16 & 7;
  const size_t base = ((size_t)u * (a.Cpad / 128) + t) * TC_STAGE + cb * 16384 + (rr >> 3) * 1024 + (rr & 7) * 128 +
                      ((cc ^ (rr & 7)) << 4) + (lane & 1) * 8;
  uint2 vh, vl;
  vh.x = (uint32_t)__bfloat16_as_ushort(hi[0]) | ((uint32_t)__bfloat16_as_ushort(hi[1]) << 16);
  vh.y = (uint32_t)__bfloat16_as_ushort(hi[2]) | ((uint32_t)__bfloat16_as_ushort(hi[3]) << 16);
  vl.x = (uint32_t)__bfloat16_as_ushort(lo[0]) | ((uint32_t)__bfloat16_as_ushort(lo[1]) << 16);
  vl.y = (uint32_t)__bfloat16_as_ushort(lo[2]) | ((uint32_t)__bfloat16_as_ushort(lo[3]) << 16);
  *reinterpret_cast<uint2*>(a.bimg + base) = vh;
  *reinterpret_cast<uint2*>(a.bimg + base + 32768) = vl;
}

// ---------------------------------------------------------------- B1
__global__ void km_init_kernel(const KmArgs a, const int* __restrict__ init) {
  const int u = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + warp;
  if (j >= a.Cpad) return;
  if (j >= a.C) {  // padding centroid: never the argmin
    if (lane == 0) a.cnorm[(size_t)u * a.Cpad + j] = INFINITY;
    return;
  }
  const int tok = init[(size_t)u * a.C + j];
  const __nv_bfloat16* r = krow(a.K, a.sb, a.sh, a.sn, a.Hkv, u, tok) + lane * 4;
  float4 c;
  c.x = __bfloat162float(r[0]);
  c.y = __bfloat162float(r[1]);
  c.z = __bfloat162float(r[2]);
  c.w = __bfloat162float(r[3]);
  store_centroid(a, u, j, c);
}

// ---------------------------------------------------------------- B2 (tcgen05)
// Persistent: one CTA per SM walks the (unit, 256-key block) items.  Warp 0 lane 0 is the
// producer: each block's two 128-key A tiles arrive by TMA (SWIZZLE_128B boxes of 64 dims
// x 128 rows from the caller's K; rows past n zero-filled) into one of two A buffers, so
// the next block's keys land while the current block computes; the centroid tile images
// stream as 32 KB halves (hi, then lo) through TC_BST stages.  Warp 1 lane 0 issues the
// MMAs (per half: 2 A tiles x 8 K-steps, M = N = 128, K = 16) into a double-buffered
// accumulator [2][TC_KA][128 columns]; warps 2-9 run the argmin epilogue of tile t while
// the MMAs of tile t + 1 run.
__global__ void __launch_bounds__(320, 1)
    km_assign_tc_kernel(const KmArgs a, const __grid_constant__ CUtensorMap tmK, int iter, int* __restrict__ changed) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;                          // [2 buffers][TC_KA][128 keys x 128 dims]
  uint8_t* sB = sm + 2 * TC_KA * TC_A;       // [TC_BST][32 KB half tile]
  uint64_t* bars = (uint64_t*)(sB + TC_BST * TC_HALF);
  uint64_t* afull = bars;                    // [2]
  uint64_t* aempty = bars + 2;               // [2]
  uint64_t* bfull = bars + 4;                // [TC_BST]
  uint64_t* bempty = bars + 4 + TC_BST;      // [TC_BST]
  uint64_t* tfull = bars + 4 + 2 * TC_BST;   // [2]
  uint64_t* tempty = bars + 6 + 2 * TC_BST;  // [2]
  uint32_t* tmem_slot = (uint32_t*)(bars + 8 + 2 * TC_BST);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = a.Cpad / 128;
  const int nkb = (a.n + 128 * TC_KA - 1) / (128 * TC_KA);
  const int items = a.units * nkb;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    for (int i = 0; i < TC_BST; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256 * TC_KA);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // producer
      prefetch_tmap(&tmK);
      uint32_t g = 0, li = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int u = it / nkb, kb = it - u * nkb;
        if (a.converged[u] != 0) continue;
        const int ab = li & 1;
        mbar_wait(&aempty[ab], ((li >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&afull[ab], TC_KA * TC_A);
        const int bb = u / a.Hkv, hh = u - bb * a.Hkv;
#pragma unroll
        for (int at = 0; at < TC_KA; ++at)
#pragma unroll
          for (int cb = 0; cb < 2; ++cb)
            tma_load_4d(sA + (ab * TC_KA + at) * TC_A + cb * 16384, &tmK, cb * 64, kb * 128 * TC_KA + at * 128, hh,
                        bb, &afull[ab]);
        const uint8_t* img = a.bimg + (size_t)u * ntiles * TC_STAGE;
        for (int h = 0; h < 2 * ntiles; ++h, ++g) {
          const uint32_t st = g % TC_BST;
          mbar_wait(&bempty[st], ((g / TC_BST) & 1) ^ 1);
          mbar_arrive_expect_tx(&bfull[st], TC_HALF);
          bulk_g2s(sB + st * TC_HALF, img + (size_t)h * TC_HALF, TC_HALF, &bfull[st]);
        }
        ++li;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = umma_idesc_bf16(128, 128);
      uint32_t g = 0, tt = 0, li = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int u = it / nkb;
        if (a.converged[u] != 0) continue;
        const int ab = li & 1;
        mbar_wait(&afull[ab], (li >> 1) & 1);
        tc_fence_after();
        for (int t = 0; t < ntiles; ++t, ++tt) {
          const uint32_t acc = tt & 1;
          mbar_wait(&tempty[acc], ((tt >> 1) & 1) ^ 1);
          tc_fence_after();
#pragma unroll 1
          for (int h = 0; h < 2; ++h, ++g) {
            const uint32_t st = g % TC_BST;
            mbar_wait(&bfull[st], (g / TC_BST) & 1);
            tc_fence_after();
            const uint32_t baddr = smem_u32(sB + st * TC_HALF);
#pragma unroll
            for (int at = 0; at < TC_KA; ++at) {
              const uint32_t aaddr = smem_u32(sA + (ab * TC_KA + at) * TC_A);
              const uint32_t dcol = tmem + acc * (128 * TC_KA) + at * 128;
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const uint32_t koff = (kk >> 2) * 16384 + (kk & 3) * 32;
                tc_mma_f16(dcol, umma_desc_sw128(aaddr + koff), umma_desc_sw128(baddr + koff), idesc,
                           (h | kk) ? 1u : 0u);
              }
            }
            tc_commit(&bempty[st]);
          }
          tc_commit(&tfull[acc]);
        }
        tc_commit(&aempty[ab]);
        ++li;
      }
    }
  } else {
    // epilogue: warp w (2..9) reads TMEM lane quadrant w % 4 of A tile (w - 2) / 4, so a
    // thread owns one key row; four independent argmin chains (columns i % 4) keep the
    // compare/select dependency off the critical path, merged at the block's end with the
    // same rule (smallest distance, then lowest centroid index)
    const int q = warp & 3, at = (warp - 2) >> 2;
    uint32_t tt = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      const int u = it / nkb, kb = it - u * nkb;
      if (a.converged[u] != 0) continue;
      float best[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
      int arg[4] = {0, 0, 0, 0};
      const float* cn = a.cnorm + (size_t)u * a.Cpad;
      for (int t = 0; t < ntiles; ++t, ++tt) {
        const uint32_t acc = tt & 1;
        mbar_wait(&tfull[acc], (tt >> 1) & 1);
        tc_fence_after();
        // the tile's 128 columns in two TMEM round trips: columns 64..127 load while the
        // argmin runs over 0..63, and the accumulator goes back to the MMA issuer as soon as
        // the second load has landed (before the rest of the argmin)
        uint32_t v[4][32];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + acc * (128 * TC_KA) + at * 128;
        tmem_ld32(taddr, v[0]);
        tmem_ld32(taddr + 32, v[1]);
        tmem_ld_wait();
        tmem_ld32(taddr + 64, v[2]);
        tmem_ld32(taddr + 96, v[3]);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          if (ch == 2) {
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
          }
          const int jb = t * 128 + ch * 32;
          float cv[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 c4 = __ldg(reinterpret_cast<const float4*>(cn + jb) + i);
            cv[4 * i] = c4.x; cv[4 * i + 1] = c4.y; cv[4 * i + 2] = c4.z; cv[4 * i + 3] = c4.w;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float dist = fmaf(-2.f, __uint_as_float(v[ch][i]), cv[i]);
            if (dist < best[i & 3]) { best[i & 3] = dist; arg[i & 3] = jb + i; }
          }
        }
      }
      float bv = best[0];
      int ba = arg[0];
#pragma unroll
      for (int c = 1; c < 4; ++c)
        if (best[c] < bv || (best[c] == bv && arg[c] < ba)) { bv = best[c]; ba = arg[c]; }
      int ch = 0;
      const int row = kb * 128 * TC_KA + at * 128 + q * 32 + lane;
      if (row < a.n) {
        int* ap = a.assign + (size_t)u * a.n + row;
        ch = (*ap != ba) ? 1 : 0;
        *ap = ba;
      }
      ch = __reduce_add_sync(0xffffffffu, ch);
      if (lane == 0 && ch) atomicAdd(&changed[(size_t)iter * a.units + u], ch);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 256 * TC_KA);
}

// ---------------------------------------------------------------- B2 (CUDA cores, debug)
__global__ void __launch_bounds__(128) km_assign_simt_kernel(const KmArgs a, int iter, int* __restrict__ changed) {
  constexpr int CT = 16;
  __shared__ __nv_bfloat16 sK[128][130];  // [dim][token]
  __shared__ float sC[CT][128];
  __shared__ float sN[CT];
  const int u = blockIdx.y;
  if (a.converged[u] != 0) return;
  const int row0 = blockIdx.x * 128, t = threadIdx.x;
  for (int r = 0; r < 128; ++r) {
    const int row = row0 + r;
    sK[t][r] = row < a.n ? krow(a.K, a.sb, a.sh, a.sn, a.Hkv, u, row)[t] : __float2bfloat16_rn(0.f);
  }
  float best = INFINITY;
  int arg = 0;
  const int ntiles = a.Cpad / 128;
  for (int jt = 0; jt < a.Cpad; jt += CT) {
    __syncthreads();
    // rebuild hi + lo of centroids jt..jt+CT-1 from the tile image
    for (int e = t; e < CT * 128; e += 128) {
      const int jj = e >> 7, d = e & 127;
      const int j = jt + jj;
      const int tt = j >> 7, rr = j & 127, c16 = d >> 3, cb = c16 >> 3, cc = c16 & 7;
      const size_t base = ((size_t)u * ntiles + tt) * TC_STAGE + cb * 16384 + (rr >> 3) * 1024 + (rr & 7) * 128 +
                          ((cc ^ (rr & 7)) << 4) + (d & 7) * 2;
      const float h = __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(a.bimg + base));
      const float l = __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(a.bimg + base + 32768));
      sC[jj][d] = h + l;
    }
    if (t < CT) sN[t] = a.cnorm[(size_t)u * a.Cpad + jt + t];
    __syncthreads();
    float dot[CT];
#pragma unroll
    for (int jj = 0; jj < CT; ++jj) dot[jj] = 0.f;
    for (int d = 0; d < 128; ++d) {
      const float kv = __bfloat162float(sK[d][t]);
#pragma unroll
      for (int jj = 0; jj < CT; ++jj) dot[jj] = fmaf(kv, sC[jj][d], dot[jj]);
    }
#pragma unroll
    for (int jj = 0; jj < CT; ++jj) {
      const float dist = fmaf(-2.f, dot[jj], sN[jj]);
      if (dist < best) { best = dist; arg = jt + jj; }
    }
  }
  int ch = 0;
  const int row = row0 + t;
  if (row < a.n) {
    int* ap = a.assign + (size_t)u * a.n + row;
    ch = (*ap != arg) ? 1 : 0;
    *ap = arg;
  }
  ch = __reduce_add_sync(0xffffffffu, ch);
  if ((t & 31) == 0 && ch) atomicAdd(&changed[(size_t)iter * a.units + u], ch);
}

__device__ __forceinline__ bool km_skip(const KmArgs& a, int u, int iter) {
  const int c = a.converged[u];
  return c != 0 && c < iter;
}

// ---------------------------------------------------------------- B3 histogram
__global__ void km_count_kernel(const KmArgs a, int iter, const int* __restrict__ changed) {
  extern __shared__ int hist[];
  const int u = blockIdx.y, blk = blockIdx.x;
  if (km_skip(a, u, iter)) return;
  if (iter >= 2 && blk == 0 && threadIdx.x == 0 && a.converged[u] == 0 &&
      changed[(size_t)iter * a.units + u] == 0)
    a.converged[u] = iter;  // B4: fixpoint reached at this iteration
  for (int j = threadIdx.x; j < a.C; j += blockDim.x) hist[j] = 0;
  __syncthreads();
  const int i = blk * KM_BLK + threadIdx.x;
  if (i < a.n) atomicAdd(&hist[a.assign[(size_t)u * a.n + i]], 1);
  __syncthreads();
  int* bc = a.blk_counts + ((size_t)u * a.nblk + blk) * a.C;
  for (int j = threadIdx.x; j < a.C; j += blockDim.x) bc[j] = hist[j];
}

// Per-cluster exclusive prefix over the histogram blocks (in place) and each cluster's
// size.  CTA = 32 clusters (lanes) x 32 block groups (warps); a thread sums its group's
// blocks (loads batched, all in flight), the group prefixes come from shared memory, and
// a second pass writes the exclusive prefixes.  Exact integer arithmetic: any order.
__global__ void __launch_bounds__(1024) km_scan_kernel(const KmArgs a, int iter) {
  __shared__ int part[32][33];
  const int u = blockIdx.y, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (km_skip(a, u, iter)) return;
  const int j = blockIdx.x * 32 + lane;
  const int per = (a.nblk + 31) / 32;
  const int b0 = w * per, b1 = min(a.nblk, b0 + per);
  const bool col_ok = j < a.C;
  int* col = a.blk_counts + (size_t)u * a.nblk * a.C + (col_ok ? j : 0);
  int sum = 0;
  for (int b = b0; b < b1; b += 8) {
    int v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = (col_ok && b + q < b1) ? col[(size_t)(b + q) * a.C] : 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) sum += v[q];
  }
  part[w][lane] = sum;
  __syncthreads();
  int run = 0;
  for (int x = 0; x < w; ++x) run += part[x][lane];
  if (w == 31 && col_ok) a.col_tot[(size_t)u * a.C + j] = run + sum;
  if (!col_ok) return;
  for (int b = b0; b < b1; b += 8) {
    int v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = b + q < b1 ? col[(size_t)(b + q) * a.C] : 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (b + q < b1) col[(size_t)(b + q) * a.C] = run;
      run += v[q];
    }
  }
}

// Stable scatter: one warp walks its block's tokens in order (match_any ranks equal
// clusters within a step).  The block's assignments are loaded up front; the cluster
// offsets are the exclusive prefix of the cluster sizes, which every CTA derives itself
// (block 0 publishes them for the update and the layout) -- no separate offsets pass.
__global__ void __launch_bounds__(32) km_scatter_kernel(const KmArgs a, int iter) {
  extern __shared__ int cnt[];
  const int u = blockIdx.y, blk = blockIdx.x, lane = threadIdx.x;
  if (km_skip(a, u, iter)) return;
  const int* as = a.assign + (size_t)u * a.n;
  int cl[KM_BLK / 32];
#pragma unroll
  for (int step = 0; step < KM_BLK / 32; ++step) {
    const int i = blk * KM_BLK + step * 32 + lane;
    cl[step] = i < a.n ? as[i] : -1;
  }
  // lane owns clusters [lane * per, lane * per + per)
  const int* tot = a.col_tot + (size_t)u * a.C;
  const int per = (a.C + 31) / 32;
  int own = 0;
  for (int k0 = 0; k0 < per; k0 += 16) {
    int v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int jj = lane * per + k0 + q;
      v[q] = (k0 + q < per && jj < a.C) ? tot[jj] : 0;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) own += v[q];
  }
  int inc = own;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  int run = inc - own;
  int* off = a.offsets + (size_t)u * (a.C + 1);
  for (int k0 = 0; k0 < per; k0 += 16) {
    int v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int jj = lane * per + k0 + q;
      v[q] = (k0 + q < per && jj < a.C) ? tot[jj] : 0;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int jj = lane * per + k0 + q;
      if (k0 + q < per && jj < a.C) {
        cnt[jj] = run;
        if (blk == 0) off[jj] = run;
      }
      run += v[q];
    }
  }
  if (blk == 0 && lane == 31) off[a.C] = run;
  __syncwarp();
  const int* bc = a.blk_counts + ((size_t)u * a.nblk + blk) * a.C;
  for (int jj = lane; jj < a.C; jj += 32) cnt[jj] += bc[jj];
  __syncwarp();
  int* perm = a.perm + (size_t)u * a.n;
#pragma unroll
  for (int step = 0; step < KM_BLK / 32; ++step) {
    const int i = blk * KM_BLK + step * 32 + lane;
    const int c = cl[step];
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    if (c >= 0) perm[cnt[c] + __popc(peers & ((1u << lane) - 1u))] = i;
    __syncwarp();
    if (c >= 0 && (__ffs(peers) - 1) == lane) cnt[c] += __popc(peers);
    __syncwarp();
  }
}

// ---------------------------------------------------------------- B3 means
// One CTA per cluster: its 8 warps take every 8th member row (8 independent gather
// streams per cluster instead of one dependent walk), fp64 per-warp partial sums, combined
// in warp order -- deterministic; the member mean in fp64 as before.
__global__ void __launch_bounds__(256) km_update_kernel(const KmArgs a, int iter) {
  __shared__ double part[8][128];
  const int u = blockIdx.y, j = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (km_skip(a, u, iter)) return;
  if (j >= a.C) return;
  const int* off = a.offsets + (size_t)u * (a.C + 1);
  const int* perm = a.perm + (size_t)u * a.n;
  const int s = off[j], e = off[j + 1];
  if (e <= s) {
    if (warp == 0) {
      const float4 c = *reinterpret_cast<const float4*>(a.cent + ((size_t)u * a.C + j) * 128 + lane * 4);
      store_centroid(a, u, j, c);
    }
    return;
  }
  // warp w sums rows s + w, s + w + 8, ... in that order (the unit's row base hoisted: the
  // compiler unrolls the loop with several perm -> row gathers in flight; an explicit
  // 8-row batch with shuffled indices measured 1.8x slower: 177 vs 96 us per C2 iteration)
  double acc[4] = {0, 0, 0, 0};
  const __nv_bfloat16* Ku = krow(a.K, a.sb, a.sh, a.sn, a.Hkv, u, 0) + lane * 4;
  for (int r = s + warp; r < e; r += 8) {
    const uint2 raw = *reinterpret_cast<const uint2*>(Ku + (long long)perm[r] * a.sn);
    const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
    const float2 f0 = __bfloat1622float2(k2[0]), f1 = __bfloat1622float2(k2[1]);
    acc[0] += f0.x; acc[1] += f0.y; acc[2] += f1.x; acc[3] += f1.y;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) part[warp][lane * 4 + i] = acc[i];
  __syncthreads();
  if (warp == 0) {
    double t[4] = {0, 0, 0, 0};
#pragma unroll
    for (int w = 0; w < 8; ++w)
#pragma unroll
      for (int i = 0; i < 4; ++i) t[i] += part[w][lane * 4 + i];
    const double inv = (double)(e - s);
    store_centroid(a, u, j, make_float4((float)(t[0] / inv), (float)(t[1] / inv), (float)(t[2] / inv),
                                        (float)(t[3] / inv)));
  }
}

// B3 as a streaming pass (a.acc): the member rows in cluster order (perm), each warp over 128
// consecutive positions with 8 rows in flight (a half-warp per row, 16 bytes per lane), the
// running sum of the current cluster in registers and flushed with fp64 reductions at every
// cluster boundary; km_update_fin_kernel divides by the sizes.  The fp64 sums of bf16 rows
// are exact (8-bit mantissas, < 2^17 terms over a bounded exponent range), so the order of
// the reductions does not change the means.
__global__ void __launch_bounds__(256) km_update_seg_kernel(const KmArgs a, int iter) {
  const int u = blockIdx.y;
  if (km_skip(a, u, iter)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, half = lane >> 4, l16 = lane & 15;
  const int p_begin = (blockIdx.x * 8 + warp) * 128;
  if (p_begin >= a.n) return;
  const int p_end = min(a.n, p_begin + 128);
  const int* perm = a.perm + (size_t)u * a.n;
  const int* asg = a.assign + (size_t)u * a.n;
  const __nv_bfloat16* Ku = krow(a.K, a.sb, a.sh, a.sn, a.Hkv, u, 0) + l16 * 8;
  double* accu = a.acc + (size_t)u * a.C * 128 + l16 * 8;
  double sacc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) sacc[i] = 0.0;
  int cur = -1;  // the cluster being summed (warp-uniform)
  auto flush = [&]() {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      sacc[i] += __shfl_xor_sync(0xffffffffu, sacc[i], 16);
      if (half == 0) atomicAdd(accu + (size_t)cur * 128 + i, sacc[i]);
      sacc[i] = 0.0;
    }
  };
  auto add = [&](const uint4& raw) {
    const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(k2[i]);
      sacc[2 * i] += f.x;
      sacc[2 * i + 1] += f.y;
    }
  };
  for (int p0 = p_begin; p0 < p_end; p0 += 8) {
    uint4 raw[4];
    int cj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int p = p0 + 2 * q + half;
      const bool ok = p < p_end;
      const int key = ok ? __ldg(perm + p) : 0;
      cj[q] = ok ? __ldg(asg + key) : -1;
      raw[q] = ok ? __ldg(reinterpret_cast<const uint4*>(Ku + (long long)key * a.sn)) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c0 = __shfl_sync(0xffffffffu, cj[q], 0), c1 = __shfl_sync(0xffffffffu, cj[q], 16);
      if (c0 < 0) continue;  // past the warp's positions
      if (cur < 0) cur = c0;
      if (c0 != cur) {  // both rows start a later cluster
        flush();
        cur = c0;
      }
      if (c1 >= 0 && c1 != cur) {  // the half-0 row ends cluster cur, the half-1 row starts c1
        if (half == 0) add(raw[q]);
        flush();
        cur = c1;
        if (half == 1) add(raw[q]);
      } else if (half == 0 || c1 >= 0) {
        add(raw[q]);
      }
    }
  }
  if (cur >= 0) flush();
}

// means from the streamed sums: one warp per cluster (lane: dims 4 lane .. 4 lane + 3); an
// empty cluster keeps its centroid; the sums are zeroed for the next iteration
__global__ void __launch_bounds__(256) km_update_fin_kernel(const KmArgs a, int iter) {
  const int u = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (km_skip(a, u, iter)) return;
  const int j = blockIdx.x * 8 + warp;
  if (j >= a.C) return;
  const int* off = a.offsets + (size_t)u * (a.C + 1);
  const int sz = off[j + 1] - off[j];
  double* acc = a.acc + ((size_t)u * a.C + j) * 128 + lane * 4;
  if (sz <= 0) {
    const float4 c = *reinterpret_cast<const float4*>(a.cent + ((size_t)u * a.C + j) * 128 + lane * 4);
    store_centroid(a, u, j, c);
    return;
  }
  const double2 s01 = *reinterpret_cast<const double2*>(acc), s23 = *reinterpret_cast<const double2*>(acc + 2);
  *reinterpret_cast<double2*>(acc) = make_double2(0.0, 0.0);
  *reinterpret_cast<double2*>(acc + 2) = make_double2(0.0, 0.0);
  const double inv = (double)sz;
  store_centroid(a, u, j, make_float4((float)(s01.x / inv), (float)(s01.y / inv), (float)(s23.x / inv),
                                      (float)(s23.y / inv)));
}

// ---------------------------------------------------------------- B5 / B6
__global__ void km_relayout_kernel(const KmArgs a) {
  const int u = blockIdx.y;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int r = warp * 2 + (lane >> 4);
  if (r >= a.n) return;
  const int l16 = lane & 15;
  const int src = a.perm[(size_t)u * a.n + r];
  const uint4 kv = *reinterpret_cast<const uint4*>(krow(a.K, a.sb, a.sh, a.sn, a.Hkv, u, src) + l16 * 8);
  const uint4 vv = *reinterpret_cast<const uint4*>(krow(a.V, a.sb, a.sh, a.sn, a.Hkv, u, src) + l16 * 8);
  const size_t dst = ((size_t)u * a.n + r) * 128 + swz_chunk(l16, r) * 8;
  *reinterpret_cast<uint4*>(a.Kp + dst) = kv;
  *reinterpret_cast<uint4*>(a.Vp + dst) = vv;
}

__global__ void km_all_list_kernel(const KmArgs a, int iters) {
  __shared__ int red[32];
  __shared__ int tot_c, tot_t;
  const int u = blockIdx.x;
  const int* off = a.offsets + (size_t)u * (a.C + 1);
  const int per = (a.C + blockDim.x - 1) / blockDim.x;
  const int j0 = threadIdx.x * per;
  int lc = 0, lt = 0;
  for (int j = j0; j < j0 + per && j < a.C; ++j)
    if (off[j + 1] > off[j]) { ++lc; lt += off[j + 1] - off[j]; }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // two exclusive scans (count, tokens) packed in one pass each
  int vals[2] = {lc, lt}, bases[2];
  for (int q = 0; q < 2; ++q) {
    int inc = vals[q];
    for (int o = 1; o < 32; o <<= 1) {
      int x = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += x;
    }
    __syncthreads();
    if (lane == 31) red[w] = inc;
    __syncthreads();
    if (w == 0) {
      int s = lane < nw ? red[lane] : 0, si = s;
      for (int o = 1; o < 32; o <<= 1) {
        int x = __shfl_up_sync(0xffffffffu, si, o);
        if (lane >= o) si += x;
      }
      if (lane < nw) red[lane] = si - s;
      if (lane == nw - 1) { if (q == 0) tot_c = si; else tot_t = si; }
    }
    __syncthreads();
    bases[q] = red[w] + inc - vals[q];
  }
  int* ul = a.all_list + (size_t)u * a.C;
  int* up = a.all_prefix + (size_t)u * (a.C + 1);
  int cb = bases[0], tb = bases[1];
  for (int j = j0; j < j0 + per && j < a.C; ++j)
    if (off[j + 1] > off[j]) {
      ul[cb] = off[j];  // segment = first layout row of the cluster
      up[cb] = tb;
      ++cb;
      tb += off[j + 1] - off[j];
    }
  __syncthreads();
  for (int k = tot_c + threadIdx.x; k <= a.C; k += blockDim.x) {
    up[k] = tot_t;
    if (k < a.C) ul[k] = 0;
  }
  if (threadIdx.x == 0) a.iters_run[u] = a.converged[u] ? a.converged[u] : iters;
}

// sum over cluster j's rows of |k - c_j|^2 in fp64, read from the cluster-contiguous
// layout.  One CTA per cluster: warp w takes rows r0 + w, r0 + w + 8, ... (8 rows' loads in
// flight), the 8 warp partials are added in warp order -- deterministic, and the largest
// cluster no longer sets the kernel time on one warp (one warp per cluster: 406 us at C2).
__global__ void __launch_bounds__(256) km_inertia_kernel(const KmArgs a, double* __restrict__ part) {
  __shared__ double wsum[8];
  const int u = blockIdx.y, j = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* off = a.offsets + (size_t)u * (a.C + 1);
  const float4 c = *reinterpret_cast<const float4*>(a.cent + ((size_t)u * a.C + j) * 128 + lane * 4);
  double s = 0.0;
  const int r0 = off[j], r1 = off[j + 1];
  for (int rb = r0 + warp; rb < r1; rb += 64) {
    uint2 raw[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = rb + 8 * i;
      // dims 4*lane..4*lane+3 live in logical chunk lane/2, half lane%2
      raw[i] = r < r1 ? *reinterpret_cast<const uint2*>(a.Kp + ((size_t)u * a.n + r) * 128 +
                                                        swz_chunk(lane >> 1, r) * 8 + (lane & 1) * 4)
                      : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (rb + 8 * i >= r1) break;
      const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&raw[i]);
      const float2 x0 = __bfloat1622float2(k2[0]), x1 = __bfloat1622float2(k2[1]);
      const double d0 = (double)x0.x - c.x, d1 = (double)x0.y - c.y;
      const double d2 = (double)x1.x - c.z, d3 = (double)x1.y - c.w;
      s += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
    }
  }
  s = warp_sum_d(s);
  if (lane == 0) wsum[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += wsum[w];
    part[(size_t)u * a.C + j] = t;
  }
}

__global__ void km_finite_kernel(const KmArgs a, int* __restrict__ flag) {
  const int u = blockIdx.y;
  const int i = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4);
  if (i >= a.n) return;
  const int l16 = threadIdx.x & 15;
  const uint4 kv = *reinterpret_cast<const uint4*>(krow(a.K, a.sb, a.sh, a.sn, a.Hkv, u, i) + l16 * 8);
  const uint4 vv = *reinterpret_cast<const uint4*>(krow(a.V, a.sb, a.sh, a.sn, a.Hkv, u, i) + l16 * 8);
  const uint32_t w[8] = {kv.x, kv.y, kv.z, kv.w, vv.x, vv.y, vv.z, vv.w};
  bool bad = false;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    bad |= ((w[q] & 0x7F80u) == 0x7F80u) || ((w[q] & 0x7F800000u) == 0x7F800000u);
  }
  if (bad) atomicOr(flag, 1);
}

// ---------------------------------------------------------------- launchers
cudaError_t km_init_centroids(const KmArgs& a, const int* init_dev, cudaStream_t s) {
  km_init_kernel<<<dim3((a.Cpad + 7) / 8, a.units), 256, 0, s>>>(a, init_dev);
  return cudaGetLastError();
}

cudaError_t km_assign(const KmArgs& a, const CUtensorMap* tmK, int iter, bool simt, cudaStream_t s) {
  if (simt) {
    km_assign_simt_kernel<<<dim3((a.n + 127) / 128, a.units), 128, 0, s>>>(a, iter, a.changed);
    return cudaGetLastError();
  }
  cudaError_t e = func_smem_optin((const void*)km_assign_tc_kernel, TC_SMEM);
  if (e != cudaSuccess) return e;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  }
  const long long items = (long long)a.units * ((a.n + 128 * TC_KA - 1) / (128 * TC_KA));
  km_assign_tc_kernel<<<(unsigned)std::min<long long>(items, sms), 320, TC_SMEM, s>>>(a, *tmK, iter, a.changed);
  return cudaGetLastError();
}

cudaError_t km_count_scan_scatter(const KmArgs& a, int iter, cudaStream_t s) {
  km_count_kernel<<<dim3(a.nblk, a.units), KM_BLK, (size_t)a.C * 4, s>>>(a, iter, a.changed);
  km_scan_kernel<<<dim3((a.C + 31) / 32, a.units), 1024, 0, s>>>(a, iter);
  km_scatter_kernel<<<dim3(a.nblk, a.units), 32, (size_t)a.C * 4, s>>>(a, iter);
  return cudaGetLastError();
}

cudaError_t km_update(const KmArgs& a, int iter, cudaStream_t s) {
  if (a.acc) {  // streaming pass over the member rows + means (16-byte row slices)
    km_update_seg_kernel<<<dim3((a.n + 1023) / 1024, a.units), 256, 0, s>>>(a, iter);
    km_update_fin_kernel<<<dim3((a.C + 7) / 8, a.units), 256, 0, s>>>(a, iter);
    return cudaGetLastError();
  }
  km_update_kernel<<<dim3(a.C, a.units), 256, 0, s>>>(a, iter);
  return cudaGetLastError();
}

cudaError_t km_finalize(const KmArgs& a, cudaStream_t s) {
  km_relayout_kernel<<<dim3((a.n + 15) / 16, a.units), 256, 0, s>>>(a);
  km_all_list_kernel<<<a.units, 1024, 0, s>>>(a, a.iters_req);
  return cudaGetLastError();
}

cudaError_t km_inertia(const KmArgs& a, double* part, cudaStream_t s) {
  km_inertia_kernel<<<dim3(a.C, a.units), 256, 0, s>>>(a, part);
  return cudaGetLastError();
}

cudaError_t km_check_finite(const KmArgs& a, int* flag, cudaStream_t s) {
  km_finite_kernel<<<dim3((a.n + 15) / 16, a.units), 256, 0, s>>>(a, flag);
  return cudaGetLastError();
}

}  // namespace tactic
