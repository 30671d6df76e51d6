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

#include "common.cuh"
#include "internal.h"

namespace tactic {

constexpr int KM_BLK = 1024;         // tokens per histogram / scatter block
constexpr int TC_STAGE = 65536;      // one centroid tile image: hi 32 KB | lo 32 KB
constexpr int TC_A = 32768;          // 128 keys x 128 dims bf16
constexpr int TC_KA = 2;             // A tiles (128 keys each) per CTA: every centroid tile
                                     // streamed from L2 feeds 256 keys (halves B traffic)
constexpr size_t TC_SMEM = 1024 + TC_KA * (size_t)TC_A + 2 * (size_t)TC_STAGE + 256;

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
__global__ void __launch_bounds__(192, 1) km_assign_tc_kernel(const KmArgs a, int iter, int* __restrict__ changed) {
  extern __shared__ uint8_t smraw[];
  const int u = blockIdx.y;
  if (a.converged[u] != 0) return;
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;                       // [TC_KA][128 keys x 128 dims], SWIZZLE_128B K-major
  uint8_t* sB = sm + TC_KA * TC_A;
  uint64_t* bars = (uint64_t*)(sB + 2 * TC_STAGE);
  uint64_t* full = bars;          // [2]
  uint64_t* empty = bars + 2;     // [2]
  uint64_t* tfull = bars + 4;     // [2]
  uint64_t* tempty = bars + 6;    // [2]
  uint32_t* tmem_slot = (uint32_t*)(bars + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * (128 * TC_KA);
  const int ntiles = a.Cpad / 128;

  // A tiles: 128 * TC_KA keys, SWIZZLE_128B K-major (two 64-dim column blocks per tile),
  // loaded by the epilogue warps with cp.async; rows past n are zero.
  if (warp >= 2) {
    const int t = threadIdx.x - 64;  // 0..127
    for (int c = t; c < TC_KA * 128 * 16; c += 128) {
      const int ra = c >> 4, ch = c & 15;
      const int at = ra >> 7, r = ra & 127;
      const int cb = ch >> 3, cc = ch & 7;
      const bool valid = row0 + ra < a.n;
      const __nv_bfloat16* src = krow(a.K, a.sb, a.sh, a.sn, a.Hkv, u, valid ? row0 + ra : 0) + ch * 8;
      cp_async16(sA + at * TC_A + cb * 16384 + (r >> 3) * 1024 + (r & 7) * 128 + ((cc ^ (r & 7)) << 4), src,
                 valid);
    }
    cp_async_commit();
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  // accumulators: [2 buffers][TC_KA A tiles][128 columns]
  if (warp == 1) tmem_alloc(tmem_slot, 256 * TC_KA);
  if (warp >= 2) cp_async_wait_all();
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint8_t* img = a.bimg + (size_t)u * ntiles * TC_STAGE;

  if (warp == 0) {
    if (lane == 0) {  // producer: centroid tile images
      for (int t = 0; t < ntiles; ++t) {
        const int s = t & 1;
        const uint32_t ph = (t >> 1) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], TC_STAGE);
        bulk_g2s(sB + s * TC_STAGE, img + (size_t)t * TC_STAGE, TC_STAGE, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = umma_idesc_bf16(128, 128);
      for (int t = 0; t < ntiles; ++t) {
        const int s = t & 1, acc = t & 1;
        const uint32_t ph = (t >> 1) & 1;
        mbar_wait(&tempty[acc], ph ^ 1);
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t baddr = smem_u32(sB + s * TC_STAGE);
#pragma unroll
        for (int at = 0; at < TC_KA; ++at) {
          const uint32_t aaddr = smem_u32(sA + at * TC_A);
          const uint32_t dcol = tmem + acc * (128 * TC_KA) + at * 128;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t koff = (kk >> 2) * 16384 + (kk & 3) * 32;
            const uint64_t ad = umma_desc_sw128(aaddr + koff);
            tc_mma_f16(dcol, ad, umma_desc_sw128(baddr + koff), idesc, kk > 0 ? 1u : 0u);
            tc_mma_f16(dcol, ad, umma_desc_sw128(baddr + 32768 + koff), idesc, 1u);
          }
        }
        tc_commit(&empty[s]);
        tc_commit(&tfull[acc]);
      }
    }
  } else {
    // epilogue: thread <-> key row (TMEM lane) of every A tile; argmin over all centroids
    const int q = warp & 3;
    float best[TC_KA];
    int arg[TC_KA];
#pragma unroll
    for (int at = 0; at < TC_KA; ++at) {
      best[at] = INFINITY;
      arg[at] = 0;
    }
    const float* cn = a.cnorm + (size_t)u * a.Cpad;
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t & 1;
      const uint32_t ph = (t >> 1) & 1;
      mbar_wait(&tfull[acc], ph);
      tc_fence_after();
#pragma unroll 1
      for (int ch = 0; ch < 4; ++ch) {
        const int jb = t * 128 + ch * 32;
        float cv[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 c4 = __ldg(reinterpret_cast<const float4*>(cn + jb) + i);
          cv[4 * i] = c4.x; cv[4 * i + 1] = c4.y; cv[4 * i + 2] = c4.z; cv[4 * i + 3] = c4.w;
        }
#pragma unroll
        for (int at = 0; at < TC_KA; ++at) {
          uint32_t v[32];
          tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * (128 * TC_KA) + at * 128 + ch * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float dist = fmaf(-2.f, __uint_as_float(v[i]), cv[i]);
            if (dist < best[at]) { best[at] = dist; arg[at] = jb + i; }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    int ch = 0;
#pragma unroll
    for (int at = 0; at < TC_KA; ++at) {
      const int row = row0 + at * 128 + q * 32 + lane;
      if (row < a.n) {
        int* ap = a.assign + (size_t)u * a.n + row;
        ch += (*ap != arg[at]) ? 1 : 0;
        *ap = arg[at];
      }
    }
    ch = __reduce_add_sync(0xffffffffu, ch);
    if (lane == 0 && ch) atomicAdd(&changed[(size_t)iter * a.units + u], ch);
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

// per-cluster exclusive prefix over blocks (in place) + cluster offsets
__global__ void __launch_bounds__(1024) km_scan_kernel(const KmArgs a, int iter) {
  __shared__ int red[32];
  __shared__ int total_sh;
  const int u = blockIdx.x;
  if (km_skip(a, u, iter)) return;
  const int per = (a.C + blockDim.x - 1) / blockDim.x;
  const int j0 = threadIdx.x * per;
  int tot[4] = {0, 0, 0, 0};
  for (int k = 0; k < per && k < 4; ++k) {
    const int j = j0 + k;
    if (j >= a.C) break;
    // column scan over the blocks, 16 independent loads in flight per batch
    int run = 0;
    int* col = a.blk_counts + (size_t)u * a.nblk * a.C + j;
    for (int b0 = 0; b0 < a.nblk; b0 += 16) {
      int v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = b0 + q < a.nblk ? col[(size_t)(b0 + q) * a.C] : 0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (b0 + q < a.nblk) col[(size_t)(b0 + q) * a.C] = run;
        run += v[q];
      }
    }
    tot[k] = run;
  }
  int loc = 0;
  for (int k = 0; k < per && k < 4; ++k) loc += tot[k];
  // block exclusive scan
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int inc = loc;
  for (int o = 1; o < 32; o <<= 1) {
    int x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  if (lane == 31) red[w] = inc;
  __syncthreads();
  if (w == 0) {
    int s = lane < nw ? red[lane] : 0, si = s;
    for (int o = 1; o < 32; o <<= 1) {
      int x = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += x;
    }
    if (lane < nw) red[lane] = si - s;
    if (lane == nw - 1) total_sh = si;
  }
  __syncthreads();
  int base = red[w] + inc - loc;
  int* off = a.offsets + (size_t)u * (a.C + 1);
  for (int k = 0; k < per && k < 4; ++k) {
    const int j = j0 + k;
    if (j >= a.C) break;
    off[j] = base;
    base += tot[k];
  }
  if (threadIdx.x == 0) off[a.C] = total_sh;
}

// stable scatter: one warp walks its block's tokens in order
__global__ void km_scatter_kernel(const KmArgs a, int iter) {
  extern __shared__ int cnt[];
  const int u = blockIdx.y, blk = blockIdx.x, lane = threadIdx.x;
  if (km_skip(a, u, iter)) return;
  const int* off = a.offsets + (size_t)u * (a.C + 1);
  const int* bc = a.blk_counts + ((size_t)u * a.nblk + blk) * a.C;
  for (int j = lane; j < a.C; j += 32) cnt[j] = off[j] + bc[j];
  __syncwarp();
  const int* as = a.assign + (size_t)u * a.n;
  int* perm = a.perm + (size_t)u * a.n;
  for (int step = 0; step < KM_BLK / 32; ++step) {
    const int i = blk * KM_BLK + step * 32 + lane;
    const bool valid = i < a.n;
    const int c = valid ? as[i] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    if (valid) {
      const int rank = __popc(peers & ((1u << lane) - 1u));
      perm[cnt[c] + rank] = i;
    }
    __syncwarp();
    if (valid && (__ffs(peers) - 1) == lane) cnt[c] += __popc(peers);
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
  double acc[4] = {0, 0, 0, 0};
  for (int r = s + warp; r < e; r += 8) {
    const __nv_bfloat16* k = krow(a.K, a.sb, a.sh, a.sn, a.Hkv, u, perm[r]) + lane * 4;
    const uint2 raw = *reinterpret_cast<const uint2*>(k);
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
// layout (one warp per cluster, member order): deterministic per-cluster partials.
__global__ void km_inertia_kernel(const KmArgs a, double* __restrict__ part) {
  const int u = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + warp;
  if (j >= a.C) return;
  const int* off = a.offsets + (size_t)u * (a.C + 1);
  const float4 c = *reinterpret_cast<const float4*>(a.cent + ((size_t)u * a.C + j) * 128 + lane * 4);
  // the cluster's member rows in order, 8 rows' loads in flight per warp (a lone dependent
  // walk ran at ~0.3 TB/s); per-row sums added in row order, so the result is deterministic
  double s = 0.0;
  const int r0 = off[j], r1 = off[j + 1];
  for (int rb = r0; rb < r1; rb += 8) {
    uint2 raw[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = rb + i;
      // dims 4*lane..4*lane+3 live in logical chunk lane/2, half lane%2
      raw[i] = r < r1 ? *reinterpret_cast<const uint2*>(a.Kp + ((size_t)u * a.n + r) * 128 +
                                                        swz_chunk(lane >> 1, r) * 8 + (lane & 1) * 4)
                      : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (rb + i >= r1) break;
      const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&raw[i]);
      const float2 x0 = __bfloat1622float2(k2[0]), x1 = __bfloat1622float2(k2[1]);
      const double d0 = (double)x0.x - c.x, d1 = (double)x0.y - c.y;
      const double d2 = (double)x1.x - c.z, d3 = (double)x1.y - c.w;
      s += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
    }
  }
  s = warp_sum_d(s);
  if (lane == 0) part[(size_t)u * a.C + j] = s;
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

cudaError_t km_assign(const KmArgs& a, int iter, bool simt, cudaStream_t s) {
  const dim3 grid((a.n + 127) / 128, a.units);
  const dim3 grid_tc((a.n + 128 * TC_KA - 1) / (128 * TC_KA), a.units);
  if (simt) {
    km_assign_simt_kernel<<<grid, 128, 0, s>>>(a, iter, a.changed);
    return cudaGetLastError();
  }
  cudaError_t e = func_smem_optin((const void*)km_assign_tc_kernel, TC_SMEM);
  if (e != cudaSuccess) return e;
  km_assign_tc_kernel<<<grid_tc, 192, TC_SMEM, s>>>(a, iter, a.changed);
  return cudaGetLastError();
}

cudaError_t km_count_scan_scatter(const KmArgs& a, int iter, cudaStream_t s) {
  km_count_kernel<<<dim3(a.nblk, a.units), KM_BLK, (size_t)a.C * 4, s>>>(a, iter, a.changed);
  km_scan_kernel<<<a.units, 1024, 0, s>>>(a, iter);
  km_scatter_kernel<<<dim3(a.nblk, a.units), 32, (size_t)a.C * 4, s>>>(a, iter);
  return cudaGetLastError();
}

cudaError_t km_update(const KmArgs& a, int iter, cudaStream_t s) {
  km_update_kernel<<<dim3(a.C, a.units), 256, 0, s>>>(a, iter);
  return cudaGetLastError();
}

cudaError_t km_finalize(const KmArgs& a, cudaStream_t s) {
  km_relayout_kernel<<<dim3((a.n + 15) / 16, a.units), 256, 0, s>>>(a);
  km_all_list_kernel<<<a.units, 1024, 0, s>>>(a, a.iters_req);
  return cudaGetLastError();
}

cudaError_t km_inertia(const KmArgs& a, double* part, cudaStream_t s) {
  km_inertia_kernel<<<dim3((a.C + 7) / 8, a.units), 256, 0, s>>>(a, part);
  return cudaGetLastError();
}

cudaError_t km_check_finite(const KmArgs& a, int* flag, cudaStream_t s) {
  km_finite_kernel<<<dim3((a.n + 15) / 16, a.units), 256, 0, s>>>(a, flag);
  return cudaGetLastError();
}

}  // namespace tactic
