// select.cu -- decode-time selection S1, S4-S7 (§4.3-§4.6, App. B Alg. 1).
//
//  score_kernel    S1  crit[u][g][j] = q_g . c_j in float64 (products of a
//                      bf16 query and a float32 centroid are exact in fp64, so only the
//                      summation order differs from the oracle).  A warp scores 32/G
//                      centroids for all G heads and reduce-scatters the 32 partial sums
//                      with a shuffle butterfly (31 exchanges instead of 5 per value).
//                      Used before score_rank_kernel when the clusters span several waves.
//  (S1 + S2 + S3 run in rank_cluster.cu: scores, sorted order, end ranks, row map)
//  sample_kernel   S4  exact logits q.k/sqrt(d) of the sampled ranks: the first N ranks
//                      and two windows of 2w+1 ranks around x1, x2 (Alg. 1 l.4,
//                      readings 8-11), with per-block summaries for the fit.
//  fit_unit_kernel S5-S7 per unit (one warp per head): shift m, E_N, window means,
//                      two-point fit y = a/x + b, W, minimal k with
//                      cum(k) >= p W (Alg. 1 l.10) at cluster granularity (reading
//                      14), the GQA union compacted into the attention work list.
//                      Sequence-sharded mode (reading 23): stage 1 = the fit only, stage 2
//                      = the shared threshold theta* selects a rank prefix per head.
//  stage1b_kernel  sharded stage 1b: the shard's mass above every grid point.
// The clamp-aware tail sum  sum_{i=N+1}^{k} max(0, a/i + b)  uses harmonic numbers from
// the asymptotic digamma series (fitmath.cuh) instead of a table.
#include <cuda_bf16.h>
#include <float.h>
#include <limits.h>
#include <stdlib.h>

#include "common.cuh"
#include "internal.h"
#include "fitmath.cuh"

namespace tactic {

// exclusive scan of per-thread totals across the block; returns this thread's offset
template <typename T>
__device__ T block_exclusive_scan(T v, T* red, T* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  __syncthreads();
  if (lane == 31) red[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = lane < nw ? red[lane] : (T)0;
    T si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T x = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += x;
    }
    if (lane < nw) red[lane] = si - s;
    if (lane == nw - 1 && total) *total = si;
  }
  __syncthreads();
  T r = red[w] + inc - v;
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ S1
// Each warp scores CPW = 32/G centroids; value index v = jj*G + g ends on lane v.
template <int G>
__global__ void __launch_bounds__(256) score_kernel(const __nv_bfloat16* __restrict__ q,
                                                    const float* __restrict__ cent, int C,
                                                    double* __restrict__ crit, unsigned long long* tlog) {
  constexpr int CPW = 32 / G;
  const bool tl_first = blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
  if (threadIdx.x == 0) tl_mark(tlog, 0, 0, tl_first);
  pdl_wait();
  if (threadIdx.x == 0) tl_mark(tlog, 0, 1, tl_first);
  const int u = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double qd[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint2 raw = *reinterpret_cast<const uint2*>(q + ((size_t)u * G + g) * 128 + lane * 4);
    const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
    const float2 a = __bfloat1622float2(q2[0]), b = __bfloat1622float2(q2[1]);
    qd[g][0] = a.x; qd[g][1] = a.y; qd[g][2] = b.x; qd[g][3] = b.y;
  }
  const int j0 = (blockIdx.x * (blockDim.x >> 5) + warp) * CPW;
  if (j0 >= C) return;
  float4 c[CPW];
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
    c[jj] = j0 + jj < C ? *reinterpret_cast<const float4*>(cent + ((size_t)u * C + j0 + jj) * 128 + lane * 4)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
  double v[32];
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double s = qd[g][0] * (double)c[jj].x;
      s = fma(qd[g][1], (double)c[jj].y, s);
      s = fma(qd[g][2], (double)c[jj].z, s);
      s = fma(qd[g][3], (double)c[jj].w, s);
      v[jj * G + g] = s;
    }
  // butterfly reduce-scatter: after the level with offset o, lanes keep the half of the
  // values selected by their bit o; after 5 levels lane L holds the total of value L.
#pragma unroll
  for (int o = 16, half = 16; o >= 1; o >>= 1, half >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = upper ? v[i] : v[i + half];
      const double keep = upper ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  const int jj = lane / G, g = lane % G;
  if (j0 + jj < C) crit[((size_t)u * G + g) * C + j0 + jj] = v[0];
  if (threadIdx.x == 0) tl_mark(tlog, 0, 2, tl_first);
  pdl_launch_dependents();
}

// sampled slot -> 1-based rank in the partially sorted token list (O6/O7)
__device__ __forceinline__ int slot_rank(int slot, const SampleConsts& sc) {
  if (sc.fallback) return slot + 1;
  const int W1 = 2 * sc.w + 1;
  if (slot < sc.N) return slot + 1;
  if (slot < sc.N + W1) return sc.x1 - sc.w + (slot - sc.N);
  return sc.x2 - sc.w + (slot - sc.N - W1);
}

// ------------------------------------------------------------------ S4 (sampled logits)

// One CTA = SB consecutive slots of one head: slot rows come from the rank kernel's row
// map; every warp finds the contiguous runs among its 32 rows (ballot of run breaks) and
// the first lane of each run bulk-copies it (1-D TMA) into shared memory; logits are
// then computed on the tensor cores (mma.sync m16n8k16, q in the n=8 dimension, only
// column 0 live).  The CTA also emits a summary for the fit: its local max logit and the
// sums of exp(l - m_local) over its exact-head, window-1 and window-2 slots.
constexpr int SB = 64;

__global__ void __launch_bounds__(SB) sample_kernel(const __nv_bfloat16* __restrict__ q,
                                                    const __nv_bfloat16* __restrict__ Kp,
                                                    const int* __restrict__ rowmap, int n, int G, SampleConsts sc,
                                                    float* __restrict__ logits, float* __restrict__ summ, int nb,
                                                    unsigned long long* tlog) {
  __shared__ __align__(128) uint8_t rows_s[SB * 256];
  __shared__ float lg_s[SB];
  __shared__ uint64_t bar;
  __shared__ float redd[SB / 32][3];
  __shared__ float redf[SB / 32];
  const int g = blockIdx.y, u = blockIdx.z;
  const size_t ug = (size_t)u * G + g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool tl_first = blockIdx.x == 0 && g == 0 && u == 0;
  if (tid == 0) {
    tl_mark(tlog, 2, 0, tl_first);
    mbar_init(&bar, SB);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  if (tid == 0) tl_mark(tlog, 2, 1, tl_first);
  const int slot = blockIdx.x * SB + tid;
  const bool valid = slot < sc.slots;
  const int row = valid ? rowmap[ug * sc.slots + slot] : -1;
  {
    const int prev = __shfl_up_sync(0xffffffffu, row, 1);
    const bool start = row >= 0 && (lane == 0 || prev != row - 1);
    const unsigned brk = __ballot_sync(0xffffffffu, start || row < 0);
    if (start) {
      const unsigned later = brk & ~((2u << lane) - 1u);
      const int len = (later ? __ffs(later) - 1 : 32) - lane;
      mbar_arrive_expect_tx(&bar, (uint32_t)len * 256u);
      bulk_g2s(rows_s + tid * 256, Kp + ((size_t)u * n + row) * 128, (uint32_t)len * 256u, &bar);
    } else {
      mbar_arrive(&bar);
    }
  }
  // B fragment (k = dim, n = head column): only column 0 (lanes 0..3) carries q
  uint32_t qb[8][2];
  {
    const uint32_t* q32 = reinterpret_cast<const uint32_t*>(q + ug * 128);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qb[ks][0] = lane < 4 ? q32[(ks * 16 + 2 * lane) >> 1] : 0u;
      qb[ks][1] = lane < 4 ? q32[(ks * 16 + 8 + 2 * lane) >> 1] : 0u;
    }
  }
  mbar_wait(&bar, 0);
  const uint32_t sbase = smem_u32(rows_s);
#pragma unroll
  for (int gi = 0; gi < 2; ++gi) {
    const int i = (lane & 7) + ((lane >> 3) & 1) * 8;  // row of the 16-row group (ldmatrix)
    const int li = warp * 32 + gi * 16 + i;
    const int grow = __shfl_sync(0xffffffffu, row, gi * 16 + i);
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t af[4];
      ldsm_x4(af[0], af[1], af[2], af[3], sbase + li * 256 + (swz_chunk(2 * ks + (lane >> 4), grow) << 4));
      mma_bf16_16816(s, af, qb[ks][0], qb[ks][1]);
    }
    if ((lane & 3) == 0) {
      lg_s[warp * 32 + gi * 16 + (lane >> 2)] = s[0] * 0.08838834764831845f;
      lg_s[warp * 32 + gi * 16 + (lane >> 2) + 8] = s[2] * 0.08838834764831845f;
    }
  }
  __syncthreads();
  const float lg = lg_s[tid];
  if (valid) logits[ug * sc.slots + slot] = lg;
  float mx = valid ? lg : -INFINITY;
  mx = warp_max(mx);
  if (lane == 0) redf[warp] = mx;
  __syncthreads();
  float mb = redf[0];
#pragma unroll
  for (int w = 1; w < SB / 32; ++w) mb = fmaxf(mb, redf[w]);
  const float e = valid ? __expf(lg - mb) : 0.f;
  const int W1 = 2 * sc.w + 1;
  float sh = 0.f, s1 = 0.f, s2 = 0.f;
  if (sc.fallback || slot < sc.N) sh = e;
  else if (slot < sc.N + W1) s1 = e;
  else s2 = e;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sh += __shfl_xor_sync(0xffffffffu, sh, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) { redd[warp][0] = sh; redd[warp][1] = s1; redd[warp][2] = s2; }
  __syncthreads();
  if (tid == 0) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
    for (int w = 0; w < SB / 32; ++w) { a0 += redd[w][0]; a1 += redd[w][1]; a2 += redd[w][2]; }
    *reinterpret_cast<float4*>(summ + (ug * nb + blockIdx.x) * 4) = make_float4(mb, a0, a1, a2);
    tl_mark(tlog, 2, 2, tl_first);
  }
  pdl_launch_dependents();
}

// ------------------------------------------------------------------ S5-S7 from the summaries
struct FitParams {
  const float* summ;      // [units][G][nb][4]: m_b, head sum, window-1 sum, window-2 sum
  const float* logits;    // [units][G][slots]
  const int* order;
  const int* ends;
  const int* offsets;
  int n, C, G, units, nb;
  SampleConsts sc;
  double p;
  double* fit;
  float* mref;            // [units][G] log2-domain shift for the attention's merge (m log2 e)
  int* J;
  uint8_t* umask;
  int* ulist;
  int* uprefix;
  long long* unit_prefix;
  unsigned int* unit_cnt;
  unsigned long long* tlog;  // nullable debug stamps
  int need_unit_prefix;      // global attention split (units > CTAs/2): compute unit_prefix
  int tail_len;              // recent-token tail per unit (counted in unit_prefix)
  int fixed_budget;          // > 0: Quest-like fixed token budget per head (NEXT 4 baseline)
  int windows_exact;         // SPEC variant: window ranks keep their exact weights
  // sequence-sharded mode (reading 23): 0 = Alg. 1 selection; 2 = stage 1 (fit only:
  // local shift m, theta_max, E_N, W; no selection); 1 = stage 2 (the shared threshold
  // theta* from the all-reduced mass vector selects a rank prefix per head)
  int shard_mode;
  const double* crit;        // [units][G][C] (stage 1's criticalities)
  const double* gmax;        // stage 2: [units][G][2] global (m, theta_max)
  const double* gmass;       // stage 2: [units][G][1 + T] global (W, M(theta_t))
  double* local_max;         // stage 1: [units][G][2] local (m, theta_max)
  double* en_out;            // stage 1: [units][G][2] (E_N, 0) for stage 1b
};

// ------------------------------------------------------------------ S5-S7, one CTA per unit
// One warp per query head does the whole fit (Alg. 1 l.4-10) with warp-level reductions
// and no block barrier on the per-head critical path; the G heads run concurrently and
// OR their selected clusters into a shared-memory mask that the CTA compacts into the
// attention work list (S7).  Float32 arithmetic throughout: on sm_100a a dependent fp64
// exp/log costs ~170/~290 cycles against ~55 for the fp32 special-function unit, and the
// fit is one long dependency chain.  fp32 keeps every decision within the parity
// contract's 1e-5 threshold band (the sums are tree reductions of <= 4K terms).

// Warp-cooperative count of the leading falses of a monotone predicate over [0, len)
// (false ... false true ... true): 32 probes per round, 2 rounds for len <= 1024.
template <typename Pred>
__device__ __forceinline__ int warp_count_false(int len, Pred pred) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = len;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) >> 5;
    const int idx = lo + lane * step;
    const int c = __popc(__ballot_sync(0xffffffffu, idx < hi && !pred(idx)));
    const int nlo = c > 0 ? lo + (c - 1) * step + 1 : lo;
    const int nhi = lo + c * step < hi ? lo + c * step : hi;
    lo = nlo;
    hi = nhi;
  }
  const int idx = lo + lane;
  return lo + __popc(__ballot_sync(0xffffffffu, idx < hi && !pred(idx)));
}

// windows-exact variant: estimated cumulative mass at rank k > N, i.e. E_N + the fitted
// tail, corrected on the window ranks [x_w - w, x_w + w] to their exact weights (xw: the
// inclusive prefix of the exact window weights, window 1 then window 2)
__device__ __noinline__ float windows_cum(float EN, TailF tail, const float* xw, const SampleConsts sc, int k) {
  float c = EN + tail(k);
  const int W1 = 2 * sc.w + 1;
  const int lo0 = sc.x1 - sc.w, hi0 = sc.x1 + sc.w, lo1 = sc.x2 - sc.w, hi1 = sc.x2 + sc.w;
  if (k >= lo0) {
    const int kk = k < hi0 ? k : hi0;
    c += xw[kk - lo0] - (tail(kk) - tail(lo0 - 1));
  }
  if (k >= lo1) {
    const int kk = k < hi1 ? k : hi1;
    c += xw[W1 + kk - lo1] - (tail(kk) - tail(lo1 - 1));
  }
  return c;
}

constexpr int FITU_THREADS = 256;

// GEN = false: the plain Alg. 1 decode (no sharded stages, windows-exact variant, fixed
// budget or unit prefix) compiled without those paths -- the fit is a chain of single-warp
// steps, and its code arrives cold after every other layer's traffic has passed through L2
// (the smaller kernel runs ~1 us faster per layer-step)
// MODE 0: the plain decode; 1 / 2: sharded stage 2 / stage 1 alone; 3: generic (any mode
// with the windows-exact variant, a fixed budget or the global unit prefix)
template <int MODE>
__global__ void __launch_bounds__(FITU_THREADS) fit_unit_kernel(const FitParams P) {
  constexpr bool GEN = MODE == 3;
  const int shard_mode = GEN ? P.shard_mode : (MODE == 4 ? 0 : MODE);
  const int fixed_budget = GEN ? P.fixed_budget : 0;
  const bool windows_exact = GEN && P.windows_exact;
  const bool need_unit_prefix = GEN && P.need_unit_prefix;
  extern __shared__ __align__(16) uint8_t fsm[];
  __shared__ int s_J[8];
  __shared__ bool s_last;
  const int u = blockIdx.x, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int C = P.C, n = P.n, nb = P.nb, G = P.G;
  const SampleConsts sc = P.sc;
  float* sm = (float*)fsm;                           // [G][nb][4]
  int* s_off = (int*)(sm + (((size_t)G * nb * 4 + 3) & ~(size_t)3));  // [C+1]
  int* s_end = s_off + ((C + 1 + 3) & ~3);           // [G][C] (16-byte aligned for bulk copies)
  int* s_ord = s_end + (size_t)G * C;                // [G][C]
  uint8_t* mask = (uint8_t*)(s_ord + (size_t)G * C); // [C]
  // windows-exact variant: every head's window logits (slots N .. N + 2 W1), then their
  // inclusive prefix of exp(l - m) in place: [G][wx_stride] floats, 16-byte aligned
  const int W1s = 2 * sc.w + 1;
  const int wx_stride = ((2 * W1s + 3 + 3) & ~3) + 4;
  float* s_wx = windows_exact ? (float*)(((uintptr_t)(mask + C) + 15) & ~(uintptr_t)15) : nullptr;
  const bool stamp_on = P.tlog != nullptr && u == 0;
  auto stamp = [&](int i) {  // debug: CTA of unit 0 at tlog[256 + i]
    if (stamp_on && tid == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      P.tlog[256 + i] = t_;
    }
  };
  auto wstamp = [&](int i) {  // debug: warp 0 (head 0) of unit 0 at tlog[1700 + i]
    if (stamp_on && tid == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      P.tlog[1700 + i] = t_;
      P.tlog[1710 + i] = clock64();
    }
  };
  stamp(0);
  if (tid == 0) tl_mark(P.tlog, 3, 0, u == 0);
  // index data (not produced by the previous kernels): before the dependency wait
  for (int i = tid; i <= C; i += nt) s_off[i] = P.offsets[(size_t)u * (C + 1) + i];
  __shared__ uint64_t sbar, obar;
  const size_t ub = (size_t)u * G;
  const bool bulk_ok = ((ub * C) % 4 == 0) && (((size_t)G * C) % 4 == 0);
  if (tid == 0) {
    mbar_init(&sbar, 1);
    mbar_init(&obar, 1);
    fence_barrier_init();
  }
  for (int i = tid; i < C; i += nt) mask[i] = 0;
  __syncthreads();
  // The unit's order / end ranks (score_rank) are complete before the dependency wait:
  // this grid starts only after the sample kernel passed ITS wait on score_rank.  Stage
  // them now; only the sample kernel's summaries remain for after the wait.
  if (tid == 0 && bulk_ok) {
    const uint32_t be = (uint32_t)G * C * 4;
    mbar_arrive_expect_tx(&obar, 2 * be);
    bulk_g2s(s_end, P.ends + ub * C, be, &obar);
    bulk_g2s(s_ord, P.order + ub * C, be, &obar);
  }
  if (!bulk_ok)
    for (int i = tid; i < G * C; i += nt) {
      s_end[i] = P.ends[ub * C + i];
      s_ord[i] = P.order[ub * C + i];
    }
  if (bulk_ok) mbar_wait(&obar, 0);
  __syncthreads();
  {
    pdl_wait();
    stamp(1);
    if (tid == 0) tl_mark(P.tlog, 3, 1, u == 0);
    // stage the sample kernel's summaries (one round trip; + the window logits of every
    // head for the windows-exact variant, from the 16-byte aligned slot at or below N);
    // sharded stage 2 needs none (its rule reads the mass vector)
    if (tid == 0 && shard_mode != 1) {
      const uint32_t bs = (uint32_t)G * nb * 16;
      uint32_t lb = 0;
      if (s_wx)
        for (int g = 0; g < G; ++g) {
          const size_t st = (ub + g) * sc.slots + sc.N, al = st & ~(size_t)3;
          lb += (uint32_t)((((st - al) + 2 * W1s) * 4 + 15) & ~(size_t)15);
        }
      mbar_arrive_expect_tx(&sbar, bs + lb);
      bulk_g2s(sm, P.summ + ub * nb * 4, bs, &sbar);
      if (s_wx)
        for (int g = 0; g < G; ++g) {
          const size_t st = (ub + g) * sc.slots + sc.N, al = st & ~(size_t)3;
          bulk_g2s(s_wx + (size_t)g * wx_stride, P.logits + al,
                   (uint32_t)((((st - al) + 2 * W1s) * 4 + 15) & ~(size_t)15), &sbar);
        }
    }
    if (shard_mode != 1) mbar_wait(&sbar, 0);
    __syncthreads();
    stamp(2);
    if (stamp_on && tid == 0) P.tlog[1709] = clock64();
  }
  if constexpr (MODE == 4) {
    // paired plain decode (G <= 4, C <= 1024): warp 2g computes head g's W while warp 2g + 1
    // evaluates the first round of the J search (the probes need a, b, E_N, not W) and then
    // finishes the selection -- the W evaluation leaves the head's critical path
    __shared__ float s_W[8];
    if (warp < 2 * G) {
      const int g = warp >> 1, role = warp & 1;
      const float* sg = sm + (size_t)g * nb * 4;
      float mf = -INFINITY;
      for (int b = lane; b < nb; b += 32) mf = fmaxf(mf, sg[b * 4]);
      const float m = warp_max(mf);
      float eh = 0.f, e1 = 0.f, e2 = 0.f;
      for (int b = lane; b < nb; b += 32) {
        const float4 v = *reinterpret_cast<const float4*>(sg + b * 4);
        const float f = __expf(v.x - m);
        eh = fmaf(v.y, f, eh);
        e1 = fmaf(v.z, f, e1);
        e2 = fmaf(v.w, f, e2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        eh += __shfl_xor_sync(0xffffffffu, eh, o);
        e1 += __shfl_xor_sync(0xffffffffu, e1, o);
        e2 += __shfl_xor_sync(0xffffffffu, e2, o);
      }
      const float EN = eh;
      float a = 0.f, b = 0.f, mu1 = 0.f, mu2 = 0.f;
      TailF tail = {0.f, 0.f, 1, 0};
      if (!sc.fallback) {
        const float W1 = (float)(2 * sc.w + 1);
        mu1 = e1 / W1;
        mu2 = e2 / W1;
        const float x1 = (float)sc.x1, x2 = (float)sc.x2;
        a = (mu1 - mu2) * (x1 * x2 / (x2 - x1));  // O8 / Alg. 1 l.4
        b = mu1 - a / x1;
        tail = make_tail_f(a, b, sc.N, n);
      }
      if (role == 0) {
        const float W = sc.fallback ? EN : EN + tail(n);
        if (lane == 0) s_W[g] = W;
        asm volatile("bar.arrive %0, 64;" ::"r"(2 + g) : "memory");
      } else {
        const int* eg = s_end + (size_t)g * C;
        // round 1 of the search over the cluster ends (see warp_count_false): its probes
        const int step = (C + 31) >> 5;
        const int idx1 = lane * step;
        bool past = false;
        float v1 = -INFINITY;
        if (idx1 < C) {
          const int e = eg[idx1];
          past = e > sc.N;
          if (past && !sc.fallback) v1 = EN + tail(e);
        }
        asm volatile("bar.sync %0, 64;" ::"r"(2 + g) : "memory");
        const float W = s_W[g];
        int J = C;  // p >= 1: every cluster (reading 15)
        if (P.p < 1.0) {
          const float target = (float)P.p * W;
          if (EN >= target) {
            // the crossing lies inside the exact head: the crossing block of the per-block
            // prefix, then the slot inside it (one global round trip)
            const int nex = sc.fallback ? n : sc.N;
            const int nbh = (nex + SB - 1) / SB;
            float carry = 0.f, before = 0.f;
            int bs = nbh - 1;
            for (int b0 = 0; b0 < nbh; b0 += 32) {
              const int bb = b0 + lane;
              const float vo = bb < nbh ? sg[bb * 4 + 1] * __expf(sg[bb * 4] - m) : 0.f;
              float v = vo;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const float x = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += x;
              }
              const unsigned hit = __ballot_sync(0xffffffffu, bb < nbh && carry + v >= target);
              if (hit) {
                const int hl = __ffs(hit) - 1;
                bs = b0 + hl;
                before = carry + __shfl_sync(0xffffffffu, v, hl) - __shfl_sync(0xffffffffu, vo, hl);
                break;
              }
              carry += __shfl_sync(0xffffffffu, v, 31);
              before = carry;
            }
            const int s0 = bs * SB, s1 = min(nex, s0 + SB);
            constexpr int PER = SB / 32;
            float w[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
              const int s = s0 + PER * lane + k;
              w[k] = s < s1 ? __expf(__ldcg(P.logits + (ub + g) * sc.slots + s) - m) : 0.f;
            }
#pragma unroll
            for (int k = 1; k < PER; ++k) w[k] += w[k - 1];
            float v = w[PER - 1];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const float x = __shfl_up_sync(0xffffffffu, v, o);
              if (lane >= o) v += x;
            }
            const float excl = before + v - w[PER - 1];
            int kl = PER;
#pragma unroll
            for (int k = PER - 1; k >= 0; --k)
              if (s0 + PER * lane + k < s1 && excl + w[k] >= target) kl = k;
            const unsigned hit = __ballot_sync(0xffffffffu, kl < PER);
            const int hl = hit ? __ffs(hit) - 1 : 31;
            const int kls = __shfl_sync(0xffffffffu, kl, hl);
            const int kstar = hit ? s0 + PER * hl + kls + 1 : s1;
            J = 1 + warp_count_false(C - 1, [&](int r) { return eg[r] >= kstar; });
          } else {
            // past the head: the first cluster end whose estimated mass reaches the target
            const int c1 = __popc(__ballot_sync(0xffffffffu, idx1 < C && !(past && v1 >= target)));
            const int lo = c1 > 0 ? (c1 - 1) * step + 1 : 0, hi = min(c1 * step, C);
            const int idx = lo + lane;
            const bool nf = idx < hi && !(eg[idx] > sc.N && EN + tail(eg[idx]) >= target);
            const int r = lo + __popc(__ballot_sync(0xffffffffu, nf));
            J = r < C ? r + 1 : C;
          }
        }
        if (lane == 0) {
          s_J[g] = J;
          P.J[ub + g] = J;
          double* f = P.fit + (ub + g) * 6;
          f[0] = a; f[1] = b; f[2] = m; f[3] = W; f[4] = mu1; f[5] = mu2;
          P.mref[ub + g] = m * 1.4426950408889634f;
        }
        const int* ord = s_ord + (size_t)g * C;
        __syncwarp();
        for (int r = lane; r < J; r += 32) {
          const int cid = ord[r];
          if (s_off[cid + 1] > s_off[cid]) mask[cid] = 1;
        }
      }
    }
  } else {
  if (warp < G && shard_mode == 1) {
    // sharded stage 2 (reading 23): theta* = the largest grid point theta_t whose
    // all-reduced mass reaches p W (none: every cluster); the head selects the rank prefix
    // of clusters with crit / sqrt(d) >= theta* (the order is by descending crit)
    const int g = warp;
    const double* gm = P.gmass + (ub + g) * (1 + TACTIC_SHARD_GRID_T);
    const double thmax = P.gmax[(ub + g) * 2 + 1], Wt = gm[0];
    int tmin = TACTIC_SHARD_GRID_T + 1;
    if (P.p < 1.0)
      for (int t0 = 1; t0 <= TACTIC_SHARD_GRID_T; t0 += 32) {
        const unsigned hit = __ballot_sync(0xffffffffu, t0 + lane <= TACTIC_SHARD_GRID_T && gm[t0 + lane] >= P.p * Wt);
        if (hit) {
          tmin = t0 + __ffs(hit) - 1;
          break;
        }
      }
    const double thstar = tmin <= TACTIC_SHARD_GRID_T ? thmax - (double)tmin * TACTIC_SHARD_GRID_STEP : -INFINITY;
    const double* cr = P.crit + (ub + g) * C;
    const int* ord = s_ord + (size_t)g * C;
    const double isd = 1.0 / sqrt(128.0);
    const int J = warp_count_false(C, [&](int r) { return cr[ord[r]] * isd < thstar; });
    if (lane == 0) {
      P.J[ub + g] = J;
      double* f = P.fit + (ub + g) * 6;
      f[0] = thstar; f[1] = Wt; f[2] = P.gmax[(ub + g) * 2]; f[3] = thmax; f[4] = 0; f[5] = 0;
      P.mref[ub + g] = (float)(P.gmax[(ub + g) * 2] * 1.4426950408889634);
    }
    __syncwarp();
    for (int r = lane; r < J; r += 32) {
      const int cid = ord[r];
      if (s_off[cid + 1] > s_off[cid]) mask[cid] = 1;
    }
  } else if (warp < G) {
    const int g = warp;
    const float* sg = sm + (size_t)g * nb * 4;
    // common shift m = max of the block maxima (reading 13), then the three region sums
    float mf = -INFINITY;
    for (int b = lane; b < nb; b += 32) mf = fmaxf(mf, sg[b * 4]);
    const float m = warp_max(mf);
    float eh = 0.f, e1 = 0.f, e2 = 0.f;
    for (int b = lane; b < nb; b += 32) {
      const float4 v = *reinterpret_cast<const float4*>(sg + b * 4);
      const float f = __expf(v.x - m);
      eh = fmaf(v.y, f, eh);
      e1 = fmaf(v.z, f, e1);
      e2 = fmaf(v.w, f, e2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // three interleaved butterflies
      eh += __shfl_xor_sync(0xffffffffu, eh, o);
      e1 += __shfl_xor_sync(0xffffffffu, e1, o);
      e2 += __shfl_xor_sync(0xffffffffu, e2, o);
    }
    const float EN = eh;
    wstamp(0);
    float a = 0.f, b = 0.f, mu1 = 0.f, mu2 = 0.f, W = EN;
    TailF tail = {0.f, 0.f, 1, 0};
    if (!sc.fallback) {
      const float W1 = (float)(2 * sc.w + 1);
      mu1 = e1 / W1;
      mu2 = e2 / W1;
      const float x1 = (float)sc.x1, x2 = (float)sc.x2;
      a = (mu1 - mu2) * (x1 * x2 / (x2 - x1));  // O8 / Alg. 1 l.4
      b = mu1 - a / x1;
      tail = make_tail_f(a, b, sc.N, n);
      W = EN + tail(n);
    }
    // windows-exact variant ("exact values taking precedence"): the window
    // ranks [lo_w, hi_w] carry their exact weights; xw = in-place inclusive prefix of
    // exp(l - m) over the head's window slots (window 1 then window 2)
    float* xw = nullptr;
    if (s_wx && !sc.fallback) {
      xw = s_wx + (size_t)g * wx_stride + (((ub + g) * sc.slots + sc.N) & 3);
      for (int wi = 0; wi < 2; ++wi) {
        float carry = 0.f;
        for (int i0 = 0; i0 < W1s; i0 += 32) {
          const int i = wi * W1s + i0 + lane;
          float v = i0 + lane < W1s ? __expf(xw[i] - m) : 0.f;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const float x = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += x;
          }
          if (i0 + lane < W1s) xw[i] = carry + v;
          carry += __shfl_sync(0xffffffffu, v, 31);
        }
      }
      __syncwarp();
      W = windows_cum(EN, tail, xw, sc, n);
    }
    wstamp(1);
    if (shard_mode == 2) {  // sharded stage 1: the local fit only (stage 1b uses it)
      if (lane == 0) {
        double* f = P.fit + (ub + g) * 6;
        f[0] = a; f[1] = b; f[2] = m; f[3] = W; f[4] = mu1; f[5] = mu2;
        P.en_out[(ub + g) * 2] = EN;
        P.en_out[(ub + g) * 2 + 1] = 0.0;
        P.local_max[(ub + g) * 2] = m;
        P.local_max[(ub + g) * 2 + 1] = P.crit[(ub + g) * C + s_ord[(size_t)g * C]] / sqrt(128.0);
      }
    } else {  // the selection (stage 1 selects nothing)
      int J = C;  // p >= 1: every cluster (reading 15)
      if (fixed_budget > 0) {
        // Quest-like baseline: clusters in criticality order until the head
        // holds fixed_budget tokens (rounded up to the cluster end, as reading 14)
        const int* eg = s_end + (size_t)g * C;
        J = 1 + warp_count_false(C - 1, [&](int r) { return eg[r] >= fixed_budget; });
      } else if (P.p < 1.0) {
        const float target = (float)P.p * W;
        const int* eg = s_end + (size_t)g * C;
        if (EN >= target) {
          // the crossing lies inside the exact head (slots 0..nex-1 = ranks 1..nex): the
          // block of SB slots that crosses, then the slot inside it (one global round trip)
          const int nex = sc.fallback ? n : sc.N;
          const int nbh = (nex + SB - 1) / SB;
          float carry = 0.f, before = 0.f;
          int bs = nbh - 1;
          for (int b0 = 0; b0 < nbh; b0 += 32) {
            const int bb = b0 + lane;
            const float vo = bb < nbh ? sg[bb * 4 + 1] * __expf(sg[bb * 4] - m) : 0.f;
            float v = vo;
  #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const float x = __shfl_up_sync(0xffffffffu, v, o);
              if (lane >= o) v += x;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, bb < nbh && carry + v >= target);
            if (hit) {
              const int hl = __ffs(hit) - 1;
              bs = b0 + hl;
              before = carry + __shfl_sync(0xffffffffu, v, hl) - __shfl_sync(0xffffffffu, vo, hl);
              break;
            }
            carry += __shfl_sync(0xffffffffu, v, 31);
            before = carry;
          }
          const int s0 = bs * SB, s1 = min(nex, s0 + SB);
          constexpr int PER = SB / 32;  // consecutive slots per lane
          float w[PER];
  #pragma unroll
          for (int k = 0; k < PER; ++k) {
            const int s = s0 + PER * lane + k;
            w[k] = s < s1 ? __expf(__ldcg(P.logits + (ub + g) * sc.slots + s) - m) : 0.f;
          }
  #pragma unroll
          for (int k = 1; k < PER; ++k) w[k] += w[k - 1];
          float v = w[PER - 1];
  #pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const float x = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += x;
          }
          const float excl = before + v - w[PER - 1];
          int kl = PER;
  #pragma unroll
          for (int k = PER - 1; k >= 0; --k)
            if (s0 + PER * lane + k < s1 && excl + w[k] >= target) kl = k;
          const unsigned hit = __ballot_sync(0xffffffffu, kl < PER);
          const int hl = hit ? __ffs(hit) - 1 : 31;
          const int kls = __shfl_sync(0xffffffffu, kl, hl);
          // k* = the 1-based rank of the crossing slot (rounding guard: the block's last slot)
          const int kstar = hit ? s0 + PER * hl + kls + 1 : s1;
          J = 1 + warp_count_false(C - 1, [&](int r) { return eg[r] >= kstar; });
        } else {
          // past the head: cum(e_r) = EN + tail(e_r) at the cluster ends; the first cluster
          // whose end reaches the target (ends are non-decreasing in rank)
          const int r = xw ? warp_count_false(C, [&](int r) { return eg[r] > sc.N && windows_cum(EN, tail, xw, sc, eg[r]) >= target; })
                           : warp_count_false(C, [&](int r) { return eg[r] > sc.N && EN + tail(eg[r]) >= target; });
          J = r < C ? r + 1 : C;
        }
      }
      wstamp(3);
      if (lane == 0) {
        s_J[g] = J;
        P.J[ub + g] = J;
        double* f = P.fit + (ub + g) * 6;
        f[0] = a; f[1] = b; f[2] = m; f[3] = W; f[4] = mu1; f[5] = mu2;
        P.mref[ub + g] = m * 1.4426950408889634f;
      }
      // mark this head's selected non-empty clusters (the OR over heads is the GQA union)
      const int* ord = s_ord + (size_t)g * C;
      __syncwarp();
      for (int r = lane; r < J; r += 32) {
        const int cid = ord[r];
        if (s_off[cid + 1] > s_off[cid]) mask[cid] = 1;
      }
    }
    wstamp(4);
  }
  }
  __syncthreads();
  stamp(3);
  if (shard_mode == 2) {
    pdl_launch_dependents();
    return;
  }
  // ---- S7: compact the union (cluster-id order) into the work list.  Thread t owns a
  // contiguous cluster chunk; one packed (tokens << 20 | clusters) block scan places it.
  {
    __shared__ unsigned long long w_sum[FITU_THREADS / 32];
    const int nw = nt >> 5;
    const int per = (C + nt - 1) / nt;
    const int j0 = tid * per, j1 = min(C, j0 + per);
    unsigned long long loc = 0;
    // four clusters per thread (C = 4 x threads): the thread's mask bytes and offsets as
    // one 32-bit and one 16-byte load, kept in registers for the second pass
    const bool quad = per == 4 && j1 - j0 == 4 && (C & 3) == 0;
    uint32_t q_mk = 0;
    int4 q_off = make_int4(0, 0, 0, 0);
    int q_end = 0;
    if (quad) {
      q_mk = *reinterpret_cast<const uint32_t*>(mask + j0);
      q_off = *reinterpret_cast<const int4*>(s_off + j0);
      q_end = s_off[j0 + 4];
      const int o[5] = {q_off.x, q_off.y, q_off.z, q_off.w, q_end};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((q_mk >> (8 * k)) & 0xFFu) loc += ((unsigned long long)(o[k + 1] - o[k]) << 20) | 1ull;
    } else {
      for (int j = j0; j < j1; ++j)
        if (mask[j]) loc += ((unsigned long long)(s_off[j + 1] - s_off[j]) << 20) | 1ull;
    }
    unsigned long long incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    if (lane == 31) w_sum[warp] = incl;
    __syncthreads();
    // the warp totals: lane w holds warp w's, one shuffle scan gives this warp's base
    const unsigned long long ws = lane < nw ? w_sum[lane] : 0ull;
    unsigned long long wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long x = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += x;
    }
    const unsigned long long base = incl - loc + __shfl_sync(0xffffffffu, wi - ws, warp);
    const unsigned long long tot = __shfl_sync(0xffffffffu, wi, 31);
    int cb = (int)(base & 0xFFFFFull), tb = (int)(base >> 20);
    int* ul = P.ulist + (size_t)u * C;
    int* up = P.uprefix + (size_t)u * (C + 1);
    uint8_t* um = P.umask + (size_t)u * C;
    if (quad) {
      *reinterpret_cast<uint32_t*>(um + j0) = q_mk;
      const int o[5] = {q_off.x, q_off.y, q_off.z, q_off.w, q_end};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((q_mk >> (8 * k)) & 0xFFu) {
          ul[cb] = o[k];
          up[cb] = tb;
          ++cb;
          tb += o[k + 1] - o[k];
        }
    } else {
      for (int j = j0; j < j1; ++j) {
        const uint8_t mk = mask[j];
        um[j] = mk;
        if (mk) {
          ul[cb] = s_off[j];
          up[cb] = tb;
          ++cb;
          tb += s_off[j + 1] - s_off[j];
        }
      }
    }
    // entries past the union: total tokens (keeps the prefix monotone for searches)
    const int ctot = (int)(tot & 0xFFFFFull), ttot = (int)(tot >> 20);
    for (int k = ctot + tid; k <= C; k += nt) {
      up[k] = ttot;
      if (k < C) ul[k] = 0;
    }
  }
  stamp(4);
  // the unit-aligned attention split reads only the per-unit totals (uprefix[u][C]); the
  // global split needs unit_prefix, computed by the last CTA to finish
  if (!need_unit_prefix) {
    if (tid == 0) tl_mark(P.tlog, 3, 2, u == 0);
    return;
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(P.unit_cnt, 1u);
    s_last = (prev == (unsigned)P.units - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    const int units = P.units;
    const int per = (units + nt - 1) / nt;
    const int b0 = tid * per;
    long long loc = 0;
    for (int v = b0; v < b0 + per && v < units; ++v) loc += __ldcg(P.uprefix + (size_t)v * (C + 1) + C) + P.tail_len;
    __shared__ long long s_tot;  // block_exclusive_scan writes the total from one thread
    long long run = block_exclusive_scan<long long>(loc, (long long*)fsm, &s_tot);
    for (int v = b0; v < b0 + per && v < units; ++v) {
      P.unit_prefix[v] = run;
      run += __ldcg(P.uprefix + (size_t)v * (C + 1) + C) + P.tail_len;
    }
    if (tid == 0) {
      P.unit_prefix[units] = s_tot;
      *P.unit_cnt = 0u;
    }
  }
  if (tid == 0) tl_mark(P.tlog, 3, 2, u == 0);
}

// ------------------------------------------------------------------ sharded stage 1b
// One CTA per (unit, head) (reading 23): the shard's estimated mass of the clusters above
// every grid point theta_t = theta_max - t / 16 (t = 1..T) of the GLOBAL frame, re-expressed
// with the global shift: M_s(theta_t) = cum(e_{r_t}) exp(m_s - m) where r_t = #clusters
// with crit / sqrt(d) >= theta_t (a rank prefix) and cum(e) = the exact prefix for e <= N,
// E_N + tail(e) beyond (the stage-1 fit).  The criticalities in rank order, the end ranks
// and the exact head prefix are staged in shared memory once (three round trips), so each
// grid point is a binary search in shared memory.
constexpr int S1B_THREADS = 256;
__global__ void __launch_bounds__(S1B_THREADS) stage1b_kernel(const double* __restrict__ crit,
                                                              const int* __restrict__ order,
                                                              const int* __restrict__ ends,
                                                              const float* __restrict__ logits,
                                                              const double* __restrict__ fit,
                                                              const double* __restrict__ en,
                                                              const double* __restrict__ gmax, int C, int n,
                                                              SampleConsts sc, double* __restrict__ mass) {
  extern __shared__ __align__(16) uint8_t s1b[];
  __shared__ float red[S1B_THREADS / 32];
  const size_t ug = blockIdx.x;
  const int tid = threadIdx.x;
  double* th = (double*)s1b;             // [C] theta in rank order
  int* se = (int*)(th + C);              // [C] end ranks
  const int nex = sc.fallback ? n : sc.N;
  float* hp = (float*)(se + C);          // [nex] inclusive exact-head prefix (local frame)
  const double ms = fit[ug * 6 + 2], Ws = fit[ug * 6 + 3];
  const float a = (float)fit[ug * 6 + 0], b = (float)fit[ug * 6 + 1];
  const float EN = (float)en[ug * 2];
  const double mg = gmax[ug * 2], thmax = gmax[ug * 2 + 1];
  const double f = exp(ms - mg);
  const double isd = 1.0 / sqrt(128.0);
#pragma unroll 4
  for (int r = tid; r < C; r += S1B_THREADS) {
    th[r] = crit[ug * C + __ldcg(order + ug * C + r)] * isd;
    se[r] = __ldcg(ends + ug * C + r);
  }
  // exact head weights exp(l - m_s) of ranks 1..nex: coalesced loads into shared memory,
  // then the inclusive prefix over contiguous per-thread chunks
  const float* lg = logits + ug * sc.slots;
  const float msf = (float)ms;
#pragma unroll 4
  for (int k = tid; k < nex; k += S1B_THREADS) hp[k] = __expf(__ldcg(lg + k) - msf);
  __syncthreads();
  const int per = (nex + S1B_THREADS - 1) / S1B_THREADS, k0 = tid * per, k1 = min(nex, k0 + per);
  float loc = 0.f;
  for (int k = k0; k < k1; ++k) loc += hp[k];
  float inc = loc;
  const int lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  if (lane == 31) red[w] = inc;
  __syncthreads();
  float run = inc - loc;
  for (int i = 0; i < w; ++i) run += red[i];
  for (int k = k0; k < k1; ++k) {
    run += hp[k];
    hp[k] = run;
  }
  __syncthreads();
  TailF tail = {0.f, 0.f, 1, 0};
  if (!sc.fallback) tail = make_tail_f(a, b, sc.N, n);
  double* out = mass + ug * (1 + TACTIC_SHARD_GRID_T);
  for (int t = tid; t <= TACTIC_SHARD_GRID_T; t += S1B_THREADS) {
    if (t == 0) {
      out[0] = Ws * f;
      continue;
    }
    const double tht = thmax - (double)t * TACTIC_SHARD_GRID_STEP;
    int lo = 0, hi = C;  // r_t: clusters (a prefix of the order) with theta >= tht
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (th[mid] >= tht) lo = mid + 1;
      else hi = mid;
    }
    double cum = 0.0;
    if (lo > 0) {
      const int e = se[lo - 1];
      cum = e <= 0 ? 0.0 : (e <= nex ? (double)hp[e - 1] : (double)(EN + tail(e)));
    }
    out[t] = cum * f;
  }
}

size_t stage1b_smem_bytes(const tactic_index_s* x) {
  const int nex = x->sc.fallback ? x->n : x->sc.N;
  return (size_t)x->C * 12 + (size_t)(nex > 0 ? nex : 1) * 4 + 16;
}

// ------------------------------------------------------------------ launchers
static cudaLaunchConfig_t make_cfg(dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                                   cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  return cfg;
}

cudaError_t launch_score(const SelArgs& a, cudaStream_t s, bool pdl) { return launch_score_all(a.q, a.idx, s, pdl); }

cudaError_t launch_score_all(const __nv_bfloat16* q, tactic_index_s* x, cudaStream_t s, bool pdl) {
  struct { const __nv_bfloat16* q; } a = {q};
  cudaLaunchAttribute attr[1];
  const int per_block = 8 * (32 / x->G);
  auto cfg = make_cfg(dim3((x->C + per_block - 1) / per_block, x->units), dim3(256), 0, s, pdl, attr);
  switch (x->G) {
    case 1: return cudaLaunchKernelEx(&cfg, score_kernel<1>, a.q, (const float*)x->cent, x->C, x->crit, x->tlog);
    case 2: return cudaLaunchKernelEx(&cfg, score_kernel<2>, a.q, (const float*)x->cent, x->C, x->crit, x->tlog);
    case 4: return cudaLaunchKernelEx(&cfg, score_kernel<4>, a.q, (const float*)x->cent, x->C, x->crit, x->tlog);
    case 8: return cudaLaunchKernelEx(&cfg, score_kernel<8>, a.q, (const float*)x->cent, x->C, x->crit, x->tlog);
  }
  return cudaErrorInvalidValue;
}

static cudaError_t ensure_smem(const void* fn, size_t smem) {
  // static smem counts against the 48 KB default too
  return smem > 40 * 1024 ? func_smem_optin(fn, smem) : cudaSuccess;
}

int sample_blocks(int slots) { return (slots + SB - 1) / SB; }

cudaError_t launch_sample(const SelArgs& a, cudaStream_t s, bool pdl) {
  tactic_index_s* x = a.idx;
  const int nb = sample_blocks(x->sc.slots);
  cudaLaunchAttribute attr[1];
  auto cfg = make_cfg(dim3(nb, x->G, x->units), dim3(SB), 0, s, pdl, attr);
  return cudaLaunchKernelEx(&cfg, sample_kernel, a.q, (const __nv_bfloat16*)x->Kp, (const int*)x->rowmap, x->n,
                            x->G, x->sc, x->logits, x->summ, nb, x->tlog);
}

size_t fit_smem_bytes(const tactic_index_s* x, bool windows_exact) {
  const int nb = sample_blocks(x->sc.slots);
  return (size_t)x->G * nb * 16 + 16 + (size_t)(x->C + 4) * 4 + (size_t)2 * x->G * x->C * 4 + (size_t)x->C + 64 +
         (windows_exact ? (size_t)x->G * ((((size_t)2 * (2 * x->sc.w + 1) + 6) & ~(size_t)3) + 4) * 4 + 16 : 0);
}

cudaError_t launch_fit(const SelArgs& a, cudaStream_t s, bool pdl) {
  tactic_index_s* x = a.idx;
  FitParams P = {};
  P.summ = x->summ;
  P.logits = x->logits;
  P.order = x->order;
  P.ends = x->ends;
  P.offsets = x->offsets;
  P.n = x->n;
  P.C = x->C;
  P.G = x->G;
  P.units = x->units;
  P.nb = sample_blocks(x->sc.slots);
  P.sc = x->sc;
  P.p = a.p;
  P.fit = x->fit;
  P.mref = x->mref;
  P.J = x->J;
  P.umask = x->umask;
  P.ulist = x->union_list;
  P.uprefix = x->union_prefix;
  P.unit_prefix = x->unit_prefix;
  P.unit_cnt = x->counter;
  P.tlog = x->tlog;
  P.need_unit_prefix = !unit_split_ok(x->units, x->num_ctas);
  P.tail_len = x->tail_len;
  P.fixed_budget = x->fixed_budget;
  P.windows_exact = (x->options & 1u) ? 1 : 0;
  P.shard_mode = a.mode;  // 0 Alg. 1, 1 sharded stage 2, 2 sharded stage 1
  P.crit = x->crit;
  P.gmax = a.gmax;
  P.gmass = a.gmass;
  P.local_max = a.local_max;
  P.en_out = x->stage;
  cudaLaunchAttribute attr[1];
  const size_t smem = fit_smem_bytes(x, P.windows_exact != 0);
  int mode = (P.windows_exact || P.fixed_budget > 0 || P.need_unit_prefix) ? 3 : P.shard_mode;
  static const bool no_pair = getenv("TACTIC_FIT_UNPAIRED") != nullptr;
  if (mode == 0 && x->G <= 4 && x->C <= 1024 && !no_pair) mode = 4;  // paired W / search warps
  void (*kern)(const FitParams) = mode == 0 ? fit_unit_kernel<0> : mode == 1 ? fit_unit_kernel<1>
                                : mode == 2 ? fit_unit_kernel<2> : mode == 3 ? fit_unit_kernel<3>
                                : fit_unit_kernel<4>;
  cudaError_t e = ensure_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  auto cfg = make_cfg(dim3(x->units), dim3(FITU_THREADS), smem, s, pdl, attr);
  return cudaLaunchKernelEx(&cfg, kern, P);
}

cudaError_t launch_stage1b(const SelArgs& a, cudaStream_t s) {
  tactic_index_s* x = a.idx;
  const size_t smem = stage1b_smem_bytes(x);
  cudaError_t e = ensure_smem((const void*)stage1b_kernel, smem);
  if (e != cudaSuccess) return e;
  stage1b_kernel<<<x->units * x->G, S1B_THREADS, smem, s>>>(x->crit, x->order, x->ends, x->logits, x->fit, x->stage,
                                                             a.gmax, x->C, x->n, x->sc, a.mass_out);
  return cudaGetLastError();
}

}  // namespace tactic
