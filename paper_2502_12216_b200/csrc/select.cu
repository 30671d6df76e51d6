// select.cu -- decode-time selection S1-S7 (§4.3-§4.6, App. B Alg. 1).
//
//  score_kernel   S1  crit[u][g][j] = q_g . c_j in float64 (products of a
//                     bf16 query and a float32 centroid are exact in fp64, so only the
//                     summation order differs from the oracle).
//  sort_kernel    S2  bitonic sort of (-crit, j) per (unit, head) in shared memory;
//                 S3  inclusive scan of cluster sizes in rank order -> end ranks e_r.
//  sample_kernel  S4  exact logits q.k/sqrt(d) of the sampled ranks: the first N ranks
//                     and two windows of 2w+1 ranks around x1, x2 (Alg. 1 l.4,
//                     readings 8-11); rank -> row through e_r, order, offsets.
//  select_kernel  S4-S6 shift m, exact head weights + prefix, window means, two-point
//                     fit y = a/x + b, estimated total W, minimal k with
//                     cum(k) >= p W (Alg. 1 l.10) at cluster granularity
//                     (reading 14); S7 union over the G heads, compacted work
//                     list, and a global token prefix over units (sub-requests)
//                     computed by the last block to finish.
// The clamp-aware tail sum  sum_{i=N+1}^{k} max(0, a/i + b)  uses harmonic numbers
// from the asymptotic digamma series (exact sums below 20) instead of a table.
#include <cuda_bf16.h>
#include <float.h>
#include <limits.h>

#include "common.cuh"
#include "internal.h"

namespace tactic {

constexpr int SEL_THREADS = 512;

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ unsigned long long desc_key(double x) {
  if (x == 0.0) x = 0.0;  // -0 == +0
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  u = (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);  // ascending order
  return ~u;                                                           // descending
}

__device__ double harmonic(long long k) {
  if (k <= 0) return 0.0;
  if (k < 20) {
    double s = 0.0;
    for (long long i = k; i >= 1; --i) s += 1.0 / (double)i;
    return s;
  }
  const double x = (double)k, x2 = 1.0 / (x * x);
  return log(x) + 0.57721566490153286061 + 0.5 / x -
         x2 * (1.0 / 12.0 - x2 * (1.0 / 120.0 - x2 * (1.0 / 252.0 - x2 * (1.0 / 240.0 - x2 * (1.0 / 132.0)))));
}

// sum_{i=N+1}^{k} max(0, a/i + b)
__device__ double tail_mass(double a, double b, long long N, long long k) {
  if (k <= N) return 0.0;
  if (a >= 0.0 && b >= 0.0) return a * (harmonic(k) - harmonic(N)) + b * (double)(k - N);
  if (a <= 0.0 && b <= 0.0) return 0.0;
  if (a > 0.0) {  // b < 0: positive while i < a/(-b)
    const double t = a / (-b);
    long long top = t >= 9.0e15 ? k : (long long)floor(t);
    if (top > k) top = k;
    while (top < k && a / (double)(top + 1) + b > 0.0) ++top;
    while (top > N && !(a / (double)top + b > 0.0)) --top;
    if (top <= N) return 0.0;
    return a * (harmonic(top) - harmonic(N)) + b * (double)(top - N);
  }
  // a < 0, b > 0: positive once i > (-a)/b
  const double t = (-a) / b;
  long long lo = t >= 9.0e15 ? k + 1 : (long long)floor(t) + 1;
  if (lo < N + 1) lo = N + 1;
  while (lo > N + 1 && a / (double)(lo - 1) + b > 0.0) --lo;
  while (lo <= k && !(a / (double)lo + b > 0.0)) ++lo;
  if (lo > k) return 0.0;
  return a * (harmonic(k) - harmonic(lo - 1)) + b * (double)(k - lo + 1);
}

template <typename T> __device__ __forceinline__ T lowest();
template <> __device__ __forceinline__ float lowest<float>() { return -INFINITY; }
template <> __device__ __forceinline__ double lowest<double>() { return -INFINITY; }
template <> __device__ __forceinline__ int lowest<int>() { return INT_MIN; }

template <typename T>
__device__ T block_reduce(T v, T* red, bool is_max) {
  const T ident = is_max ? lowest<T>() : (T)0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T x = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? (x > v ? x : v) : v + x;
  }
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < nw ? red[lane] : ident;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      T x = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? (x > v ? x : v) : v + x;
    }
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  T r = red[0];
  __syncthreads();
  return r;
}

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

// smallest k in [lo, hi] with pred(k) true; pred(hi) must hold; pred monotone.
template <typename Pred>
__device__ long long block_lower_bound(long long lo, long long hi, Pred pred, long long* sh) {
  while (lo < hi) {
    const long long cnt = hi - lo + 1;
    const long long step = (cnt + blockDim.x - 1) / blockDim.x;
    const long long k = lo + (long long)threadIdx.x * step;
    if (threadIdx.x == 0) sh[0] = LLONG_MAX;
    __syncthreads();
    if (k <= hi && pred(k)) atomicMin((unsigned long long*)sh, (unsigned long long)threadIdx.x);
    __syncthreads();
    const long long t = sh[0];
    __syncthreads();
    if (t == LLONG_MAX) return hi;  // unreachable when pred(hi) holds (kept for safety)
    const long long nhi = lo + t * step;
    const long long nlo = t > 0 ? lo + (t - 1) * step + 1 : lo;
    lo = nlo;
    hi = nhi < hi ? nhi : hi;
    if (step == 1) return hi;
  }
  return lo;
}

// ------------------------------------------------------------------ S1
template <int G>
__global__ void __launch_bounds__(128) score_kernel(const __nv_bfloat16* __restrict__ q,
                                                    const float* __restrict__ cent, int C,
                                                    double* __restrict__ crit) {
  pdl_wait();
  const int u = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double qd[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const __nv_bfloat16* qq = q + ((size_t)u * G + g) * 128 + lane * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) qd[g][i] = (double)__bfloat162float(qq[i]);
  }
  const int j0 = blockIdx.x * 32 + warp * 8;
  for (int jj = 0; jj < 8; ++jj) {
    const int j = j0 + jj;
    if (j >= C) break;
    const float4 c = *reinterpret_cast<const float4*>(cent + ((size_t)u * C + j) * 128 + lane * 4);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double s = qd[g][0] * (double)c.x;
      s = fma(qd[g][1], (double)c.y, s);
      s = fma(qd[g][2], (double)c.z, s);
      s = fma(qd[g][3], (double)c.w, s);
      s = warp_sum_d(s);
      if (lane == 0) crit[((size_t)u * G + g) * C + j] = s;
    }
  }
  pdl_launch_dependents();
}

// ------------------------------------------------------------------ S2 + S3
__global__ void __launch_bounds__(SEL_THREADS) sort_kernel(const double* __restrict__ crit,
                                                           const int* __restrict__ offsets, int C, int Cp,
                                                           int G, int* __restrict__ order,
                                                           int* __restrict__ ends) {
  extern __shared__ uint8_t sm[];
  unsigned long long* key = (unsigned long long*)sm;
  int* id = (int*)(key + Cp);
  __shared__ int red[32];
  pdl_wait();
  const int g = blockIdx.x, u = blockIdx.y;
  const double* cr = crit + ((size_t)u * G + g) * C;
  for (int i = threadIdx.x; i < Cp; i += blockDim.x) {
    if (i < C) {
      key[i] = desc_key(cr[i]);
      id[i] = i;
    } else {
      key[i] = ~0ull;
      id[i] = 0x7fffffff;
    }
  }
  __syncthreads();
  for (int k = 2; k <= Cp; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < Cp; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long ki = key[i], kl = key[l];
          const int ii = id[i], il = id[l];
          const bool gt = (ki > kl) || (ki == kl && ii > il);
          const bool asc = (i & k) == 0;
          if (gt == asc) {
            key[i] = kl; key[l] = ki;
            id[i] = il; id[l] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
  // S3: inclusive scan of sizes in rank order
  const int* off = offsets + (size_t)u * (C + 1);
  const int per = (C + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  int loc = 0;
  for (int r = b0; r < b0 + per && r < C; ++r) loc += off[id[r] + 1] - off[id[r]];
  int base = block_exclusive_scan<int>(loc, red, (int*)nullptr);
  int* ord = order + ((size_t)u * G + g) * C;
  int* en = ends + ((size_t)u * G + g) * C;
  for (int r = b0; r < b0 + per && r < C; ++r) {
    base += off[id[r] + 1] - off[id[r]];
    ord[r] = id[r];
    en[r] = base;
  }
  pdl_launch_dependents();
}

// ------------------------------------------------------------------ S4 (logits)
__device__ __forceinline__ int slot_rank(int slot, const SampleConsts& sc) {
  if (sc.fallback) return slot + 1;
  const int W1 = 2 * sc.w + 1;
  if (slot < sc.N) return slot + 1;
  if (slot < sc.N + W1) return sc.x1 - sc.w + (slot - sc.N);
  return sc.x2 - sc.w + (slot - sc.N - W1);
}

__global__ void __launch_bounds__(128) sample_kernel(const __nv_bfloat16* __restrict__ q,
                                                     const __nv_bfloat16* __restrict__ Kp,
                                                     const int* __restrict__ offsets,
                                                     const int* __restrict__ order, const int* __restrict__ ends,
                                                     int n, int C, int G, SampleConsts sc,
                                                     float* __restrict__ logits) {
  extern __shared__ int s_ends[];
  pdl_wait();
  const int g = blockIdx.y, u = blockIdx.z;
  const int* en = ends + ((size_t)u * G + g) * C;
  for (int i = threadIdx.x; i < C; i += blockDim.x) s_ends[i] = en[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, l16 = lane & 15;
  float qf[8];
  {
    const __nv_bfloat16* qq = q + ((size_t)u * G + g) * 128 + l16 * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) qf[i] = __bfloat162float(qq[i]);
  }
  const int* ord = order + ((size_t)u * G + g) * C;
  const int* off = offsets + (size_t)u * (C + 1);
  const float inv_sqrt_d = 0.08838834764831845f;
  const int base_slot = blockIdx.x * 64 + warp * 16;
  for (int it = 0; it < 8; ++it) {
    const int slot = base_slot + it * 2 + half;
    float dot = 0.f;
    const bool valid = slot < sc.slots;
    if (valid) {
      const int rank = slot_rank(slot, sc);
      int lo = 0, hi = C - 1;  // smallest r with ends[r] >= rank
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_ends[mid] >= rank) hi = mid; else lo = mid + 1;
      }
      const int cid = ord[lo];
      const int sr = lo ? s_ends[lo - 1] : 0;
      const int row = off[cid] + (rank - 1 - sr);
      const uint4 kv = *reinterpret_cast<const uint4*>(Kp + ((size_t)u * n + row) * 128 + swz_chunk(l16, row) * 8);
      const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(k2[i]);
        dot = fmaf(qf[2 * i], f.x, dot);
        dot = fmaf(qf[2 * i + 1], f.y, dot);
      }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (valid && l16 == 0) logits[((size_t)u * G + g) * sc.slots + slot] = dot * inv_sqrt_d;
  }
  pdl_launch_dependents();
}

// ------------------------------------------------------------------ S4-S7
// mode 0: Alg. 1 selection; mode 1: sharded stage 2 (grid threshold); mode 2: sharded
// stage 1 (fit only: local (m, theta_max) and cumulative mass at cluster ends).
__global__ void __launch_bounds__(SEL_THREADS) select_kernel(
    const float* __restrict__ logits, const int* __restrict__ order, const int* __restrict__ ends,
    const int* __restrict__ offsets, const double* __restrict__ crit, int n, int C, int G, SampleConsts sc,
    double p, int mode, const double* __restrict__ gmax, const double* __restrict__ gmass,
    double* __restrict__ fit, int* __restrict__ Jout, uint8_t* __restrict__ umask, int* __restrict__ ulist,
    int* __restrict__ uprefix, long long* __restrict__ unit_prefix, unsigned int* __restrict__ counter,
    double* __restrict__ cumend, double* __restrict__ local_max, int units) {
  extern __shared__ uint8_t smraw[];
  double* epref = (double*)smraw;                       // [max(N or n, 1)]
  const int nex = sc.fallback ? n : sc.N;
  int* s_ends = (int*)(epref + (nex > 0 ? nex : 1));     // [C]
  uint8_t* mask = (uint8_t*)(s_ends + C);                // [C]
  __shared__ double redd[32];
  __shared__ float redf[32];
  __shared__ int redi[32];
  __shared__ double sh_d[8];
  __shared__ long long sh_k;
  __shared__ bool s_last;
  pdl_wait();
  const int u = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int* off = offsets + (size_t)u * (C + 1);
  for (int j = tid; j < C; j += nt) mask[j] = 0;
  __syncthreads();

  for (int g = 0; g < G; ++g) {
    const size_t ug = (size_t)u * G + g;
    const int* ord = order + ug * C;
    long long kstar = (long long)n + 1;  // p >= 1: every rank
    if (mode == 1) {
      // ---- sharded stage 2: theta* from the all-reduced mass vector
      const double* gm = gmass + ug * (1 + TACTIC_SHARD_GRID_T);
      const double thmax = gmax[ug * 2 + 1];
      const double Wt = gm[0];
      double thstar = -INFINITY;
      if (p < 1.0) {
        if (tid == 0) {
          int t = 1;
          for (; t <= TACTIC_SHARD_GRID_T; ++t)
            if (gm[t] >= p * Wt) break;
          sh_d[0] = t <= TACTIC_SHARD_GRID_T ? thmax - (double)t * TACTIC_SHARD_GRID_STEP : -INFINITY;
        }
        __syncthreads();
        thstar = sh_d[0];
        __syncthreads();
      }
      const double* cr = crit + ug * C;
      const double isd = 1.0 / sqrt(128.0);
      int cnt = 0;
      for (int j = tid; j < C; j += nt) {
        const bool sel = (off[j + 1] > off[j]) && (cr[j] * isd >= thstar);
        if (sel) { mask[j] = 1; ++cnt; }
      }
      cnt = block_reduce<int>(cnt, redi, false);
      if (tid == 0) {
        Jout[ug] = cnt;
        double* f = fit + ug * 6;
        f[0] = thstar; f[1] = Wt; f[2] = gmax[ug * 2]; f[3] = thmax; f[4] = 0; f[5] = 0;
      }
      continue;
    }
    for (int r = tid; r < C; r += nt) s_ends[r] = ends[ug * C + r];
    const float* L = logits + ug * sc.slots;
    // shift m = max sampled logit (reading 13)
    float mf = -INFINITY;
    for (int i = tid; i < sc.slots; i += nt) mf = fmaxf(mf, L[i]);
    mf = block_reduce<float>(mf, redf, true);
    const double m = (double)mf;
    // exact head weights e_i = exp(l_i - m), i <= nex, and their inclusive prefix
    const int per = (nex + nt - 1) / nt;
    const int b0 = tid * per;
    double loc = 0.0;
    for (int i = b0; i < b0 + per && i < nex; ++i) loc += exp((double)L[i] - m);
    double run = block_exclusive_scan<double>(loc, redd, (double*)nullptr);
    for (int i = b0; i < b0 + per && i < nex; ++i) {
      run += exp((double)L[i] - m);
      epref[i] = run;
    }
    __syncthreads();
    const double EN = epref[nex - 1];
    double a = 0.0, b = 0.0, mu1 = 0.0, mu2 = 0.0, W;
    if (sc.fallback) {
      W = EN;
    } else {
      const int W1 = 2 * sc.w + 1;
      double s1 = 0.0, s2 = 0.0;
      for (int i = tid; i < W1; i += nt) {
        s1 += exp((double)L[sc.N + i] - m);
        s2 += exp((double)L[sc.N + W1 + i] - m);
      }
      s1 = block_reduce<double>(s1, redd, false);
      s2 = block_reduce<double>(s2, redd, false);
      mu1 = s1 / (double)W1;
      mu2 = s2 / (double)W1;
      const double x1 = (double)sc.x1, x2 = (double)sc.x2;
      a = (mu1 - mu2) * x1 * x2 / (x2 - x1);   // O8 / Alg. 1 l.4
      b = mu1 - a / x1;
      W = EN + tail_mass(a, b, sc.N, n);
    }
    if (mode == 2) {
      // sharded stage 1: cumulative estimated mass at every cluster end (local frame)
      double* ce = cumend + ug * C;
      for (int r = tid; r < C; r += nt) {
        const long long e = s_ends[r];
        double v;
        if (e <= 0) v = 0.0;
        else if (e <= nex) v = epref[e - 1];
        else v = EN + tail_mass(a, b, sc.N, e);
        ce[r] = v;
      }
      if (tid == 0) {
        double* f = fit + ug * 6;
        f[0] = a; f[1] = b; f[2] = m; f[3] = W; f[4] = mu1; f[5] = mu2;
        local_max[ug * 2] = m;
        local_max[ug * 2 + 1] = crit[ug * C + ord[0]] / sqrt(128.0);
      }
      __syncthreads();
      continue;
    }
    if (p < 1.0) {
      const double target = p * W;
      if (EN >= target) {
        kstar = 1 + block_lower_bound(0, nex - 1, [&](long long i) { return epref[i] >= target; }, &sh_k);
      } else {
        const double aa = a, bb = b, en_ = EN;
        const long long NN = sc.N;
        kstar = block_lower_bound(NN + 1, n, [&](long long k) { return en_ + tail_mass(aa, bb, NN, k) >= target; },
                                  &sh_k);
      }
    }
    // J = #{r : s_r < k*}, s_r = e_{r-1}; mark the selected non-empty clusters
    int cnt = 0;
    for (int r = tid; r < C; r += nt) {
      const long long sr = r ? s_ends[r - 1] : 0;
      if (sr < kstar) {
        ++cnt;
        const int cid = ord[r];
        if (off[cid + 1] > off[cid]) mask[cid] = 1;
      }
    }
    cnt = block_reduce<int>(cnt, redi, false);
    if (tid == 0) {
      Jout[ug] = cnt;
      double* f = fit + ug * 6;
      f[0] = a; f[1] = b; f[2] = m; f[3] = W; f[4] = mu1; f[5] = mu2;
    }
    __syncthreads();
  }

  if (mode == 2) return;
  // ---- S7: compact the union (cluster-id order) into the work list
  {
    __shared__ int s_totc, s_tott;
    const int per = (C + nt - 1) / nt;
    const int b0 = tid * per;
    int lc = 0, lt = 0;
    for (int j = b0; j < b0 + per && j < C; ++j)
      if (mask[j]) { ++lc; lt += off[j + 1] - off[j]; }
    int cbase = block_exclusive_scan<int>(lc, redi, &s_totc);
    int tbase = block_exclusive_scan<int>(lt, redi, &s_tott);
    int* ul = ulist + (size_t)u * C;
    int* up = uprefix + (size_t)u * (C + 1);
    uint8_t* um = umask + (size_t)u * C;
    for (int j = b0; j < b0 + per && j < C; ++j) {
      um[j] = mask[j];
      if (mask[j]) {
        ul[cbase] = j;
        up[cbase] = tbase;
        ++cbase;
        tbase += off[j + 1] - off[j];
      }
    }
    const int ucount = s_totc, tot = s_tott;
    for (int k = ucount + tid; k <= C; k += nt) {
      up[k] = tot;
      if (k < C) ul[k] = 0;
    }
  }
  // ---- global token prefix over units: done by the last block to finish
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    s_last = (prev == (unsigned)units - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    const int per = (units + nt - 1) / nt;
    const int b0 = tid * per;
    long long loc = 0;
    for (int v = b0; v < b0 + per && v < units; ++v) loc += __ldcg(uprefix + (size_t)v * (C + 1) + C);
    long long run = block_exclusive_scan<long long>(loc, (long long*)redd, (long long*)nullptr);
    for (int v = b0; v < b0 + per && v < units; ++v) {
      unit_prefix[v] = run;
      run += __ldcg(uprefix + (size_t)v * (C + 1) + C);
    }
    if (b0 < units && b0 + per >= units) unit_prefix[units] = run;
    if (units <= b0 && tid == 0 && units == 0) unit_prefix[0] = 0;
    if (tid == 0) *counter = 0u;
  }
  pdl_launch_dependents();
}

// ------------------------------------------------------------------ sharded stage 1b
__global__ void stage1b_kernel(const double* __restrict__ crit, const int* __restrict__ order,
                               const double* __restrict__ cumend, const double* __restrict__ fit,
                               const double* __restrict__ gmax, int C, int G, double* __restrict__ mass) {
  const size_t ug = blockIdx.x;
  const double* cr = crit + ug * C;
  const int* ord = order + ug * C;
  const double* ce = cumend + ug * C;
  const double ms = fit[ug * 6 + 2], Ws = fit[ug * 6 + 3];
  const double mg = gmax[ug * 2], thmax = gmax[ug * 2 + 1];
  const double f = exp(ms - mg);
  const double isd = 1.0 / sqrt(128.0);
  double* out = mass + ug * (1 + TACTIC_SHARD_GRID_T);
  for (int t = threadIdx.x; t <= TACTIC_SHARD_GRID_T; t += blockDim.x) {
    if (t == 0) {
      out[0] = Ws * f;
      continue;
    }
    const double th = thmax - (double)t * TACTIC_SHARD_GRID_STEP;
    int lo = 0, hi = C;  // number of clusters (a prefix of the order) with theta >= th
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cr[ord[mid]] * isd >= th) lo = mid + 1; else hi = mid;
    }
    out[t] = lo > 0 ? ce[lo - 1] * f : 0.0;
  }
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
  cfg.numAttrs = pdl ? 1 : 0;
  return cfg;
}

cudaError_t launch_score(const SelArgs& a, cudaStream_t s, bool pdl) {
  tactic_index_s* x = a.idx;
  cudaLaunchAttribute attr[1];
  auto cfg = make_cfg(dim3((x->C + 31) / 32, x->units), dim3(128), 0, s, pdl, attr);
  switch (x->G) {
    case 1: return cudaLaunchKernelEx(&cfg, score_kernel<1>, a.q, (const float*)x->cent, x->C, x->crit);
    case 2: return cudaLaunchKernelEx(&cfg, score_kernel<2>, a.q, (const float*)x->cent, x->C, x->crit);
    case 4: return cudaLaunchKernelEx(&cfg, score_kernel<4>, a.q, (const float*)x->cent, x->C, x->crit);
    case 8: return cudaLaunchKernelEx(&cfg, score_kernel<8>, a.q, (const float*)x->cent, x->C, x->crit);
  }
  return cudaErrorInvalidValue;
}

static int pow2_at_least(int c) {
  int p = 2;
  while (p < c) p <<= 1;
  return p;
}

cudaError_t launch_sort(const SelArgs& a, cudaStream_t s, bool pdl) {
  tactic_index_s* x = a.idx;
  const int Cp = pow2_at_least(x->C);
  const size_t smem = (size_t)Cp * (8 + 4);
  static size_t set_smem = 0;
  if (smem > 48 * 1024 && smem > set_smem) {
    cudaError_t e = cudaFuncSetAttribute(sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set_smem = smem;
  }
  cudaLaunchAttribute attr[1];
  auto cfg = make_cfg(dim3(x->G, x->units), dim3(SEL_THREADS), smem, s, pdl, attr);
  return cudaLaunchKernelEx(&cfg, sort_kernel, (const double*)x->crit, (const int*)x->offsets, x->C, Cp, x->G,
                            x->order, x->ends);
}

cudaError_t launch_sample(const SelArgs& a, cudaStream_t s, bool pdl) {
  tactic_index_s* x = a.idx;
  cudaLaunchAttribute attr[1];
  auto cfg = make_cfg(dim3((x->sc.slots + 63) / 64, x->G, x->units), dim3(128), (size_t)x->C * 4, s, pdl, attr);
  return cudaLaunchKernelEx(&cfg, sample_kernel, a.q, (const __nv_bfloat16*)x->Kp, (const int*)x->offsets,
                            (const int*)x->order, (const int*)x->ends, x->n, x->C, x->G, x->sc, x->logits);
}

static size_t select_smem(const tactic_index_s* x) {
  const int nex = x->sc.fallback ? x->n : x->sc.N;
  return (size_t)(nex > 0 ? nex : 1) * 8 + (size_t)x->C * 4 + (size_t)x->C + 16;
}

cudaError_t launch_select(const SelArgs& a, cudaStream_t s, bool pdl) {
  tactic_index_s* x = a.idx;
  const size_t smem = select_smem(x);
  static size_t set_smem = 0;
  if (smem > 48 * 1024 && smem > set_smem) {
    cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set_smem = smem;
  }
  cudaLaunchAttribute attr[1];
  auto cfg = make_cfg(dim3(x->units), dim3(SEL_THREADS), smem, s, pdl, attr);
  return cudaLaunchKernelEx(&cfg, select_kernel, (const float*)x->logits, (const int*)x->order,
                            (const int*)x->ends, (const int*)x->offsets, (const double*)x->crit, x->n, x->C, x->G,
                            x->sc, a.p, a.mode, a.gmax, a.gmass, x->fit, x->J, x->umask, x->union_list,
                            x->union_prefix, x->unit_prefix, x->counter, x->cumend, a.local_max, x->units);
}

cudaError_t launch_stage1b(const SelArgs& a, cudaStream_t s) {
  tactic_index_s* x = a.idx;
  stage1b_kernel<<<x->units * x->G, 256, 0, s>>>(x->crit, x->order, x->cumend, x->fit, a.gmax, x->C, x->G,
                                                  a.mass_out);
  return cudaGetLastError();
}

}  // namespace tactic
