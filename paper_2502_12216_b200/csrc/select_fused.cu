// select_fused.cu -- the whole selection S1-S7 of one unit in ONE kernel: a thread-block
// cluster of R CTAs per unit (R = 1..16), phases separated by cluster barriers, small
// cross-CTA data exchanged through distributed shared memory (DSMEM).
//
//   phase 1  S1  CTA r scores clusters [r C/R, (r+1) C/R) for all G heads (float64,
//                 warp butterfly reduce-scatter) -> crit in global (L2).
//   phase 2  S2+S3  each CTA ranks the clusters of its head(s) (bucketed ranks on a
//                 monotone map of crit; ties by id) -> order, end ranks, layout rows (smem).
//   phase 3  S4  Q = R/G CTAs share a head's sampled slots (first N ranks, two windows
//                 around x1, x2): gather the K rows, exact logits, local max,
//                 and local sums of exp(l - m_local) per region.
//   phase 4  S5+S6 the head's CTAs combine their summaries through DSMEM (common shift m),
//                 fit y = a/x + b, estimate W, and find the minimal k with
//                 cum(k) >= p W (Alg. 1 l.10): inside the exact head the CTA that owns the
//                 crossing refines it on its own weights; past the head the clamp-aware
//                 closed form is searched (block-parallel).
//   phase 5  S7  the selected clusters of every head are OR-ed into CTA 0's mask (DSMEM);
//                 CTA 0 compacts the GQA union into the attention work list; the last unit
//                 to finish writes the global token prefix over units.
// Numerics follow select.cu (identical readings); the multi-kernel path in select.cu is
// kept for the sequence-sharded stages and for shapes that exceed this kernel's smem.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <limits.h>

#include "common.cuh"
#include "internal.h"

namespace tactic {

constexpr int FS_THREADS = 256;
constexpr int FS_NB = 1024;    // rank buckets
constexpr int FS_STAGES = 8;   // sampled-row staging pipeline depth
constexpr int FS_CH = 32;      // rows per stage (one warp resolves and issues a stage)

__device__ double harmonic_f(long long k) {
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

// sum_{i=N+1}^{k} max(0, a/i + b)   (same reading as select.cu)
__device__ double tail_mass_f(double a, double b, long long N, long long k) {
  if (k <= N) return 0.0;
  if (a >= 0.0 && b >= 0.0) return a * (harmonic_f(k) - harmonic_f(N)) + b * (double)(k - N);
  if (a <= 0.0 && b <= 0.0) return 0.0;
  if (a > 0.0) {
    const double t = a / (-b);
    long long top = t >= 9.0e15 ? k : (long long)floor(t);
    if (top > k) top = k;
    while (top < k && a / (double)(top + 1) + b > 0.0) ++top;
    while (top > N && !(a / (double)top + b > 0.0)) --top;
    if (top <= N) return 0.0;
    return a * (harmonic_f(top) - harmonic_f(N)) + b * (double)(top - N);
  }
  const double t = (-a) / b;
  long long lo = t >= 9.0e15 ? k + 1 : (long long)floor(t) + 1;
  if (lo < N + 1) lo = N + 1;
  while (lo > N + 1 && a / (double)(lo - 1) + b > 0.0) --lo;
  while (lo <= k && !(a / (double)lo + b > 0.0)) ++lo;
  if (lo > k) return 0.0;
  return a * (harmonic_f(k) - harmonic_f(lo - 1)) + b * (double)(k - lo + 1);
}

// ------------------------------------------------------------ block helpers (256 threads)
template <typename T>
__device__ __forceinline__ T bsum(T v, T* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  T r = 0;
#pragma unroll
  for (int i = 0; i < FS_THREADS / 32; ++i) r += red[i];
  __syncthreads();
  return r;
}
__device__ __forceinline__ float bmaxf(float v, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float r = -INFINITY;
#pragma unroll
  for (int i = 0; i < FS_THREADS / 32; ++i) r = fmaxf(r, red[i]);
  __syncthreads();
  return r;
}
__device__ __forceinline__ double bminmax(double v, double* red, bool mx) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, v, o);
    v = mx ? fmax(v, x) : fmin(v, x);
  }
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
#pragma unroll
  for (int i = 1; i < FS_THREADS / 32; ++i) r = mx ? fmax(r, red[i]) : fmin(r, red[i]);
  __syncthreads();
  return r;
}
template <typename T>
__device__ T bscan_excl(T v, T* red, T* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  __syncthreads();
  if (lane == 31) red[w] = inc;
  __syncthreads();
  T base = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < FS_THREADS / 32; ++i) {
    if (i < w) base += red[i];
    tot += red[i];
  }
  if (total) *total = tot;
  __syncthreads();
  return base + inc - v;
}
template <typename Pred>
__device__ long long blower_bound(long long lo, long long hi, Pred pred, unsigned long long* sh) {
  while (lo < hi) {
    const long long cnt = hi - lo + 1;
    const long long step = (cnt + FS_THREADS - 1) / FS_THREADS;
    const long long k = lo + (long long)threadIdx.x * step;
    if (threadIdx.x == 0) *sh = ~0ull;
    __syncthreads();
    if (k <= hi && pred(k)) atomicMin(sh, (unsigned long long)threadIdx.x);
    __syncthreads();
    const unsigned long long t = *sh;
    __syncthreads();
    if (t == ~0ull) return hi;
    const long long nhi = lo + (long long)t * step;
    const long long nlo = t > 0 ? lo + ((long long)t - 1) * step + 1 : lo;
    lo = nlo;
    hi = nhi < hi ? nhi : hi;
    if (step == 1) return hi;
  }
  return lo;
}

struct FusedParams {
  const __nv_bfloat16* q;
  const float* cent;
  const int* offsets;
  const __nv_bfloat16* Kp;
  int n, C, G, units, R;
  SampleConsts sc;
  double p;
  double* crit;           // [units][G][C]
  int* order;             // [units][G][C] (debug)
  int* ends;              // [units][G][C] (debug)
  float* logits;          // [units][G][slots] (debug)
  double* fit;            // [units][G][6]
  int* J;                 // [units][G]
  uint8_t* umask;         // [units][C]
  int* ulist;             // [units][C]
  int* uprefix;           // [units][C+1]
  long long* unit_prefix; // [units+1]
  unsigned int* unit_cnt; // [1]
  unsigned long long* tlog; // nullable [units][16][8] phase timestamps (debug)
  int slots_per;          // ceil(slots / Q)
  int NH, Q;              // heads per CTA, CTAs per head
};

// per-(CTA, head) summary read by the head's other CTAs
struct __align__(16) HeadSummary {
  double m;        // local max logit (as double)
  double s_head;   // sum exp(l - m) over local exact-head slots
  double s_w1, s_w2;
  long long kstar; // written by the CTA owning the crossing (or -1)
};

template <int G>
__global__ void __launch_bounds__(FS_THREADS, 1) select_fused_kernel(const FusedParams P) {
  extern __shared__ __align__(16) uint8_t smraw[];
  const int C = P.C, n = P.n, NH = P.NH, Q = P.Q;
  const SampleConsts sc = P.sc;
  const int u = blockIdx.y;
  const int r = (int)cluster_rank();
  const int R = P.R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- smem carve-up
  uint8_t* p = smraw;
  HeadSummary* summ = (HeadSummary*)p;              p += sizeof(HeadSummary) * 8;
  uint64_t* fullb = (uint64_t*)p;                    p += sizeof(uint64_t) * (FS_STAGES + 2);
  int* st_rows = (int*)p;                            p += sizeof(int) * FS_STAGES * FS_CH;
  float* qs = (float*)p;                             p += sizeof(float) * NH * 128;
  int* csize = (int*)p;                              p += (size_t)C * 4;
  uint8_t* mask = p;                                 p += ((size_t)C + 15) / 16 * 16;
  int* h_ord = (int*)p;                              p += (size_t)NH * C * 4;
  int* h_end = (int*)p;                              p += (size_t)NH * C * 4;
  int* h_row = (int*)p;                              p += (size_t)NH * C * 4;
  float* h_w = (float*)p;                            p += ((size_t)NH * P.slots_per * 4 + 127) / 128 * 128;
  // union region: phase-2 temporaries | phase-3 staging buffers
  uint8_t* stage = p;                                // [FS_STAGES][FS_CH][256 B]
  double* kcrit = (double*)p;                        p += (size_t)C * 8;
  int* bkt = (int*)p;                                p += (size_t)C * 4;
  int* members = (int*)p;                            p += (size_t)C * 4;
  int* bcnt = (int*)p;                               p += FS_NB * 4;
  int* btok = (int*)p;                               p += FS_NB * 4;
  int* bpos = (int*)p;                               p += FS_NB * 4;
  int* btp = (int*)p;                                p += FS_NB * 4;
  int* bcur = (int*)p;
  __shared__ double redd[FS_THREADS / 32];
  __shared__ float redf[FS_THREADS / 32];
  __shared__ int redi[FS_THREADS / 32];
  __shared__ long long redl[FS_THREADS / 32];
  __shared__ unsigned long long sh_u64;
  __shared__ int s_flag;

  if (tid == 0) {
    for (int i = 0; i < FS_STAGES; ++i) mbar_init(&fullb[i], FS_CH);
    mbar_init(&fullb[FS_STAGES], 1);  // centroid staging
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
#define TLOG(i)                                                                               \
  if (P.tlog && tid == 0) {                                                                   \
    unsigned long long t_;                                                                    \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
    P.tlog[((size_t)u * 16 + r) * 8 + (i)] = t_;                                              \
  }
  TLOG(0);
  const int* off = P.offsets + (size_t)u * (C + 1);
  const size_t ubase = (size_t)u * G;
  for (int j = tid; j < C; j += FS_THREADS) mask[j] = 0;

  // ================= phase 1: S1 scoring (my slice of clusters, all heads) =================
  {
    constexpr int CPW = 32 / G;
    double qd[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint2 raw = *reinterpret_cast<const uint2*>(P.q + (ubase + g) * 128 + lane * 4);
      const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
      const float2 a = __bfloat1622float2(q2[0]), b = __bfloat1622float2(q2[1]);
      qd[g][0] = a.x; qd[g][1] = a.y; qd[g][2] = b.x; qd[g][3] = b.y;
    }
    const int per = (C + R - 1) / R;
    const int js = r * per, je = min(C, js + per);
    // my centroid slice is contiguous: stream it into the staging region with 1-D bulk
    // copies of up to 128 centroids (64 KB), then score from shared memory
    constexpr int CCH = FS_STAGES * FS_CH * 256 / 512;  // centroids per staging fill
    uint64_t* cbar = &fullb[FS_STAGES];
    const float* cst = reinterpret_cast<const float*>(stage);
    int cphase = 0;
    for (int cb = js; cb < je; cb += CCH) {
      const int ce = min(je, cb + CCH);
      if (tid == 0) {
        mbar_arrive_expect_tx(cbar, (uint32_t)(ce - cb) * 512u);
        bulk_g2s(stage, P.cent + ((size_t)u * C + cb) * 128, (uint32_t)(ce - cb) * 512u, cbar);
      }
      mbar_wait(cbar, (uint32_t)cphase);
      cphase ^= 1;
    for (int j0 = cb + warp * CPW; j0 < ce; j0 += (FS_THREADS / 32) * CPW) {
      float4 c[CPW];
#pragma unroll
      for (int jj = 0; jj < CPW; ++jj)
        c[jj] = j0 + jj < ce ? *reinterpret_cast<const float4*>(cst + (size_t)(j0 + jj - cb) * 128 + lane * 4)
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
      if (j0 + jj < ce) P.crit[(ubase + g) * C + j0 + jj] = v[0];
    }
      __syncthreads();  // the staging region is refilled by the next chunk
    }
  }
  for (int j = tid; j < C; j += FS_THREADS) csize[j] = off[j + 1] - off[j];
  TLOG(1);
  cluster_sync_all();
  TLOG(2);

  // ================= phase 2: S2+S3 ranking of my head(s) =================
  for (int hi = 0; hi < NH; ++hi) {
    const int g = (R >= G) ? r / Q : r + R * hi;
    const double* cr = P.crit + (ubase + g) * C;
    double mn = INFINITY, mx = -INFINITY;
    for (int j = tid; j < C; j += FS_THREADS) {
      double x = __ldcg(cr + j);
      if (x == 0.0) x = 0.0;
      kcrit[j] = x;
      mn = fmin(mn, x);
      mx = fmax(mx, x);
    }
    for (int b = tid; b < FS_NB; b += FS_THREADS) { bcnt[b] = 0; btok[b] = 0; bcur[b] = 0; }
    mn = bminmax(mn, redd, false);
    mx = bminmax(mx, redd, true);
    const double scale = mx > mn ? (double)FS_NB / (mx - mn) : 0.0;
    for (int j = tid; j < C; j += FS_THREADS) {
      int b = (int)((mx - kcrit[j]) * scale);
      b = b < FS_NB - 1 ? b : FS_NB - 1;
      bkt[j] = b;
      atomicAdd(&bcnt[b], 1);
      atomicAdd(&btok[b], csize[j]);
    }
    __syncthreads();
    {
      constexpr int PER = FS_NB / FS_THREADS;
      int lc = 0, lt = 0;
#pragma unroll
      for (int i = 0; i < PER; ++i) { lc += bcnt[tid * PER + i]; lt += btok[tid * PER + i]; }
      int cb = bscan_excl<int>(lc, redi, (int*)nullptr);
      int tb = bscan_excl<int>(lt, redi, (int*)nullptr);
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        bpos[tid * PER + i] = cb;
        btp[tid * PER + i] = tb;
        cb += bcnt[tid * PER + i];
        tb += btok[tid * PER + i];
      }
    }
    __syncthreads();
    for (int j = tid; j < C; j += FS_THREADS) members[bpos[bkt[j]] + atomicAdd(&bcur[bkt[j]], 1)] = j;
    __syncthreads();
    int* ord = h_ord + hi * C;
    int* en = h_end + hi * C;
    int* rw = h_row + hi * C;
    const bool dbg = (R >= G) ? (r % Q == 0) : true;
    for (int j = tid; j < C; j += FS_THREADS) {
      const int b = bkt[j];
      const double kj = kcrit[j];
      int rk = bpos[b], s = btp[b];
      const int e = bpos[b] + bcnt[b];
      for (int m = bpos[b]; m < e; ++m) {
        const int i = members[m];
        const double ki = kcrit[i];
        if (ki > kj || (ki == kj && i < j)) { ++rk; s += csize[i]; }
      }
      ord[rk] = j;
      en[rk] = s + csize[j];
      rw[rk] = off[j];
      if (dbg) {
        P.order[(ubase + g) * C + rk] = j;
        P.ends[(ubase + g) * C + rk] = s + csize[j];
      }
    }
    __syncthreads();
  }

  TLOG(3);
  // ================= phase 3: S4 sampled exact logits + local summaries =================
  // Jobs = (my head hi, my slot i), head-major.  Rows are streamed through FS_STAGES
  // smem stages of FS_CH rows: thread t < FS_CH resolves job c*FS_CH + t to its layout
  // row and issues one 256-byte bulk copy (arrive.expect_tx on the stage barrier, which
  // counts FS_CH arrivals); all warps then score the staged rows.
  const int q_part = (R >= G) ? r % Q : 0;
  const int s0 = q_part * P.slots_per;
  const int s1 = min(sc.slots, s0 + P.slots_per);
  const int nmy = s1 > s0 ? s1 - s0 : 0;
  const int njobs = NH * nmy;
  const int nchunks = (njobs + FS_CH - 1) / FS_CH;
  for (int i = tid; i < NH * 128; i += FS_THREADS) {
    const int hi = i >> 7;
    const int g = (R >= G) ? r / Q : r + R * hi;
    qs[i] = __bfloat162float(P.q[(ubase + g) * 128 + (i & 127)]);
  }
  __syncthreads();
  auto issue = [&](int c) {
    if (tid < FS_CH) {
      const int st = c % FS_STAGES;
      const int job = c * FS_CH + tid;
      int row = -1;
      if (job < njobs) {
        const int hi = job / nmy, slot = s0 + job % nmy;
        const int* en = h_end + hi * C;
        int rank;
        if (sc.fallback || slot < sc.N) rank = slot + 1;
        else if (slot < sc.N + 2 * sc.w + 1) rank = sc.x1 - sc.w + (slot - sc.N);
        else rank = sc.x2 - sc.w + (slot - sc.N - 2 * sc.w - 1);
        int lo = 0, hh = C - 1;  // smallest r with ends[r] >= rank
        while (lo < hh) {
          const int mid = (lo + hh) >> 1;
          if (en[mid] >= rank) hh = mid; else lo = mid + 1;
        }
        row = h_row[hi * C + lo] + (rank - 1 - (lo ? en[lo - 1] : 0));
      }
      st_rows[st * FS_CH + tid] = row;
      // consecutive slots mostly map to consecutive layout rows (ranks inside a cluster):
      // one bulk copy per contiguous run, issued by the run's first lane; run lengths come
      // from a ballot of run starts (no serial scan)
      const int prev = __shfl_up_sync(0xffffffffu, row, 1);
      const bool start = row >= 0 && (tid == 0 || prev != row - 1);
      const unsigned starts = __ballot_sync(0xffffffffu, start || row < 0);
      if (start) {
        const unsigned later = starts & ~((2u << tid) - 1u);  // run breaks after this lane
        const int len = (later ? __ffs(later) - 1 : FS_CH) - tid;
        mbar_arrive_expect_tx(&fullb[st], (uint32_t)len * 256u);
        bulk_g2s(stage + ((size_t)st * FS_CH + tid) * 256, P.Kp + ((size_t)u * n + row) * 128, (uint32_t)len * 256u,
                 &fullb[st]);
      } else {
        mbar_arrive(&fullb[st]);
      }
    }
  };
  fence_proxy_async_smem();  // phase-2 generic writes to the staging region precede the bulk copies
  for (int c = 0; c < FS_STAGES - 1 && c < nchunks; ++c) issue(c);
  const int half = lane >> 4, l16 = lane & 15;
  for (int c = 0; c < nchunks; ++c) {
    const bool stamp = P.tlog && u == 0 && r == 0 && tid == 0 && c < 16 && R <= 8;  // debug
    unsigned long long t_a = 0, t_b = 0;
    if (stamp) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_a));
    if (c + FS_STAGES - 1 < nchunks) issue(c + FS_STAGES - 1);
    if (stamp) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_b));
    const int st = c % FS_STAGES;
    mbar_wait(&fullb[st], (uint32_t)(c / FS_STAGES) & 1u);
    if (stamp) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      P.tlog[(size_t)(8 + c / 2) * 8 + (c % 2) * 4 + 0] = t_a;
      P.tlog[(size_t)(8 + c / 2) * 8 + (c % 2) * 4 + 1] = t_b;
      P.tlog[(size_t)(8 + c / 2) * 8 + (c % 2) * 4 + 2] = t_;
    }
#pragma unroll
    for (int k = 0; k < FS_CH / 16; ++k) {  // 8 warps x 2 rows per step
      const int lr = (k * 8 + warp) * 2 + half;
      const int job = c * FS_CH + lr;
      const int row = st_rows[st * FS_CH + lr];
      float d = 0.f;
      int hi = 0;
      if (row >= 0) {
        hi = job / nmy;
        const uint4 kv = *reinterpret_cast<const uint4*>(stage + ((size_t)st * FS_CH + lr) * 256 +
                                                         swz_chunk(l16, row) * 16);
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
        const float* qh = qs + hi * 128 + l16 * 8;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(k2[i]);
          d = fmaf(qh[2 * i], f.x, d);
          d = fmaf(qh[2 * i + 1], f.y, d);
        }
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o, 16);
      if (row >= 0 && l16 == 0) {
        const float lg = d * 0.08838834764831845f;
        const int slot = s0 + job % nmy;
        h_w[(size_t)hi * P.slots_per + (slot - s0)] = lg;
        P.logits[(ubase + ((R >= G) ? r / Q : r + R * hi)) * sc.slots + slot] = lg;
      }
    }
    __syncthreads();  // stage st is re-issued by the next iteration
    if (P.tlog && u == 0 && r == 0 && tid == 0 && c < 16 && R <= 8) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      P.tlog[(size_t)(8 + c / 2) * 8 + (c % 2) * 4 + 3] = t_;
    }
  }
  for (int hi = 0; hi < NH; ++hi) {
    float* wv = h_w + (size_t)hi * P.slots_per;
    float lm = -INFINITY;
    for (int i = tid; i < nmy; i += FS_THREADS) lm = fmaxf(lm, wv[i]);
    lm = bmaxf(lm, redf);
    const float lmaxh = lm;
    const double m = (double)lmaxh;
    double sh = 0.0, s1w = 0.0, s2w = 0.0;
    const int W1 = 2 * sc.w + 1;
    for (int s = s0 + tid; s < s1; s += FS_THREADS) {
      const float e = (float)exp((double)wv[s - s0] - m);
      wv[s - s0] = e;
      if (sc.fallback || s < sc.N) sh += e;
      else if (s < sc.N + W1) s1w += e;
      else s2w += e;
    }
    sh = bsum<double>(sh, redd);
    s1w = bsum<double>(s1w, redd);
    s2w = bsum<double>(s2w, redd);
    if (tid == 0) {
      summ[hi].m = (s1 > s0) ? m : -INFINITY;
      summ[hi].s_head = sh;
      summ[hi].s_w1 = s1w;
      summ[hi].s_w2 = s2w;
      summ[hi].kstar = -1;
    }
  }
  TLOG(4);
  cluster_sync_all();
  TLOG(5);

  // ================= phase 4: S5+S6 fit and k* per head =================
  // (with Q CTAs per head, the head's CTAs are ranks g*Q .. g*Q+Q-1, summary slot 0)
  for (int hi = 0; hi < NH; ++hi) {
    const int g = (R >= G) ? r / Q : r + R * hi;
    const int sidx = (R >= G) ? 0 : hi;
    double mq[16], hq[16];
    double m = -INFINITY, w1s = 0.0, w2s = 0.0, EN = 0.0;
    for (int qq = 0; qq < Q; ++qq) {
      const int rr = (R >= G) ? g * Q + qq : r;
      const uint32_t ra = dsmem_addr(&summ[sidx], rr);
      mq[qq] = ld_dsmem_f64(ra + offsetof(HeadSummary, m));
      hq[qq] = ld_dsmem_f64(ra + offsetof(HeadSummary, s_head));
      m = fmax(m, mq[qq]);
    }
    for (int qq = 0; qq < Q; ++qq) {
      const int rr = (R >= G) ? g * Q + qq : r;
      const uint32_t ra = dsmem_addr(&summ[sidx], rr);
      const double f = mq[qq] == -INFINITY ? 0.0 : exp(mq[qq] - m);
      hq[qq] *= f;
      EN += hq[qq];
      w1s += ld_dsmem_f64(ra + offsetof(HeadSummary, s_w1)) * f;
      w2s += ld_dsmem_f64(ra + offsetof(HeadSummary, s_w2)) * f;
    }
    double a = 0.0, b = 0.0, mu1 = 0.0, mu2 = 0.0, W;
    if (sc.fallback) {
      W = EN;
    } else {
      const int W1 = 2 * sc.w + 1;
      mu1 = w1s / (double)W1;
      mu2 = w2s / (double)W1;
      const double x1 = (double)sc.x1, x2 = (double)sc.x2;
      a = (mu1 - mu2) * x1 * x2 / (x2 - x1);  // O8 / Alg. 1 l.4
      b = mu1 - a / x1;
      W = EN + tail_mass_f(a, b, sc.N, n);
    }
    const bool owner0 = (R >= G) ? (r % Q == 0) : true;
    if (owner0 && tid == 0) {
      double* f = P.fit + (ubase + g) * 6;
      f[0] = a; f[1] = b; f[2] = m; f[3] = W; f[4] = mu1; f[5] = mu2;
    }
    long long kstar = (long long)n + 1;
    if (P.p < 1.0) {
      const double target = P.p * W;
      if (EN >= target) {
        // the exact head slots are split over the Q CTAs in slot order: find the owner
        double before = 0.0;
        int qs = Q - 1;
        for (int qq = 0; qq < Q; ++qq) {
          if (before + hq[qq] >= target) { qs = qq; break; }
          before += hq[qq];
        }
        if (q_part == qs) {
          // refine on my own weights (global frame): smallest slot with prefix >= target
          const float* wv = h_w + (size_t)hi * P.slots_per;
          const int s0 = q_part * P.slots_per;
          const int nloc = min(min(sc.slots, s0 + P.slots_per), sc.fallback ? n : sc.N) - s0;
          const double f = mq[q_part] == -INFINITY ? 0.0 : exp(mq[q_part] - m);
          const int per = (nloc + FS_THREADS - 1) / FS_THREADS;
          const int b0 = tid * per;
          double loc = 0.0;
          for (int i = b0; i < b0 + per && i < nloc; ++i) loc += (double)wv[i] * f;
          double run = before + bscan_excl<double>(loc, redd, (double*)nullptr);
          int found = INT_MAX;
          for (int i = b0; i < b0 + per && i < nloc; ++i) {
            run += (double)wv[i] * f;
            if (run >= target) { found = i; break; }
          }
          // block min over found
          int lmin = found;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
          if (lane == 0) redi[warp] = lmin;
          __syncthreads();
          int fm = INT_MAX;
#pragma unroll
          for (int i = 0; i < FS_THREADS / 32; ++i) fm = min(fm, redi[i]);
          __syncthreads();
          if (fm == INT_MAX) fm = nloc - 1;  // rounding guard: the owner's last slot
          if (tid == 0) summ[sidx].kstar = nloc > 0 ? (long long)(s0 + fm + 1) : (long long)sc.N;
        }
        kstar = -2;  // to be read after the barrier
      } else {
        const double aa = a, bb = b, en_ = EN;
        const long long NN = sc.N;
        kstar = blower_bound(NN + 1, n, [&](long long k) { return en_ + tail_mass_f(aa, bb, NN, k) >= target; },
                             &sh_u64);
      }
    }
    if (tid == 0) redl[hi] = kstar;  // stash (NH <= 8)
    __syncthreads();
  }
  TLOG(6);
  cluster_sync_all();

  // resolve k* from the owning CTA, count J, mark the union in CTA 0's mask
  for (int hi = 0; hi < NH; ++hi) {
    const int g = (R >= G) ? r / Q : r + R * hi;
    const int sidx = (R >= G) ? 0 : hi;
    long long kstar = redl[hi];
    if (kstar == -2) {
      kstar = (long long)n + 1;
      for (int qq = 0; qq < Q; ++qq) {
        const int rr = (R >= G) ? g * Q + qq : r;
        const long long k = ld_dsmem_s64(dsmem_addr(&summ[sidx], rr) + offsetof(HeadSummary, kstar));
        if (k >= 0) kstar = k;
      }
    }
    const bool owner0 = (R >= G) ? (r % Q == 0) : true;
    if (!owner0) continue;
    const int* ord = h_ord + hi * C;
    const int* en = h_end + hi * C;
    const uint32_t mask0 = dsmem_addr(mask, 0);
    int cnt = 0;
    for (int rk = tid; rk < C; rk += FS_THREADS) {
      const long long sr = rk ? en[rk - 1] : 0;
      if (sr < kstar) {
        ++cnt;
        const int cid = ord[rk];
        if (csize[cid] > 0) st_dsmem_u8(mask0 + cid, 1);
      }
    }
    cnt = bsum<int>(cnt, redi);
    if (tid == 0) P.J[ubase + g] = cnt;
  }
  cluster_sync_all();
  TLOG(7);

  // ================= phase 5: S7 union compaction (CTA 0) =================
  if (r != 0) return;
  {
    const int per = (C + FS_THREADS - 1) / FS_THREADS;
    const int b0 = tid * per;
    int lc = 0, lt = 0;
    for (int j = b0; j < b0 + per && j < C; ++j)
      if (mask[j]) { ++lc; lt += csize[j]; }
    int totc = 0, tott = 0;
    int cbase = bscan_excl<int>(lc, redi, &totc);
    int tbase = bscan_excl<int>(lt, redi, &tott);
    int* ul = P.ulist + (size_t)u * C;
    int* up = P.uprefix + (size_t)u * (C + 1);
    uint8_t* um = P.umask + (size_t)u * C;
    for (int j = b0; j < b0 + per && j < C; ++j) {
      um[j] = mask[j];
      if (mask[j]) {
        ul[cbase] = off[j];
        up[cbase] = tbase;
        ++cbase;
        tbase += csize[j];
      }
    }
    for (int k = totc + tid; k <= C; k += FS_THREADS) {
      up[k] = tott;
      if (k < C) ul[k] = 0;
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(P.unit_cnt, 1u);
    s_flag = (prev == (unsigned)P.units - 1);
  }
  __syncthreads();
  if (s_flag) {
    __threadfence();
    const int units = P.units;
    const int per = (units + FS_THREADS - 1) / FS_THREADS;
    const int b0 = tid * per;
    long long loc = 0;
    for (int v = b0; v < b0 + per && v < units; ++v) loc += __ldcg(P.uprefix + (size_t)v * (C + 1) + C);
    long long tot = 0;
    long long run = bscan_excl<long long>(loc, redl, &tot);
    for (int v = b0; v < b0 + per && v < units; ++v) {
      P.unit_prefix[v] = run;
      run += __ldcg(P.uprefix + (size_t)v * (C + 1) + C);
    }
    if (tid == 0) {
      P.unit_prefix[units] = tot;
      *P.unit_cnt = 0u;
    }
  }
  pdl_launch_dependents();
}

// ------------------------------------------------------------------ launcher
static size_t fused_smem(const tactic_index_s* x, int NH, int slots_per) {
  const size_t C = x->C;
  const size_t fixed = sizeof(HeadSummary) * 8 + sizeof(uint64_t) * FS_STAGES + sizeof(int) * FS_STAGES * FS_CH +
                       sizeof(float) * NH * 128 + C * 4 + (C + 15) / 16 * 16 + (size_t)NH * C * 12 +
                       ((size_t)NH * slots_per * 4 + 127) / 128 * 128;
  const size_t phase2 = C * 8 + C * 4 * 2 + (size_t)FS_NB * 4 * 5;
  const size_t staging = (size_t)FS_STAGES * FS_CH * 256;
  return fixed + (phase2 > staging ? phase2 : staging) + 128;
}

// R = CTAs per unit (power of two <= 16); returns cudaErrorNotSupported if the fused
// kernel cannot run this shape (caller falls back to the multi-kernel path).
cudaError_t launch_select_fused(const __nv_bfloat16* q, tactic_index_s* x, double p, cudaStream_t s, bool pdl) {
  const int G = x->G;
  int R = x->fused_R;
  if (R <= 0) return cudaErrorNotSupported;
  const int NH = G > R ? G / R : 1;
  const int Q = R > G ? R / G : 1;
  const int slots_per = (x->sc.slots + Q - 1) / Q;
  const size_t smem = fused_smem(x, NH, slots_per);
  if (smem > 220 * 1024 || NH > 8) return cudaErrorNotSupported;
  FusedParams P = {};
  P.q = q;
  P.cent = x->cent;
  P.offsets = x->offsets;
  P.Kp = x->Kp;
  P.n = x->n;
  P.C = x->C;
  P.G = G;
  P.units = x->units;
  P.R = R;
  P.sc = x->sc;
  P.p = p;
  P.crit = x->crit;
  P.order = x->order;
  P.ends = x->ends;
  P.logits = x->logits;
  P.fit = x->fit;
  P.J = x->J;
  P.umask = x->umask;
  P.ulist = x->union_list;
  P.uprefix = x->union_prefix;
  P.unit_prefix = x->unit_prefix;
  P.unit_cnt = x->counter;
  P.slots_per = slots_per;
  P.tlog = x->tlog;
  P.NH = NH;
  P.Q = Q;
  void (*kern)(const FusedParams) = nullptr;
  switch (G) {
    case 1: kern = select_fused_kernel<1>; break;
    case 2: kern = select_fused_kernel<2>; break;
    case 4: kern = select_fused_kernel<4>; break;
    case 8: kern = select_fused_kernel<8>; break;
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (R > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(R, x->units);
  cfg.blockDim = dim3(FS_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = R;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, P);
}

// choose R once per index: the largest power of two <= 16 with R <= SMs / units
// (at least 1) that the device can co-schedule as a cluster.
int choose_fused_R(tactic_index_s* x) {
  int R = 1;
  while (R * 2 <= 16 && R * 2 * x->units <= x->num_sms) R *= 2;
  const int G = x->G;
  for (; R >= 1; R >>= 1) {
    const int NH = G > R ? G / R : 1;
    const int Q = R > G ? R / G : 1;
    const int slots_per = (x->sc.slots + Q - 1) / Q;
    const size_t smem = fused_smem(x, NH, slots_per);
    if (smem > 220 * 1024 || NH > 8) continue;
    void (*kern)(const FusedParams) = G == 1 ? select_fused_kernel<1>
                                      : G == 2 ? select_fused_kernel<2>
                                      : G == 4 ? select_fused_kernel<4>
                                               : select_fused_kernel<8>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) continue;
    if (R > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(R, x->units);
    cfg.blockDim = dim3(FS_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = R;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    // all of a step's clusters must be co-resident (one wave); R = 1 always qualifies
    if (nclusters >= x->units || (R == 1 && nclusters > 0)) return R;
  }
  return 0;
}

}  // namespace tactic
