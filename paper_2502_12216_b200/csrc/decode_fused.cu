// decode_fused.cu -- one decode step of Tactic (S1-S9: PAPER.md §4.3-§4.6, App. B Alg. 1)
// for one (sequence, KV head) unit inside ONE thread-block cluster, all units in one launch.
//
// Batch-1 decode is latency bound: the multi-kernel chain (score_rank -> sample -> fit ->
// attention) pays a kernel boundary and global-memory round trips between every stage.
// Here a cluster of R CTAs owns a unit (grid R x units, cluster R x 1 x 1); CTA c owns the
// M clusters [cM, cM + M) and every cross-CTA step is a DSMEM exchange + cluster barrier:
//
//  S1  crit_j = q_g . c_j in float64 for all G heads of the unit (the centroid slice is
//      bulk-copied once and read for every head; same products and butterfly tree as
//      select.cu score_kernel, so crit is bit-identical to the multi-kernel path).
//  S2  per head: bitonic sort of the CTA's M keys (-crit, id) (reading 24), exclusive
//      prefix of the sorted sizes, the sorted run pushed to every CTA; a cluster's rank
//      and end rank are its lower bounds in the R runs.
//  S3  every (head, cluster) knows its token-rank interval (s, e] in the partially sorted
//      list; its intersection with the sampled ranks (head 1..N, windows x_k +- w,
//      P:373-376, readings 8-11) is a row interval of the cluster; the CTA samples the
//      hull of those intervals over its heads.
//  S4  one bulk-copy producer warp streams the sampled K rows (contiguous within a
//      cluster) into 8 shared-memory stages; 4 consumer warps compute the G logits of
//      every row with one mma.sync (q in the n dimension), keep each head's logits of its
//      sampled ranks, write them to logits[u][g][slot] and accumulate online
//      (max, exact-head sum, window sums) per head.
//  S5  the per-CTA summaries are exchanged; every CTA combines them in CTA order (so every
//      CTA holds bit-identical values) and fits y = a/x + b through the window means
//      (Alg. 1 l.4), W = E_N + tail(n), target p W (float32, reading 18).
//  S6  cluster r is selected iff the estimated mass ranked before it is < p W (reading
//      14): a per-cluster test s <= N or E_N + tail(s) < pW; when the crossing lies in
//      the exact head (E_N >= pW, or tiny n) the crossing rank k* comes from a block scan
//      of the head's exact weights (read back from logits[], written before the exchange)
//      and the test is s < k* (a fixed budget B: s < B).  J_g = clusters passing it.
//  S7  the GQA union of the CTA's clusters, exchanged with the token counts; every
//      CTA builds the unit's work list (cluster-id order) in shared memory.
//  S8  the CTA streams an equal share of the unit's union tokens (sub-requests) plus
//      the recent-token tail: K/V runs by bulk copy into 4 stages, swap-AB mma.sync
//      flash-decode (the math of attention.cu), online softmax in the exp2 domain.
//  S9  the partial (o, lse) of every CTA is scattered over the cluster (CTA c merges a
//      1/R slice of the G x 128 outputs) and LSE-merged in CTA order.
// The selection outputs (crit, order, ends, logits, J, fit, union mask and work list) are
// written to the index workspace as the multi-kernel path writes them.
#include <cuda.h>
#include <cuda_bf16.h>
#include <limits.h>

#include "common.cuh"
#include "fitmath.cuh"
#include "internal.h"

namespace tactic {

constexpr int FZ_THREADS = 256;
constexpr int FZ_CW = 4;            // consumer warps (warps 1..4); warp 0 produces
constexpr int FZ_STG = 128 * 1024;  // stage region (also the S2 run exchange)
constexpr int FZ_SST = 8;           // sample stages: 64 K rows (16 KB)
constexpr int FZ_AST = 4;           // attention stages: 64 K + 64 V rows (32 KB)
constexpr int FZ_END = 1;
constexpr int FZ_RMAX = 16;       // CTAs per cluster (non-portable above 8)

struct __align__(16) FzMeta {
  unsigned long long mask;
  int flags;
  int pad;
};

struct FzFit {
  float a, b, EN, W, target, m, mu1, mu2;
  int lo, hi, rare, kstar;
};

// byte offsets of the exchange areas inside the centroid region (dead after S1)
template <int G, int M>
struct FzCen {
  static constexpr int SUM = 0;                                           // float4 [RMAX][G]
  static constexpr int CNT = SUM + FZ_RMAX * G * 16;                      // int [RMAX][G + 2]
  static constexpr int LIST = (CNT + FZ_RMAX * (G + 2) * 4 + 15) & ~15;  // int2 [RMAX][M]
  static constexpr int FROW = LIST + FZ_RMAX * M * 8;                     // int [RMAX * M]
  static constexpr int FPRE = FROW + FZ_RMAX * M * 4;                     // int [RMAX * M + 1]
  static constexpr int MLSE = (FPRE + (FZ_RMAX * M + 1) * 4 + 15) & ~15;  // float [RMAX][G]
  static constexpr int MO = MLSE + FZ_RMAX * G * 4;                       // float [R][VPC]
  static constexpr int END = MO + (G * 128 + FZ_RMAX) * 4;
  static_assert(END <= M * 512, "exchange areas exceed the centroid region");
};

__device__ __forceinline__ void fz_put_u32(void* p, int cc, uint32_t v, int R) {
  if (R == 1) *(volatile uint32_t*)p = v;
  else st_dsmem_u32(dsmem_addr(p, (uint32_t)cc), v);
}
__device__ __forceinline__ void fz_put_u64(void* p, int cc, unsigned long long v, int R) {
  if (R == 1) *(volatile unsigned long long*)p = v;
  else st_dsmem_u64(dsmem_addr(p, (uint32_t)cc), v);
}
__device__ __forceinline__ void fz_put_f32(void* p, int cc, float v, int R) {
  fz_put_u32(p, cc, __float_as_uint(v), R);
}
// all threads of every CTA of the cluster; orders shared (DSMEM) and global memory
__device__ __forceinline__ void fz_cluster_sync(int R) {
  if (R > 1) cluster_sync_all();
  else __syncthreads();
}

// merge (m2, s2[3]) into the online (m, s[3]) of sums of exp(l - m)
__device__ __forceinline__ void fz_merge(float& m, float* s, float m2, const float* s2) {
  if (m2 == -INFINITY) return;
  if (m == -INFINITY) {
    m = m2;
    s[0] = s2[0];
    s[1] = s2[1];
    s[2] = s2[2];
    return;
  }
  const float mm = fmaxf(m, m2), f1 = __expf(m - mm), f2 = __expf(m2 - mm);
  s[0] = s[0] * f1 + s2[0] * f2;
  s[1] = s[1] * f1 + s2[1] * f2;
  s[2] = s[2] * f1 + s2[2] * f2;
  m = mm;
}

// block-wide exclusive scan, one value per thread; total -> *tot (all threads call it)
template <typename T>
__device__ __forceinline__ T fz_block_scan(T v, T* red, T* tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  if (lane == 31) red[w] = inc;
  __syncthreads();
  T base = 0, all = 0;
#pragma unroll
  for (int i = 0; i < FZ_THREADS / 32; ++i) {
    const T t = red[i];
    base += i < w ? t : (T)0;
    all += t;
  }
  if (tot) *tot = all;
  __syncthreads();
  return base + inc - v;
}

// sampled-rank region of rank r (1-based): 0 exact head, 1 / 2 window, -1 not sampled;
// *slot = the rank's slot in logits[u][g][.] (O6/O7 layout of the multi-kernel path)
__device__ __forceinline__ int fz_region(int r, const SampleConsts& sc, int* slot) {
  if (sc.fallback || r <= sc.N) {
    *slot = r - 1;
    return 0;
  }
  const int W1 = 2 * sc.w + 1;
  if (r >= sc.x1 - sc.w && r <= sc.x1 + sc.w) {
    *slot = sc.N + (r - (sc.x1 - sc.w));
    return 1;
  }
  if (r >= sc.x2 - sc.w && r <= sc.x2 + sc.w) {
    *slot = sc.N + W1 + (r - (sc.x2 - sc.w));
    return 2;
  }
  return -1;
}

template <int G, int M>
__global__ void __launch_bounds__(FZ_THREADS, 1) decode_fused_kernel(const FusedArgs a) {
  constexpr int P = G * M;  // (head, cluster) pairs, p = g * M + j
  constexpr int NT = FZ_THREADS;
  using L = FzCen<G, M>;
  extern __shared__ uint8_t fz_raw[];
  uint8_t* stg = (uint8_t*)(((uintptr_t)fz_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* cen = stg + FZ_STG;  // centroid slice [M][128] f32, then the exchange areas
  __shared__ double s_crit[P];
  __shared__ unsigned long long s_key[P];
  __shared__ int s_start[P];  // S2: sorted-size prefix; then s = tokens ranked before (g, j)
  __shared__ int s_chunk[P / 32];
  __shared__ int s_size[M], s_row[M], s_hlo[M], s_hhi[M], s_uflag[M];
  __shared__ long long s_red64[NT / 32];
  __shared__ float s_redf[NT / 32];
  __shared__ uint32_t s_smeta[FZ_SST][64];  // sample slot: position in the cluster
  __shared__ uint16_t s_sment[FZ_SST][64];  // sample slot: candidate run (src * M + k)
  __shared__ FzMeta s_meta[FZ_SST];
  __shared__ __align__(8) uint64_t s_full[FZ_SST], s_empty[FZ_SST], s_afull[FZ_AST], s_aempty[FZ_AST], s_cbar, s_rbar, s_xbar;
  __shared__ float4 s_wsum[FZ_CW][8];
  __shared__ FzFit s_fit[G];
  __shared__ int s_Jc[G];
  __shared__ int s_ub[FZ_RMAX + 1], s_tb[FZ_RMAX + 1], s_rb[FZ_RMAX + 1];
  __shared__ int s_kstar;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x, R = gridDim.x, u = blockIdx.y;
  const int C = a.C, n = a.n;
  const int j0 = c * M;
  const int nval = C - j0 < M ? (C - j0 > 0 ? C - j0 : 0) : M;
  const SampleConsts sc = a.sc;
  const size_t ug0 = (size_t)u * G;
  float4* x_sum = (float4*)(cen + L::SUM);
  int* x_cnt = (int*)(cen + L::CNT);
  int2* x_list = (int2*)(cen + L::LIST);
  int* f_row = (int*)(cen + L::FROW);
  int* f_pre = (int*)(cen + L::FPRE);
  float* m_lse = (float*)(cen + L::MLSE);
  float* m_o = (float*)(cen + L::MO);
  // stage region during S2-S4: run blocks [R] at 0 (keys [G][M+1] u64, size prefix
  // [G][M+1] i32), candidate blocks [R] at the end (header + [M][3+G] i32); the sample
  // stages (16 KB) fill the space below the candidate blocks
  constexpr int RBLK = (G * (M + 1) * 12 + 15) & ~15;
  constexpr int CE = 3 + G;                       // candidate entry: row, count, lo, s[G]
  constexpr int CBLK = (16 + M * CE * 4 + 15) & ~15;
  const int CAND_OFF = FZ_STG - R * CBLK;
  const int NSS = CAND_OFF / 16384 < FZ_SST ? CAND_OFF / 16384 : FZ_SST;
  const int VPC = (G * 128 + R - 1) / R;                     // merged outputs per CTA (S9)
  const bool stamp_on = a.tlog != nullptr && c == 0 && u == 0 && tid == 0;
  auto stamp = [&](int i) {  // debug phase stamps of CTA (0, unit 0): tlog[3000 + i]
    if (stamp_on) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      a.tlog[3000 + i] = t_;
    }
  };
  stamp(0);
  // debug (TACTIC_FUSED_STOP=k): leave after phase k, every CTA of the cluster together
  auto stop_at = [&](int k) {
    if (a.dbg_stop != k) return false;
    fz_cluster_sync(R);
    return true;
  };

  // ------------------------------------------------------------------ prologue
  if (tid == 0) {
    for (int i = 0; i < FZ_SST; ++i) {
      mbar_init(&s_full[i], 32);          // every producer lane publishes its slot metadata
      mbar_init(&s_empty[i], FZ_CW * 32);  // every consumer lane releases its own reads
    }
    for (int i = 0; i < FZ_AST; ++i) {
      mbar_init(&s_afull[i], 1);
      mbar_init(&s_aempty[i], FZ_CW * 32);
    }
    mbar_init(&s_cbar, 1);
    mbar_init(&s_rbar, 1);
    mbar_init(&s_xbar, 1);
    fence_barrier_init();
    // the peers' run and candidate blocks arrive by bulk copy on these barriers
    mbar_arrive_expect_tx(&s_rbar, (uint32_t)((R - 1) * RBLK));
    mbar_arrive_expect_tx(&s_xbar, (uint32_t)((R - 1) * CBLK));
  }
  __syncthreads();
  if (R > 1) cluster_arrive_relaxed();  // paired with the wait before the first DSMEM store
  if (tid == 0 && nval > 0) {
    const uint32_t bytes = (uint32_t)nval * 512u;
    mbar_arrive_expect_tx(&s_cbar, bytes);
    const uint8_t* src = (const uint8_t*)(a.cent + ((size_t)u * C + j0) * 128);
    for (uint32_t o = 0; o < bytes; o += 16384u)
      bulk_g2s(cen + o, src + o, bytes - o < 16384u ? bytes - o : 16384u, &s_cbar);
  }
  for (int j = tid; j < M; j += NT) {
    const int* off = a.offsets + (size_t)u * (C + 1) + j0;
    const int o0 = j < nval ? off[j] : 0, o1 = j < nval ? off[j + 1] : 0;
    s_size[j] = o1 - o0;
    s_row[j] = o0;
    s_hlo[j] = INT_MAX;
    s_hhi[j] = -1;
    s_uflag[j] = 0;
  }
  if (tid < G) s_Jc[tid] = 0;
  pdl_wait();  // q comes from the caller's previous kernel (no-op without PDL)

  // ------------------------------------------------------------------ S1 score
  {
    double qd[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint2 raw = *reinterpret_cast<const uint2*>(a.q + (ug0 + g) * 128 + lane * 4);
      const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
      const float2 x0 = __bfloat1622float2(q2[0]), x1 = __bfloat1622float2(q2[1]);
      qd[g][0] = x0.x;
      qd[g][1] = x0.y;
      qd[g][2] = x1.x;
      qd[g][3] = x1.y;
    }
    if (nval > 0) mbar_wait(&s_cbar, 0);
    constexpr int CPW = 32 / G;
    const float* s_cent = (const float*)cen;
    for (int jb = warp * CPW; jb < M; jb += (NT / 32) * CPW) {
      float4 cv[CPW];
#pragma unroll
      for (int jj = 0; jj < CPW; ++jj)
        cv[jj] = jb + jj < nval ? reinterpret_cast<const float4*>(s_cent + (size_t)(jb + jj) * 128)[lane]
                                : make_float4(0.f, 0.f, 0.f, 0.f);
      double v[32];
#pragma unroll
      for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
        for (int g = 0; g < G; ++g) {
          double s = qd[g][0] * (double)cv[jj].x;
          s = fma(qd[g][1], (double)cv[jj].y, s);
          s = fma(qd[g][2], (double)cv[jj].z, s);
          s = fma(qd[g][3], (double)cv[jj].w, s);
          v[jj * G + g] = s;
        }
      // butterfly reduce-scatter: lane L ends with the total of value L (score_kernel)
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
      const int j = jb + lane / G, g = lane % G;
      if (j < M) s_crit[g * M + j] = j < nval ? v[0] : 0.0;
    }
  }
  __syncthreads();
  stamp(1);
  if (stop_at(1)) return;

  // ------------------------------------------------------------------ S2 rank
  for (int p = tid; p < P; p += NT) {
    const int g = p / M, j = p % M;
    if (j < nval) a.crit[(ug0 + g) * C + j0 + j] = s_crit[p];
    s_key[p] = j < nval ? crit_key(s_crit[p], j0 + j) : ~0ull;
  }
  __syncthreads();
  // bitonic sort of each head's M keys (ascending key = descending crit, then id)
  for (int k = 2; k <= M; k <<= 1)
    for (int d = k >> 1; d > 0; d >>= 1) {
      for (int t = tid; t < P / 2; t += NT) {
        const int i = 2 * t - (t & (d - 1)), l = i + d;
        const bool asc = ((i & (M - 1)) & k) == 0;
        const unsigned long long x = s_key[i], y = s_key[l];
        if ((x > y) == asc) {
          s_key[i] = y;
          s_key[l] = x;
        }
      }
      __syncthreads();
    }
  // this CTA's run block: sorted keys + exclusive prefix of the sorted sizes, per head,
  // with a sentinel (~0, total); written in place, then bulk-copied into every peer
  unsigned long long* my_key = (unsigned long long*)(stg + (size_t)c * RBLK);
  int* my_pre = (int*)(stg + (size_t)c * RBLK + (size_t)G * (M + 1) * 8);
  for (int p = tid; p < P; p += NT) {
    const unsigned long long x = s_key[p];
    const int sz = x != ~0ull ? s_size[(int)(x & 0xFFFull) - j0] : 0;
    int inc = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    s_start[p] = inc - sz;
    if (lane == 31) s_chunk[p >> 5] = inc;
  }
  __syncthreads();
  for (int p = tid; p < P + G; p += NT) {
    const int g = p < P ? p / M : p - P, i = p < P ? p % M : M;
    const int q0 = g * M;
    int carry = 0;
    for (int q = q0 >> 5; q < ((p < P ? p : q0 + M) >> 5); ++q) carry += s_chunk[q];
    my_key[g * (M + 1) + i] = p < P ? s_key[p] : ~0ull;
    my_pre[g * (M + 1) + i] = (p < P ? s_start[p] : 0) + carry;
  }
  fence_proxy_async_smem();  // generic-proxy writes of the block before the TMA reads it
  __syncthreads();
  if (R > 1) {
    cluster_wait();  // every peer has started and initialised its barriers
    if (tid < R && tid != c)
      bulk_s2cluster(dsmem_addr(stg + (size_t)c * RBLK, (uint32_t)tid), stg + (size_t)c * RBLK, (uint32_t)RBLK,
                     dsmem_addr(&s_rbar, (uint32_t)tid));
    mbar_wait(&s_rbar, 0);
  }
  stamp(2);
  if (stop_at(2)) return;
  // global rank r and end rank e of every (head, cluster), in sorted order so the lanes'
  // probes into a peer run are monotone: own position + lower bounds in the R-1 peer runs
  for (int p = tid; p < P; p += NT) {
    const int g = p / M, i = p % M;
    const unsigned long long x = my_key[g * (M + 1) + i];
    if (x == ~0ull) continue;
    const int j = (int)(x & 0xFFFull) - j0, sz = s_size[j];
    int base[FZ_RMAX];
#pragma unroll
    for (int cc = 0; cc < FZ_RMAX; ++cc) base[cc] = 0;
#pragma unroll
    for (int len = M; len > 1;) {
      const int half = len >> 1;
#pragma unroll
      for (int cc = 0; cc < FZ_RMAX; ++cc)
        if (cc < R && cc != c) {
          const unsigned long long* rk = (const unsigned long long*)(stg + (size_t)cc * RBLK) + g * (M + 1);
          if (rk[base[cc] + half - 1] < x) base[cc] += half;
        }
      len -= half;
    }
    int r = i, e = my_pre[g * (M + 1) + i] + sz;
#pragma unroll
    for (int cc = 0; cc < FZ_RMAX; ++cc)
      if (cc < R && cc != c) {
        const unsigned long long* rk = (const unsigned long long*)(stg + (size_t)cc * RBLK) + g * (M + 1);
        const int* rp = (const int*)(stg + (size_t)cc * RBLK + (size_t)G * (M + 1) * 8) + g * (M + 1);
        const int lb = base[cc] + (rk[base[cc]] < x ? 1 : 0);
        r += lb;
        e += rp[lb];
      }
    s_start[g * M + j] = e - sz;
    a.order[(ug0 + g) * C + r] = j0 + j;
    a.ends[(ug0 + g) * C + r] = e;
  }
  __syncthreads();
  stamp(3);
  if (stop_at(3)) return;

  // ------------------------------------------------------------------ S3 sampled rows
  for (int p = tid; p < P; p += NT) {
    const int j = p % M;
    const int sz = s_size[j];
    if (j >= nval || sz == 0) continue;
    const int s = s_start[p], e = s + sz;  // ranks s+1 .. e
    int lo = INT_MAX, hi = -1;
    auto take = [&](int r0, int r1) {
      const int x0 = r0 > s + 1 ? r0 : s + 1, x1 = r1 < e ? r1 : e;
      if (x0 <= x1) {
        lo = min(lo, x0 - s - 1);
        hi = max(hi, x1 - s - 1);
      }
    };
    if (sc.fallback) {
      take(1, n);
    } else {
      take(1, sc.N);
      take(sc.x1 - sc.w, sc.x1 + sc.w);
      take(sc.x2 - sc.w, sc.x2 + sc.w);
    }
    if (hi >= 0) {
      atomicMin(&s_hlo[j], lo);
      atomicMax(&s_hhi[j], hi);
    }
  }
  __syncthreads();
  // the CTA's candidate runs (hull rows of its sampled clusters, id order) with every
  // head's start rank, exchanged so that each CTA samples an equal share of all rows
  {
    const int j = tid;
    const bool f = j < M && s_hhi[j] >= 0;
    const int cnt = f ? s_hhi[j] - s_hlo[j] + 1 : 0;
    long long tot;
    const long long ex = fz_block_scan<long long>(f ? (((long long)cnt << 32) | 1ll) : 0ll, s_red64, &tot);
    int* blk = (int*)(stg + CAND_OFF + (size_t)c * CBLK);
    if (f) {
      int* ent = blk + 4 + (int)(ex & 0xFFFFFFFFll) * CE;
      ent[0] = s_row[j] + s_hlo[j];
      ent[1] = cnt;
      ent[2] = s_hlo[j];
#pragma unroll
      for (int g = 0; g < G; ++g) ent[3 + g] = s_start[g * M + j];
    }
    if (tid == 0) {
      blk[0] = (int)(tot & 0xFFFFFFFFll);
      blk[1] = (int)(tot >> 32);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (R > 1) {
      if (tid < R && tid != c)
        bulk_s2cluster(dsmem_addr(blk, (uint32_t)tid), blk, (uint32_t)CBLK, dsmem_addr(&s_xbar, (uint32_t)tid));
      mbar_wait(&s_xbar, 0);
    }
    if (tid == 0) {
      int rb = 0;
      for (int cc = 0; cc < R; ++cc) {
        s_rb[cc] = rb;
        rb += ((const int*)(stg + CAND_OFF + (size_t)cc * CBLK))[1];
      }
      s_rb[R] = rb;
    }
    __syncthreads();
  }

  // ------------------------------------------------------------------ S4 sample (logits)
  if (stop_at(4)) return;
  if (warp == 0) {
    // producer: rows [Rt c / R, Rt (c+1) / R) of the unit's candidate runs (CTA order),
    // packed into 64-slot stages; a run starts at a slot congruent to its row mod 8 (the
    // layout's row swizzle survives the copy)
    const uint8_t* Kb = (const uint8_t*)a.Kp + (size_t)u * n * 256;
    const int Rt = s_rb[R];
    int r = (int)((long long)Rt * c / R);
    const int r_end = (int)((long long)Rt * (c + 1) / R);
    int src = 0, k = 0, off = 0;
    if (r < r_end) {  // the run holding row r
      while (s_rb[src + 1] <= r) ++src;
      const int* blk = (const int*)(stg + CAND_OFF + (size_t)src * CBLK);
      int acc = s_rb[src];
      while (acc + blk[4 + k * CE + 1] <= r) acc += blk[4 + k++ * CE + 1];
      off = r - acc;
    }
    int stage = 0, nst_dbg = 0;
    uint32_t ph = 0;
    while (r < r_end) {
      mbar_wait(&s_empty[stage], ph ^ 1);
      uint8_t* sK = stg + stage * 16384;
      unsigned long long mask = 0;
      uint32_t bytes = 0;
      int s = 0;
      while (s < 64 && r < r_end) {
        const int* ent = (const int*)(stg + CAND_OFF + (size_t)src * CBLK) + 4 + k * CE;
        const int cnt = ent[1];
        const int row = ent[0] + off;
        const int s0 = s + ((row - s) & 7);
        if (s0 >= 64) break;
        int len = cnt - off < 64 - s0 ? cnt - off : 64 - s0;
        if (len > r_end - r) len = r_end - r;
        for (int t = lane; t < len; t += 32) {
          s_smeta[stage][s0 + t] = (uint32_t)(ent[2] + off + t);
          s_sment[stage][s0 + t] = (uint16_t)(src * M + k);
        }
        if (lane == 0) bulk_g2s(sK + s0 * 256, Kb + (size_t)row * 256, (uint32_t)len * 256u, &s_full[stage]);
        mask |= (len == 64 ? ~0ull : ((1ull << len) - 1ull)) << s0;
        bytes += (uint32_t)len * 256u;
        s = s0 + len;
        r += len;
        off += len;
        if (off == cnt) {
          off = 0;
          ++k;
          while (src < R && k == ((const int*)(stg + CAND_OFF + (size_t)src * CBLK))[0]) {
            ++src;
            k = 0;
          }
        }
      }
      if (lane == 0) {
        s_meta[stage].mask = mask;
        s_meta[stage].flags = 0;
        mbar_arrive_expect_tx(&s_full[stage], bytes);
      } else {
        mbar_arrive(&s_full[stage]);
      }
      if (nst_dbg++ == 0) stamp(10);
      if (++stage == NSS) {
        stage = 0;
        ph ^= 1;
      }
    }
    mbar_wait(&s_empty[stage], ph ^ 1);
    if (lane == 0) {
      s_meta[stage].mask = 0;
      s_meta[stage].flags = FZ_END;
    }
    mbar_arrive(&s_full[stage]);
    if (stamp_on) a.tlog[3011] = (unsigned long long)nst_dbg;
  } else if (warp <= FZ_CW) {
    // consumers: 16 slots each; S^T(16 rows x 8 heads) = K q^T on mma.sync
    const int cw = warp - 1, r0 = lane >> 2, h0 = 2 * (lane & 3);
    uint32_t qb[8][2];
    {
      const uint32_t* qrow = reinterpret_cast<const uint32_t*>(a.q + (ug0 + (r0 < G ? r0 : 0)) * 128);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        qb[ks][0] = r0 < G ? qrow[(ks * 16 + h0) >> 1] : 0u;
        qb[ks][1] = r0 < G ? qrow[(ks * 16 + 8 + h0) >> 1] : 0u;
      }
    }
    const int a_slot = cw * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, a_chi = lane >> 4;
    float mh[2] = {-INFINITY, -INFINITY};
    float S[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
    int stage = 0, nst_c = 0;
    uint32_t ph = 0;
    while (true) {
      mbar_wait(&s_full[stage], ph);
      const FzMeta md = s_meta[stage];
      if (a.tlog && c == 0 && u == 0 && tid == 32) {  // debug: first / last sample stage consumed
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        if (!nst_c++) a.tlog[3012] = t_;
        a.tlog[3013] = t_;
      }
      if (md.flags & FZ_END) break;
      const uint32_t mym = (uint32_t)((md.mask >> (cw * 16)) & 0xFFFFull);
      if (mym) {
        const uint32_t sK = smem_u32(stg + stage * 16384);
        float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t af[4];
          ldsm_x4(af[0], af[1], af[2], af[3], sK + a_slot * 256 + (swz_chunk(2 * ks + a_chi, a_slot) << 4));
          mma_bf16_16816(s4, af, qb[ks][0], qb[ks][1]);
        }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          if (!((mym >> (r0 + 8 * rr)) & 1u)) continue;
          const int slot_s = cw * 16 + r0 + 8 * rr;
          const int i = (int)s_smeta[stage][slot_s], e = s_sment[stage][slot_s];
          const int* ent = (const int*)(stg + CAND_OFF + (size_t)(e / M) * CBLK) + 4 + (e % M) * CE;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int g = h0 + hh;
            if (g >= G) continue;
            int slot;
            const int reg = fz_region(ent[3 + g] + 1 + i, sc, &slot);
            if (reg < 0) continue;
            const float l = s4[2 * rr + hh] * 0.08838834764831845f;  // q.k / sqrt(128)
            a.logits[(ug0 + g) * sc.slots + slot] = l;
            if (l > mh[hh]) {
              const float f = __expf(mh[hh] - l);
              S[hh][0] *= f;
              S[hh][1] *= f;
              S[hh][2] *= f;
              mh[hh] = l;
            }
            S[hh][reg] += __expf(l - mh[hh]);
          }
        }
      }
      mbar_arrive(&s_empty[stage]);
      if (++stage == NSS) {
        stage = 0;
        ph ^= 1;
      }
    }
    // combine the 8 lanes holding the same heads (lane & 3), then hand over per warp
#pragma unroll
    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        float s2[3];
        const float m2 = __shfl_xor_sync(0xffffffffu, mh[hh], o);
        s2[0] = __shfl_xor_sync(0xffffffffu, S[hh][0], o);
        s2[1] = __shfl_xor_sync(0xffffffffu, S[hh][1], o);
        s2[2] = __shfl_xor_sync(0xffffffffu, S[hh][2], o);
        fz_merge(mh[hh], S[hh], m2, s2);
      }
    if (lane < 4)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        if (h0 + hh < G) s_wsum[cw][h0 + hh] = make_float4(mh[hh], S[hh][0], S[hh][1], S[hh][2]);
  }
  __syncthreads();
  stamp(4);
  if (stop_at(5)) return;

  // ------------------------------------------------------------------ S5 exchange + fit
  if (tid < G * FZ_RMAX) {
    const int g = tid % G, cc = tid / G;
    if (cc < R) {
      float m = -INFINITY, s[3] = {0.f, 0.f, 0.f};
      for (int w = 0; w < FZ_CW; ++w) {
        const float4 v = s_wsum[w][g];
        const float s2[3] = {v.y, v.z, v.w};
        fz_merge(m, s, v.x, s2);
      }
      float* dst = reinterpret_cast<float*>(x_sum + c * G + g);
      fz_put_f32(dst + 0, cc, m, R);
      fz_put_f32(dst + 1, cc, s[0], R);
      fz_put_f32(dst + 2, cc, s[1], R);
      fz_put_f32(dst + 3, cc, s[2], R);
    }
  }
  fz_cluster_sync(R);  // also publishes every CTA's logits[] stores to the cluster
  if (tid < G) {
    const int g = tid;
    float m = -INFINITY;
    for (int cc = 0; cc < R; ++cc) m = fmaxf(m, x_sum[cc * G + g].x);
    float EN = 0.f, e1 = 0.f, e2 = 0.f;
    for (int cc = 0; cc < R; ++cc) {
      const float4 v = x_sum[cc * G + g];
      if (v.x == -INFINITY) continue;
      const float f = __expf(v.x - m);
      EN = fmaf(v.y, f, EN);
      e1 = fmaf(v.z, f, e1);
      e2 = fmaf(v.w, f, e2);
    }
    FzFit F;
    F.m = m;
    F.EN = EN;
    F.a = F.b = F.mu1 = F.mu2 = 0.f;
    F.lo = 1;
    F.hi = 0;
    F.W = EN;
    if (!sc.fallback) {
      const float W1 = (float)(2 * sc.w + 1);
      F.mu1 = e1 / W1;
      F.mu2 = e2 / W1;
      const float x1 = (float)sc.x1, x2 = (float)sc.x2;
      F.a = (F.mu1 - F.mu2) * (x1 * x2 / (x2 - x1));  // O8 / Alg. 1 l.4
      F.b = F.mu1 - F.a / x1;
      const TailF t = make_tail_f(F.a, F.b, sc.N, n);
      F.lo = t.lo;
      F.hi = t.hi;
      F.W = EN + t(n);
    }
    F.target = a.p * F.W;
    F.rare = a.fixed_budget > 0 || EN >= F.target;
    F.kstar = a.fixed_budget > 0 ? a.fixed_budget : (sc.fallback ? n : sc.N);
    s_fit[g] = F;
  }
  __syncthreads();
  // crossing inside the exact head: k* = minimal rank with sum_{i<=k} exp(l_i - m) >= pW.
  // The exact-head logits of every such head (written by all CTAs before the exchange)
  // come back in one coalesced round trip into the idle stage memory, then one block
  // scan per head.
  if (a.fixed_budget <= 0) {
    int rare = 0;
    for (int g = 0; g < G; ++g) rare |= s_fit[g].rare << g;  // block-uniform
    const int nex = sc.fallback ? n : sc.N;
    const bool in_smem = (size_t)G * nex * 4 <= (size_t)FZ_STG;
    float* hl = reinterpret_cast<float*>(stg);
    if (rare && in_smem) {
      for (int g = 0; g < G; ++g) {
        if (!((rare >> g) & 1)) continue;
        const float* lg = a.logits + (ug0 + g) * sc.slots;
#pragma unroll 8
        for (int t = tid; t < nex; t += NT) hl[g * nex + t] = __ldcg(lg + t);
      }
      __syncthreads();
    }
    for (int g = 0; g < G; ++g) {
      if (!((rare >> g) & 1)) continue;  // block-uniform
      const int per = (nex + NT - 1) / NT, k0 = tid * per, k1 = min(nex, k0 + per);
      const float m = s_fit[g].m, target = s_fit[g].target;
      const float* lg = in_smem ? hl + g * nex : a.logits + (ug0 + g) * sc.slots;
      float loc = 0.f;
      for (int k = k0; k < k1; ++k) loc += __expf(lg[k] - m);
      const float ex = fz_block_scan<float>(loc, s_redf, nullptr);
      if (tid == 0) s_kstar = nex;  // rounding guard: the last exact rank
      __syncthreads();
      if (ex < target && ex + loc >= target) {
        float run = ex;
        for (int k = k0; k < k1; ++k) {
          run += __expf(lg[k] - m);
          if (run >= target) {
            s_kstar = k + 1;
            break;
          }
        }
      }
      __syncthreads();
      if (tid == 0) s_fit[g].kstar = s_kstar;
      __syncthreads();
    }
  }
  stamp(5);
  if (stop_at(6)) return;

  // ------------------------------------------------------------------ S6 + S7 selection, union
  for (int p = tid; p < P; p += NT) {
    const int g = p / M, j = p % M;
    if (j >= nval) continue;
    const FzFit& F = s_fit[g];
    const int s = s_start[p];
    bool sel;
    if (F.rare) {
      sel = s < F.kstar;
    } else {
      const TailF t = {F.a, F.b, F.lo, F.hi};
      sel = s <= sc.N || F.EN + t(s) < F.target;
    }
    if (sel) {
      atomicAdd(&s_Jc[g], 1);
      if (s_size[j] > 0) s_uflag[j] = 1;
    }
  }
  __syncthreads();
  {
    // the CTA's union clusters in id order: (count, tokens) packed for one block scan
    const int j = tid;
    const bool f = j < M && s_uflag[j];
    const long long v = f ? (((long long)s_size[j] << 32) | 1ll) : 0ll;
    long long tot;
    const long long ex = fz_block_scan<long long>(v, s_red64, &tot);
    if (f) {
      const int k = (int)(ex & 0xFFFFFFFFll), lp = (int)(ex >> 32);
      const int2 ent = make_int2(s_row[j], lp);
      for (int cc = 0; cc < R; ++cc) fz_put_u64(x_list + c * M + k, cc, *reinterpret_cast<const unsigned long long*>(&ent), R);
    }
    if (tid < G + 2) {
      const int val = tid < G ? s_Jc[tid] : (tid == G ? (int)(tot & 0xFFFFFFFFll) : (int)(tot >> 32));
      for (int cc = 0; cc < R; ++cc) fz_put_u32(x_cnt + c * (G + 2) + tid, cc, (uint32_t)val, R);
    }
  }
  fz_cluster_sync(R);
  if (tid == 0) {
    int ub = 0, tb = 0;
    for (int cc = 0; cc < R; ++cc) {
      s_ub[cc] = ub;
      s_tb[cc] = tb;
      ub += x_cnt[cc * (G + 2) + G];
      tb += x_cnt[cc * (G + 2) + G + 1];
    }
    s_ub[R] = ub;
    s_tb[R] = tb;
  }
  __syncthreads();
  const int Utot = s_ub[R], Tu = s_tb[R];
  // the unit's work list, concatenated in CTA (= cluster-id) order, in shared memory
  for (int k = tid; k < Utot; k += NT) {
    int src = 0;
    while (src + 1 < R && s_ub[src + 1] <= k) ++src;
    const int2 e = x_list[src * M + (k - s_ub[src])];
    f_row[k] = e.x;
    f_pre[k] = s_tb[src] + e.y;
  }
  if (tid == 0) f_pre[Utot] = Tu;
  // selection outputs in the multi-kernel layout (debug, ablation, attention-only)
  {
    uint8_t* um = a.umask + (size_t)u * C;
    for (int j = tid; j < nval; j += NT) um[j0 + j] = (uint8_t)s_uflag[j];
    int* ul = a.ulist + (size_t)u * C;
    int* up = a.uprefix + (size_t)u * (C + 1);
    for (int k = tid; k < x_cnt[c * (G + 2) + G]; k += NT) {
      const int2 e = x_list[c * M + k];
      ul[s_ub[c] + k] = e.x;
      up[s_ub[c] + k] = s_tb[c] + e.y;
    }
    for (int k = Utot + c * NT + tid; k <= C; k += R * NT) {  // past the union: the total
      up[k] = Tu;
      if (k < C) ul[k] = 0;
    }
    if (c == 0 && tid < G) {
      const FzFit& F = s_fit[tid];
      int J = 0;
      for (int cc = 0; cc < R; ++cc) J += x_cnt[cc * (G + 2) + tid];
      a.J[ug0 + tid] = J;
      double* f = a.fit + (ug0 + tid) * 6;
      f[0] = F.a;
      f[1] = F.b;
      f[2] = F.m;
      f[3] = F.W;
      f[4] = F.mu1;
      f[5] = F.mu2;
    }
  }
  if (a.unit_prefix && c == 0) {  // global token prefix over units (the last unit writes it)
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      s_kstar = atomicAdd(a.unit_cnt, 1u) == (unsigned)a.units - 1;
    }
    __syncthreads();
    if (s_kstar && tid == 0) {
      __threadfence();
      long long run = 0;
      for (int v = 0; v < a.units; ++v) {
        a.unit_prefix[v] = run;
        run += __ldcg(a.uprefix + (size_t)v * (C + 1) + C) + a.tail_len;
      }
      a.unit_prefix[a.units] = run;
      *a.unit_cnt = 0u;
    }
  }
  // attention stages: zero the V halves once (never-written slots must be finite: 0 * NaN)
  for (int i = tid; i < FZ_AST * 1024; i += NT)
    reinterpret_cast<uint4*>(stg + (i >> 10) * 32768 + 16384)[i & 1023] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  __syncthreads();
  stamp(6);
  if (stop_at(7)) return;

  // ------------------------------------------------------------------ S8 attention
  const long long T = (long long)Tu + a.tail_len;
  const int lo_t = (int)(T * c / R), hi_t = (int)(T * (c + 1) / R);
  if (warp == 0) {
    // producer: the CTA's token range [lo_t, hi_t) of the work list (+ tail rows n..)
    const uint8_t* Kb = (const uint8_t*)a.Kp + (size_t)u * n * 256;
    const uint8_t* Vb = (const uint8_t*)a.Vp + (size_t)u * n * 256;
    const uint8_t* Ktb = a.Kt ? (const uint8_t*)a.Kt + (size_t)u * a.tail_cap * 256 : nullptr;
    const uint8_t* Vtb = a.Vt ? (const uint8_t*)a.Vt + (size_t)u * a.tail_cap * 256 : nullptr;
    int lt = lo_t, k = 0, k0 = 0, row = 0, left = 0, w_row = 0, w_end = 0;
    if (lt < hi_t) {
      if (lt >= Tu) {
        row = n + (lt - Tu);
        left = Tu + a.tail_len - lt;
      } else {
        k = k0 = warp_floor_search<int>(f_pre, Utot, lt);
        w_row = k0 + lane < Utot ? f_row[k0 + lane] : 0;
        w_end = k0 + lane < Utot ? f_pre[k0 + lane + 1] : 0;
        row = __shfl_sync(0xffffffffu, w_row, 0) + (lt - f_pre[k]);
        left = __shfl_sync(0xffffffffu, w_end, 0) - lt;
      }
    }
    int stage = 0;
    uint32_t ph = 0;
    while (lt < hi_t) {
      mbar_wait(&s_aempty[stage], ph ^ 1);
      uint8_t* sK = stg + stage * 32768;
      uint8_t* sV = sK + 16384;
      unsigned long long mask = 0;
      uint32_t bytes = 0;
      int s = 0;
      while (s < 64 && lt < hi_t) {
        const int avail = left < hi_t - lt ? left : hi_t - lt;
        const int s0 = s + ((row - s) & 7);
        if (s0 >= 64) break;
        const int len = avail < 64 - s0 ? avail : 64 - s0;
        if (lane == 0) {
          const bool tail = row >= n;
          const uint8_t* kb = tail ? Ktb + (size_t)(row - n) * 256 : Kb + (size_t)row * 256;
          const uint8_t* vb = tail ? Vtb + (size_t)(row - n) * 256 : Vb + (size_t)row * 256;
          bulk_g2s(sK + s0 * 256, kb, (uint32_t)len * 256u, &s_afull[stage]);
          bulk_g2s(sV + s0 * 256, vb, (uint32_t)len * 256u, &s_afull[stage]);
        }
        mask |= (len == 64 ? ~0ull : ((1ull << len) - 1ull)) << s0;
        bytes += (uint32_t)len * 512u;
        s = s0 + len;
        row += len;
        lt += len;
        left -= len;
        if (left == 0 && lt < hi_t) {
          if (lt >= Tu) {  // into the recent-token tail
            row = n + (lt - Tu);
            left = Tu + a.tail_len - lt;
          } else {
            ++k;
            if (k - k0 == 32) {
              k0 = k;
              w_row = k0 + lane < Utot ? f_row[k0 + lane] : 0;
              w_end = k0 + lane < Utot ? f_pre[k0 + lane + 1] : 0;
            }
            row = __shfl_sync(0xffffffffu, w_row, k - k0);
            left = __shfl_sync(0xffffffffu, w_end, k - k0) - lt;
          }
        }
      }
      if (lane == 0) {
        s_meta[stage].mask = mask;
        s_meta[stage].flags = 0;
        mbar_arrive_expect_tx(&s_afull[stage], bytes);
      }
      if (++stage == FZ_AST) {
        stage = 0;
        ph ^= 1;
      }
    }
    mbar_wait(&s_aempty[stage], ph ^ 1);
    if (lane == 0) {
      s_meta[stage].mask = 0;
      s_meta[stage].flags = FZ_END;
      mbar_arrive(&s_afull[stage]);
    }
  } else if (warp <= FZ_CW) {
    // consumers: S^T = K Q^T, online softmax (exp2), P^T by movmatrix, O^T += V^T P^T
    const int cw = warp - 1, ct = tid - 32;
    const int h0 = 2 * (lane & 3), r0 = lane >> 2;
    const float scale_log2 = 1.4426950408889634f * 0.08838834764831845f;  // log2(e)/sqrt(128)
    uint32_t qb[8][2];
    {
      const uint32_t* qrow = reinterpret_cast<const uint32_t*>(a.q + (ug0 + (r0 < G ? r0 : 0)) * 128);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        qb[ks][0] = r0 < G ? qrow[(ks * 16 + h0) >> 1] : 0u;
        qb[ks][1] = r0 < G ? qrow[(ks * 16 + 8 + h0) >> 1] : 0u;
      }
    }
    float o[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    const int a_slot = cw * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, a_chi = lane >> 4;
    const int v_slot = cw * 16 + (lane & 7) + (lane >> 4) * 8, v_chi = (lane >> 3) & 1;
    int stage = 0;
    uint32_t ph = 0;
    while (true) {
      mbar_wait(&s_afull[stage], ph);
      const FzMeta md = s_meta[stage];
      if (md.flags & FZ_END) break;
      const uint32_t mym = (uint32_t)((md.mask >> (cw * 16)) & 0xFFFFull);
      if (mym) {
        const uint32_t sK = smem_u32(stg + stage * 32768), sV = sK + 16384;
        float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t af[4];
          ldsm_x4(af[0], af[1], af[2], af[3], sK + a_slot * 256 + (swz_chunk(2 * ks + a_chi, a_slot) << 4));
          mma_bf16_16816(s, af, qb[ks][0], qb[ks][1]);
        }
        const bool v_lo = (mym >> r0) & 1u, v_hi = (mym >> (r0 + 8)) & 1u;
        const float x0 = v_lo ? s[0] * scale_log2 : -INFINITY;
        const float x1 = v_lo ? s[1] * scale_log2 : -INFINITY;
        const float x2 = v_hi ? s[2] * scale_log2 : -INFINITY;
        const float x3 = v_hi ? s[3] * scale_log2 : -INFINITY;
        float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);  // finite: >= 1 valid token
        const float c0 = exp2f(m0 - mn0), c1 = exp2f(m1 - mn1);
        m0 = mn0;
        m1 = mn1;
        const float p0 = exp2f(x0 - mn0), p1 = exp2f(x1 - mn1);
        const float p2 = exp2f(x2 - mn0), p3 = exp2f(x3 - mn1);
        l0 = l0 * c0 + p0 + p2;
        l1 = l1 * c1 + p1 + p3;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          o[i][0] *= c0;
          o[i][1] *= c1;
          o[i][2] *= c0;
          o[i][3] *= c1;
        }
        const uint32_t b0 = movmatrix_t(pack_bf16(p0, p1));
        const uint32_t b1 = movmatrix_t(pack_bf16(p2, p3));
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          uint32_t af[4];
          ldsm_x4_t(af[0], af[1], af[2], af[3], sV + v_slot * 256 + (swz_chunk(2 * mt + v_chi, v_slot) << 4));
          mma_bf16_16816(o[mt], af, b0, b1);
        }
      }
      mbar_arrive(&s_aempty[stage]);
      if (++stage == FZ_AST) {
        stage = 0;
        ph ^= 1;
      }
    }
    // the CTA's partial: combine the 4 consumer warps (stage memory is idle now)
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(FZ_CW * 32));
    float* sw = reinterpret_cast<float*>(stg) + cw * (8 * 128 + 16);
    if (lane < 4) {
      sw[8 * 128 + h0] = m0;
      sw[8 * 128 + h0 + 1] = m1;
      sw[8 * 128 + 8 + h0] = l0;
      sw[8 * 128 + 8 + h0 + 1] = l1;
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const int d0 = mt * 16 + r0;
      sw[h0 * 128 + d0] = o[mt][0];
      sw[(h0 + 1) * 128 + d0] = o[mt][1];
      sw[h0 * 128 + d0 + 8] = o[mt][2];
      sw[(h0 + 1) * 128 + d0 + 8] = o[mt][3];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(FZ_CW * 32));
    const float* scr = reinterpret_cast<const float*>(stg);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float mf = -INFINITY;
#pragma unroll
      for (int w = 0; w < FZ_CW; ++w) mf = fmaxf(mf, scr[w * (8 * 128 + 16) + 8 * 128 + g]);
      float lf = 0.f, of = 0.f;
      if (mf != -INFINITY) {
#pragma unroll
        for (int w = 0; w < FZ_CW; ++w) {
          const float* sww = scr + w * (8 * 128 + 16);
          const float e = exp2f(sww[8 * 128 + g] - mf);
          lf += sww[8 * 128 + 8 + g] * e;
          of += sww[g * 128 + ct] * e;
        }
      }
      const bool none = mf == -INFINITY;
      const int v = g * 128 + ct, owner = v / VPC;
      fz_put_f32(m_o + c * VPC + (v - owner * VPC), owner, none ? 0.f : of / lf, R);
      if (ct < R) fz_put_f32(m_lse + c * G + g, ct, none ? -INFINITY : (mf + log2f(lf)) * 0.6931471805599453f, R);
    }
  }
  fz_cluster_sync(R);
  stamp(7);
  if (stop_at(8)) return;

  // ------------------------------------------------------------------ S9 merge (this CTA's slice)
  for (int t = tid; t < VPC; t += NT) {
    const int v = c * VPC + t;
    if (v >= G * 128) break;
    const int g = v >> 7, d = v & 127;
    float mx = -INFINITY;
    for (int cc = 0; cc < R; ++cc) mx = fmaxf(mx, m_lse[cc * G + g]);
    float sum = 0.f, acc = 0.f;
    if (mx != -INFINITY)
      for (int cc = 0; cc < R; ++cc) {
        const float l = m_lse[cc * G + g];
        if (l == -INFINITY) continue;
        const float w = __expf(l - mx);
        sum += w;
        acc = fmaf(w, m_o[cc * VPC + t], acc);
      }
    const float val = sum > 0.f ? acc / sum : 0.f;
    const size_t orow = (ug0 + g) * 128 + d;
    if (a.out) a.out[orow] = __float2bfloat16_rn(val);
    if (a.out_f32) a.out_f32[orow] = val;
    if (a.lse && d == 0) a.lse[ug0 + g] = sum > 0.f ? mx + logf(sum) : -INFINITY;
  }
  stamp(8);
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------- host side
size_t fused_smem_bytes(int M) { return 1024 + (size_t)FZ_STG + (size_t)M * 512; }

template <int G, int M>
static cudaError_t launch_fz_t(const FusedArgs& a, int R, cudaStream_t s) {
  auto kern = decode_fused_kernel<G, M>;
  const size_t smem = fused_smem_bytes(M);
  cudaError_t e = func_smem_optin((const void*)kern, smem, R > 8);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(R, a.units);
  cfg.blockDim = dim3(FZ_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = R;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int G, int M>
static int max_clusters_t(int R) {
  auto kern = decode_fused_kernel<G, M>;
  const size_t smem = fused_smem_bytes(M);
  if (func_smem_optin((const void*)kern, smem, R > 8) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(R, 1);
  cfg.blockDim = dim3(FZ_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = R;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nc = 0;
  const cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, (const void*)kern, &cfg);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return -(int)e;
  }
  return nc;
}

#define FZ_DISPATCH(FN, ...)                                  \
  switch (G * 1000 + M) {                                     \
    case 1064: return FN<1, 64>(__VA_ARGS__);                 \
    case 1128: return FN<1, 128>(__VA_ARGS__);                \
    case 2064: return FN<2, 64>(__VA_ARGS__);                 \
    case 2128: return FN<2, 128>(__VA_ARGS__);                \
    case 4064: return FN<4, 64>(__VA_ARGS__);                 \
    case 4128: return FN<4, 128>(__VA_ARGS__);                \
    case 8064: return FN<8, 64>(__VA_ARGS__);                 \
    case 8128: return FN<8, 128>(__VA_ARGS__);                \
    default: break;                                           \
  }

cudaError_t launch_decode_fused(const FusedArgs& a, int G, int M, int R, cudaStream_t s) {
  FZ_DISPATCH(launch_fz_t, a, R, s);
  return cudaErrorInvalidValue;
}

int fused_max_active_clusters(int G, int M, int R) {
  FZ_DISPATCH(max_clusters_t, R);
  return 0;
}

}  // namespace tactic
