// rank_cluster.cu -- S1 + S2 + S3 in one cluster-launched kernel (§4.3
// P:366-376, App. B Alg. 1 l.1-4; readings 8-11 of DESIGN.md).
//
// One thread-block cluster of R CTAs per (head g, unit u); CTA c owns the M clusters
// [cM, cM + M), one per thread (M = 128 for C <= 1024, else 256; R = ceil(C / M)):
//   S1  crit_j = q_g . c_j in float64 (bf16 x fp32 products are exact in fp64; only the
//       summation order differs from the oracle).  The CTA's centroid slice is index data,
//       so it is bulk-copied (1-D TMA) into shared memory before the grid-dependency wait.
//       A warp scores 32 centroids with a shuffle butterfly reduce-scatter.
//   S2  local bitonic sort of the M keys (register shuffles for partners < 32 apart,
//       double-buffered shared memory above).  Key = order-preserving bits of -crit with
//       the low 12 bits replaced by the cluster id, so one 64-bit compare orders by
//       (-crit, id) (DESIGN reading 24: criticalities that agree in their leading 40
//       mantissa bits -- 1e-12 relative, far below the fp64 summation-order differences
//       between any two implementations of q . c -- rank by cluster id).  The
//       exclusive prefix of the sorted sizes is scanned, and the sorted run (keys, size
//       prefix) is pushed into every CTA of the cluster (DSMEM stores), one cluster barrier.
//       The global rank of a cluster is its local position plus its lower bound in the
//       other R-1 runs; its end rank e_r is its own inclusive prefix plus the other runs'
//       prefixes at those bounds -- no scatter and no second barrier.
//   S3  every cluster writes order[r], ends[r] and the row-map entries of the sampled
//       slots inside its token interval (e_r - size, e_r] (head ranks 1..N, windows
//       x1 +- w, x2 +- w); a warp writes one interval at a time with coalesced stores.
// Work per SM is what bounds this stage (it is latency and issue bound, not memory
// bound): the cluster spreads one head's sort over R SMs instead of one.
#include <cuda_bf16.h>
#include <limits.h>
#include <stdlib.h>

#include "common.cuh"
#include "internal.h"
#include "fitmath.cuh"

namespace tactic {

struct SRParams {
  const __nv_bfloat16* q;   // [units][G][128]
  const float* cent;        // [units][C][128]
  const int* offsets;       // [units][C+1]
  const __nv_bfloat16* Kp;  // [units][n][128] index layout (the sampled rows are prefetched to L2)
  int C, G, n;
  SampleConsts sc;
  double* crit;             // [units][G][C]
  __nv_bfloat16* q_copy;    // nullable [units][G][128]: CTA 0 of each head stores q here
                            // (q may live in mapped host memory; the later kernels read the copy)
  int* order;               // [units][G][C]
  int* ends;                // [units][G][C]
  int* rowmap;              // [units][G][slots]
  unsigned long long* tlog;
};

// one entry of a pushed run: sorted key and exclusive size prefix (entry M: ~0, total)
struct __align__(16) RunEnt {
  unsigned long long key;
  unsigned long long pre;
};

// PS (prescored): S1 ran in score_kernel (select.cu: one read of a unit's centroids for all
// G heads, the same products and butterfly tree: bit-identical crit); this kernel loads crit and holds no centroid slice, so more
// clusters fit per SM.  Used when the launch spans several waves (batch 64, C3).
template <int M, int R, bool PS>
constexpr size_t sr_smem() {
  return (PS ? 0 : (size_t)M * 512) + (size_t)R * (M + 1) * sizeof(RunEnt) + 2 * (size_t)M * 8 + 2 * (size_t)M * 4 + 64;
}

// SW warps per 32 clusters score (non-PS: 4, so a warp's dependent chain covers 8 centroids
// and each SM sub-partition holds several scoring warps; the extra warps leave after S1 and
// the rank part synchronises its M threads on named barrier 1)
template <bool PS>
constexpr int sr_sw() { return PS ? 1 : 4; }
template <int M>
__device__ __forceinline__ void sr_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(M) : "memory");
}

template <int M, int R, bool PS>
__global__ void __launch_bounds__(M * sr_sw<PS>()) score_rank_kernel(const SRParams P) {
  constexpr int NW = M / 32;
  constexpr int SW = sr_sw<PS>();
  const int c = blockIdx.x, g = blockIdx.y, u = blockIdx.z;  // the cluster spans grid x (R CTAs)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int C = P.C;
  extern __shared__ __align__(128) uint8_t sm[];
  float* s_cent = (float*)sm;                                // [M][128] (not PS)
  RunEnt* runs = (RunEnt*)(sm + (PS ? 0 : M * 512));          // [R][M+1]
  unsigned long long* bk = (unsigned long long*)(runs + R * (M + 1));  // [2][M]
  int* s_size = (int*)(bk + 2 * M);                           // [M]
  int* s_row = s_size + M;                                    // [M]
  __shared__ uint64_t bar, rbar;
  __shared__ int red[NW];
  __shared__ int4 s_iv[3 * M];  // S3: sampled-slot intervals (slot, count, row) of this CTA
  __shared__ int s_niv;
  const bool tl_first = c == 0 && g == 0 && u == 0;
  if (tid == 0) tl_mark(P.tlog, 1, 0, tl_first);
  const int cta_lin = (u * P.G + g) * R + c;  // debug: per-CTA start / end at tlog[3000 + 2 i]
  auto cstamp = [&](int e) {
    if (P.tlog && tid == 0 && cta_lin < 512) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      P.tlog[3000 + 2 * cta_lin + e] = t_;
    }
  };
  cstamp(0);
  auto pstamp = [&](int i) {  // debug phase stamps of CTA (0, 0, 0) at tlog[1600 + i]
    if (P.tlog && tl_first && tid == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      P.tlog[1600 + i] = t_;
    }
  };

  // ---- prologue on index data (before the dependency wait)
  const int j = c * M + tid;
  const bool valid = j < C;
  const int nval = C - c * M < M ? (C - c * M > 0 ? C - c * M : 0) : M;  // clusters of this CTA
  if (tid == 0) {
    s_niv = 0;
    mbar_init(&bar, 1);
    mbar_init(&rbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  cluster_arrive_relaxed();  // every CTA has started (and initialised rbar) before any st.async
  if (tid == 0) {
    if (!PS) {
      const uint32_t bytes = (uint32_t)nval * 512u;
      mbar_arrive_expect_tx(&bar, bytes);
      const uint8_t* src = (const uint8_t*)(P.cent + ((size_t)u * C + (size_t)c * M) * 128);
      for (uint32_t o = 0; o < bytes; o += 16384u) {
        const uint32_t b = bytes - o < 16384u ? bytes - o : 16384u;
        bulk_g2s((uint8_t*)s_cent + o, src + o, b, &bar);
      }
    }
    if (R > 1) mbar_arrive_expect_tx(&rbar, (uint32_t)(R * (M + 1) * sizeof(RunEnt)));
  }
  if (tid < M) {
    const int* off = P.offsets + (size_t)u * (C + 1);
    const int o0 = valid ? off[j] : 0, o1 = valid ? off[j + 1] : 0;
    s_size[tid] = o1 - o0;
    s_row[tid] = o0;
  }
  pdl_wait();
  if (tid == 0) tl_mark(P.tlog, 1, 1, tl_first);

  // ---- S1: crit of the warp's 32 centroids (lane L ends up with centroid 32 w + L)
  double crit;
  if constexpr (PS) {
    crit = valid ? __ldcg(P.crit + ((size_t)u * P.G + g) * C + j) : 0.0;
  } else {
      double qd[4];
    {
      const uint2 raw = *reinterpret_cast<const uint2*>(P.q + ((size_t)u * P.G + g) * 128 + lane * 4);
      const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
      const float2 a = __bfloat1622float2(q2[0]), b = __bfloat1622float2(q2[1]);
      qd[0] = a.x; qd[1] = a.y; qd[2] = b.x; qd[3] = b.y;
    }
    if (P.q_copy && c == 0 && warp == 0)
      *reinterpret_cast<uint2*>(P.q_copy + ((size_t)u * P.G + g) * 128 + lane * 4) =
          *reinterpret_cast<const uint2*>(P.q + ((size_t)u * P.G + g) * 128 + lane * 4);
    mbar_wait(&bar, 0);
    pstamp(0);
    // warp w scores the CPW = 32 / SW centroids [w CPW, (w + 1) CPW): lane L holds dims
    // 4L..4L+3 of each; a butterfly reduce-scatter over offsets 16, 8, ... leaves value
    // (L >> 2) & (CPW - 1) on lane L after log2(CPW) levels, and plain butterflies over the
    // remaining offsets finish it -- the same pairing tree as score_kernel (bit-identical crit)
    constexpr int CPW = 32 / SW;
    double v[CPW];
  #pragma unroll
    for (int jj = 0; jj < CPW; ++jj) {
      const int lc = warp * CPW + jj;
      const float4 cv = lc < nval ? reinterpret_cast<const float4*>(s_cent + lc * 128)[lane]
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
      double s = qd[0] * (double)cv.x;
      s = fma(qd[1], (double)cv.y, s);
      s = fma(qd[2], (double)cv.z, s);
      s = fma(qd[3], (double)cv.w, s);
      v[jj] = s;
    }
  #pragma unroll
    for (int o = 16, half = CPW / 2; half >= 1; o >>= 1, half >>= 1) {
      const bool upper = (lane & o) != 0;
  #pragma unroll
      for (int i = 0; i < half; ++i) {
        const double send = upper ? v[i] : v[i + half];
        const double keep = upper ? v[i + half] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    if constexpr (SW == 1) {
      crit = v[0];
    } else {
  #pragma unroll
      for (int o = SW / 2; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
      double* s_crit = reinterpret_cast<double*>(bk);  // the sort buffer is idle until S2
      if ((lane & (SW - 1)) == 0) s_crit[warp * CPW + ((lane / SW) & (CPW - 1))] = v[0];
      __syncthreads();
      if (tid >= M) return;  // the extra scoring warps are done (named barriers from here)
      crit = s_crit[tid];
    }
  }
  pstamp(1);

  // ---- S2: local bitonic sort (ascending packed keys = descending crit, then id)
  unsigned long long x = valid ? crit_key(crit, j) : ~0ull;
  int buf = 0;
#pragma unroll
  for (int k = 2; k <= M; k <<= 1) {
#pragma unroll
    for (int d = k >> 1; d > 0; d >>= 1) {
      unsigned long long o;
      if (d < 32) {
        o = __shfl_xor_sync(0xffffffffu, x, d);
      } else {
        bk[buf * M + tid] = x;
        sr_sync<M>();
        o = bk[buf * M + (tid ^ d)];
        buf ^= 1;
      }
      const bool take_min = ((tid & d) == 0) == ((tid & k) == 0);
      x = take_min ? (o < x ? o : x) : (o > x ? o : x);
    }
  }
  pstamp(2);
  // exclusive prefix of the sorted sizes
  const bool real = x != ~0ull;
  const int id = real ? (int)(x & 0xFFFull) : 0;
  const int size = real ? s_size[id - c * M] : 0;
  int incl = size;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) red[warp] = incl;
  sr_sync<M>();
  int wbase = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int t = red[w];
    wbase += w < warp ? t : 0;
    tot += t;
  }
  const int pre = wbase + incl - size;  // exclusive
  // push the sorted run into every CTA of the cluster (st.async, completes on their rbar)
  cluster_wait();
  if constexpr (R == 1) {  // a one-CTA cluster: plain stores (st.async needs a peer CTA)
    runs[tid] = RunEnt{x, (unsigned long long)pre};
    if (tid == M - 1) runs[M] = RunEnt{~0ull, (unsigned long long)tot};
  } else {
#pragma unroll
    for (int cc = 0; cc < R; ++cc) {
      const uint32_t rb = dsmem_addr(&rbar, (uint32_t)cc);
      st_async_v2u64(dsmem_addr(runs + c * (M + 1) + tid, (uint32_t)cc), x, (unsigned long long)pre, rb);
      if (tid == M - 1)
        st_async_v2u64(dsmem_addr(runs + c * (M + 1) + M, (uint32_t)cc), ~0ull, (unsigned long long)tot, rb);
    }
  }
  const size_t ug = (size_t)u * P.G + g;
  if (!PS && valid) P.crit[ug * C + j] = crit;
  pstamp(3);
  if constexpr (R == 1) sr_sync<M>();
  else mbar_wait(&rbar, 0);
  pstamp(4);

  // ---- global rank and end rank: lower bounds in all R runs (own run: the own position)
  int r = 0, end = size;
  {
    int base[R];
#pragma unroll
    for (int cc = 0; cc < R; ++cc) base[cc] = 0;
#pragma unroll
    for (int len = M; len > 1;) {
      const int half = len >> 1;
#pragma unroll
      for (int cc = 0; cc < R; ++cc)
        base[cc] = runs[cc * (M + 1) + base[cc] + half - 1].key < x ? base[cc] + half : base[cc];
      len -= half;
    }
#pragma unroll
    for (int cc = 0; cc < R; ++cc) {
      const int lb = base[cc] + (runs[cc * (M + 1) + base[cc]].key < x ? 1 : 0);
      r += lb;
      end += (int)runs[cc * (M + 1) + lb].pre;
    }
  }
  pstamp(5);
  if (P.tlog && tid == 0 && cta_lin < 512) {  // debug: per-CTA "ranked" time
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    P.tlog[4096 + cta_lin] = t_;
  }
  if (real) {
    P.order[ug * C + r] = id;
    P.ends[ug * C + r] = end;
  }

  // ---- S3: row-map entries of the sampled slots inside (end - size, end]
  {
    const SampleConsts sc = P.sc;
    const int t_lo = end - size + 1, t_hi = end;  // 1-based token ranks of this cluster
    const int row0 = real ? s_row[id - c * M] : 0;
    const int W1 = 2 * sc.w + 1;
    const int nseg = sc.fallback ? 1 : 3;
    for (int sgi = 0; sgi < nseg; ++sgi) {
      int seg_lo, seg_hi, slot_base;
      if (sc.fallback) { seg_lo = 1; seg_hi = P.n; slot_base = 0; }
      else if (sgi == 0) { seg_lo = 1; seg_hi = sc.N; slot_base = 0; }
      else if (sgi == 1) { seg_lo = sc.x1 - sc.w; seg_hi = sc.x1 + sc.w; slot_base = sc.N; }
      else { seg_lo = sc.x2 - sc.w; seg_hi = sc.x2 + sc.w; slot_base = sc.N + W1; }
      const int a = t_lo > seg_lo ? t_lo : seg_lo, b = t_hi < seg_hi ? t_hi : seg_hi;
      if (real && size > 0 && a <= b) {  // one interval of sampled slots: queue it for the CTA
        const int e = atomicAdd(&s_niv, 1);
        s_iv[e] = make_int4(slot_base + (a - seg_lo), b - a + 1, row0 + (a - t_lo), 0);
      }
    }
  }
  // the CTA's intervals round-robin over its warps (a warp holding several top-ranked
  // clusters no longer writes all of their rows alone)
  sr_sync<M>();
  {
    int* rm = P.rowmap + ug * P.sc.slots;
    const int niv = s_niv;
    for (int e = warp; e < niv; e += NW) {
      const int4 iv = s_iv[e];
      // the sample kernel reads these K rows next: start their HBM -> L2 transfer now
      if (lane == 0 && P.Kp) bulk_prefetch_l2(P.Kp + ((size_t)u * P.n + iv.z) * 128, (uint32_t)iv.y * 256u);
      for (int i = lane; i < iv.y; i += 32) rm[iv.x + i] = iv.z + i;
    }
  }
  pstamp(6);
  cstamp(1);
  if (tid == 0) tl_mark(P.tlog, 1, 2, tl_first);
  pdl_launch_dependents();
}

template <int M, int R, bool PS>
static cudaError_t launch_sr_t(const SRParams& P, int units, cudaStream_t s, bool pdl) {
  constexpr size_t smem = sr_smem<M, R, PS>();
  cudaError_t e = func_smem_optin((const void*)score_rank_kernel<M, R, PS>, smem, R > 8);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(R, P.G, units);
  cfg.blockDim = dim3(M * sr_sw<PS>());
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
  cfg.numAttrs = (pdl && pdl_enabled()) ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, score_rank_kernel<M, R, PS>, P);
}

template <int M, int R>
static cudaError_t launch_sr(const SRParams& P, int units, cudaStream_t s, bool pdl, bool ps) {
  return ps ? launch_sr_t<M, R, true>(P, units, s, pdl) : launch_sr_t<M, R, false>(P, units, s, pdl);
}

bool score_rank_prescored(const tactic_index_s* x) {
  const int C = x->C, M = C <= 1024 ? 128 : 256, R = (C + M - 1) / M;
  const int sms = x->num_sms > 0 ? x->num_sms : 148;
  const bool g_ok = x->G == 1 || x->G == 2 || x->G == 4 || x->G == 8;
  return g_ok && (long long)R * x->G * x->units > 6LL * sms;
}

cudaError_t launch_score_rank(const __nv_bfloat16* q, tactic_index_s* x, cudaStream_t s, bool pdl,
                              __nv_bfloat16* q_copy) {
  SRParams P = {};
  P.q = q;
  P.q_copy = q_copy;
  P.cent = x->cent;
  P.offsets = x->offsets;
  // prefetch the sampled rows into L2 only when they fit there with room to spare (C2: 11 MB;
  // C3's ~200 MB would be evicted before the sample kernel reads them: double HBM traffic)
  const double sampled_mb = (double)x->units * x->G * x->sc.slots * 256.0 / 1e6;
  P.Kp = (getenv("TACTIC_NO_SAMPLE_PREFETCH") || sampled_mb > 32.0) ? nullptr : (const __nv_bfloat16*)x->Kp;
  P.C = x->C;
  P.G = x->G;
  P.n = x->n;
  P.sc = x->sc;
  P.crit = x->crit;
  P.order = x->order;
  P.ends = x->ends;
  P.rowmap = x->rowmap;
  P.tlog = x->tlog;
  // M clusters per CTA, R = pow2 >= ceil(C / M) CTAs per cluster (TACTIC_MAX_CLUSTERS = 4096)
  const int C = x->C, U = x->units;
  // several waves of clusters (C3: 4096 CTAs): score all G heads from one read of the
  // centroids first (score_kernel), then rank from crit with the smaller footprint
  const int M = C <= 1024 ? 128 : 256;
  const int R = (C + M - 1) / M;
  const bool ps = score_rank_prescored(x);
  if (ps && q_copy) return cudaErrorInvalidValue;  // (the mapped-host q path is not prescored)
  if (ps) {
    cudaError_t e = launch_score_all(q, x, s, pdl);
    if (e != cudaSuccess) return e;
    pdl = true;  // the rank kernel's prologue overlaps the scoring
  }
  if (C <= 128) return launch_sr<128, 1>(P, U, s, pdl, ps);
  if (C <= 256) return launch_sr<128, 2>(P, U, s, pdl, ps);
  if (C <= 512) return launch_sr<128, 4>(P, U, s, pdl, ps);
  if (C <= 1024) return launch_sr<128, 8>(P, U, s, pdl, ps);
  if (C <= 2048) return launch_sr<256, 8>(P, U, s, pdl, ps);
  return launch_sr<256, 16>(P, U, s, pdl, ps);
}

}  // namespace tactic
