// attention.cu -- S8/S10 split-KV flash-decode over a token work list, with the S9 LSE
// merge fused in (the last CTA to finish a unit merges that unit's partials).
//
// One kernel serves the sparse path (the GQA union of selected clusters) and
// the dense baseline (all n tokens of the caller's K/V, Eq. 1-2).
// Work balancing follows the paper's sub-request idea: units (KV heads) get CTAs
// in proportion to their selected tokens and each unit's list is cut into equal
// contiguous ranges, one per CTA (unit-aligned split, see UnitSplit), so head-level
// imbalance becomes plain sequence imbalance.  With more units than CTAs/2 the lists of
// all units form one global list cut into equal ranges instead (a CTA may then hold
// pieces of several units; every unit also carries ATT_PIECE_TOKENS virtual tokens so the
// split prices a piece's fixed cost).
//
// Per CTA: 1 producer warp streams 64-token stages of K and V into shared memory
//   sparse: cp.async.bulk (1-D TMA, UBLKCP) of contiguous cluster runs from the
//           cluster-permuted, row-swizzled index layout; a run is placed at a slot
//           congruent to its row mod 8 so the swizzle survives the copy.  The run table
//           (row start, token prefix) is read 32 segments at a time into registers.
//   dense : cp.async.bulk.tensor (UTMALDG) 64x64 boxes, SWIZZLE_128B, from the caller's
//           [B][Hkv][n][128] cache.
// 4 consumer warps each own 16 token slots of a stage:
//   S^T(16 tok x 8 heads) = K(16x128) Q^T   (mma.sync m16n8k16, bf16 -> f32, swap-AB so
//   the G<=8 query heads sit in the n=8 dimension), online softmax in the exp2 domain,
//   P^T transposed in registers with movmatrix, O^T(128 x 8) += V^T P^T.
// A piece (the part of one unit inside a CTA's range) ends with a cross-warp LSE
// combine and one partial (o, lse) per head written to slot blockIdx.x (unit-aligned) or
// blockIdx.x + unit (global split); a per-unit
// arrival counter elects the last CTA of the unit, which merges its pieces (S9).  In the
// unit-aligned split the consumers do this themselves (one piece per CTA, at its end); in
// the global split a sixth warp (the piece epilogue) takes each finished piece from the
// consumers through two shared-memory buffers, so the stream does not stop at unit
// switches.
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace tactic {

constexpr int ATT_TILE = 64;
// pipeline depth: 6 stages (192 KB) when the work lists are not staged in shared memory
// (dense, global split), 4 when they are (the lists take the place of stages 4 and 5)
constexpr int ATT_STAGES = 4;
constexpr int ATT_LIST_STAGES = 4;
constexpr int ATT_CWARPS = 4;
// warp 0 producer, warps 1..ATT_CWARPS consumers, last warp the piece epilogue (global split)
constexpr int ATT_THREADS = 32 * (ATT_CWARPS + 2);
constexpr int ATT_EPI_WARP = ATT_CWARPS + 1;
constexpr int ATT_STAGE_BYTES = ATT_TILE * 256 * 2;  // K + V
constexpr int FLAG_FIRST = 1, FLAG_LAST = 2, FLAG_END = 4;
// reference-shift merge window (log2 units): a piece's scaled sums 2^(m_c - mref) (o_c, l_c)
// stay normal and finite in fp32 for l_c < 2^24 tokens and |v| < 2^60
constexpr float ACC_DMIN = 100.f, ACC_DMAX = 40.f;
constexpr int ATT_ACC_ROW = 132;  // accumulator row per (unit, head): o[128], l, padding (16-byte rows)

// G consecutive fp32 adds into global memory as 16- / 8-byte vector reductions
template <int G>
__device__ __forceinline__ void red_add_f32xG(float* p, const float* v) {
  if constexpr (G == 1) {
    atomicAdd(p, v[0]);
  } else if constexpr (G == 2) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v[0]), "f"(v[1]) : "memory");
  } else {
#pragma unroll
    for (int i = 0; i < G; i += 4)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + i), "f"(v[i]), "f"(v[i + 1]),
                   "f"(v[i + 2]), "f"(v[i + 3])
                   : "memory");
  }
}
template <int G>
__device__ __forceinline__ void ld_cg_f32xG(const float* p, float* v) {
  if constexpr (G == 1) {
    v[0] = __ldcg(p);
  } else if constexpr (G == 2) {
    const float2 x = __ldcg(reinterpret_cast<const float2*>(p));
    v[0] = x.x; v[1] = x.y;
  } else {
#pragma unroll
    for (int i = 0; i < G; i += 4) {
      const float4 x = __ldcg(reinterpret_cast<const float4*>(p + i));
      v[i] = x.x; v[i + 1] = x.y; v[i + 2] = x.z; v[i + 3] = x.w;
    }
  }
}
// OR of a predicate over the 128 consumer threads (named barrier 1), a barrier as well
__device__ __forceinline__ int bar_red_or(int x) {
  int r;
  asm volatile("{\n .reg .pred p, q;\n setp.ne.s32 q, %1, 0;\n bar.red.or.pred p, 1, %2, q;\n selp.s32 %0, 1, 0, p;\n}"
               : "=r"(r) : "r"(x), "n"(ATT_CWARPS * 32) : "memory");
  return r;
}

struct __align__(16) StageMeta {
  unsigned long long mask;
  int unit;
  int flags;
};

constexpr int SCRATCH_FLOATS = ATT_CWARPS * (8 * 128 + 16);
// unit-aligned split: the unit's work list (segment rows + token prefix) staged in smem
// (or, when they fit, every unit's lists: one bulk copy of each array, no separate round
// trip for the per-unit totals of the split)
constexpr int LIST_INTS = 16400;
constexpr size_t ATT_BODY = (size_t)ATT_STAGES * ATT_STAGE_BYTES >
                                    (size_t)ATT_LIST_STAGES * ATT_STAGE_BYTES + LIST_INTS * sizeof(int)
                                ? (size_t)ATT_STAGES * ATT_STAGE_BYTES
                                : (size_t)ATT_LIST_STAGES * ATT_STAGE_BYTES + LIST_INTS * sizeof(int);
constexpr size_t ATT_SMEM = ATT_BODY + ATT_STAGES * sizeof(StageMeta) + 4 * ATT_STAGES * sizeof(uint64_t) +
                            SCRATCH_FLOATS * sizeof(float) + 1024;
static_assert(ATT_BODY % 16 == 0, "stage metadata alignment");
static_assert(ATT_SMEM <= 227 * 1024, "attention shared memory");
static_assert(LIST_INTS >= 2 * SCRATCH_FLOATS, "epilogue buffers in the list area");

size_t attention_smem_bytes() { return ATT_SMEM; }

// byte offset of (slot s, 16-byte logical chunk c) inside a 16 KB K or V stage tile
template <bool DENSE>
__device__ __forceinline__ uint32_t tile_off(int s, int c) {
  if (DENSE) return (uint32_t)((c >> 3) * 8192 + s * 128 + (((c ^ s) & 7) << 4));
  return (uint32_t)(s * 256 + (swz_chunk(c, s) << 4));
}

__device__ __forceinline__ int pieces_of_unit(long long us, long long ue, long long T, int P, int* c0) {
  const int a = cta_of(us, T, P), b = cta_of(ue - 1, T, P);
  *c0 = a;
  if (T >= P) return b - a + 1;
  int cnt = 0;
  for (int c = a; c <= b; ++c) cnt += range_start(c, T, P) != range_start(c + 1, T, P);
  return cnt;
}

// warp_floor_search over arr[i] + i x (arr non-decreasing, x >= 0)
__device__ __forceinline__ int warp_floor_search_off(const long long* arr, int count, long long key, long long x) {
  const int lane = threadIdx.x & 31;
  int base = 0, len = count;
  while (len > 32) {
    const int stride = (len + 31) >> 5;
    const int idx = base + lane * stride;
    const bool ok = idx < base + len && arr[idx] + (long long)idx * x <= key;
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    const int h = 31 - __clz(bal);
    const int nb = base + h * stride;
    const int end = base + len;
    base = nb;
    len = (nb + stride < end ? nb + stride : end) - nb;
  }
  const bool ok = lane < len && arr[base + lane] + (long long)(base + lane) * x <= key;
  const unsigned bal = __ballot_sync(0xffffffffu, ok);
  return base + (31 - __clz(bal));
}

// Unit-aligned split (units <= CTAs / 2): every CTA works on exactly one unit.  Unit v
// (T_v work-list tokens, S_v = tokens of the units before it, T = all tokens) owns CTAs
// [cb_v, cb_{v+1}) with cb_v = v + floor((P - U) S_v / T): one CTA each plus a share of
// the rest proportional to its tokens; CTA j of the unit's n_v owns tokens
// [T_v j / n_v, T_v (j+1) / n_v) (possibly empty when T_v < n_v).  Every warp computes it
// from the per-unit totals (seg_prefix[v][C]) with two shuffle scans, so the selection
// needs no cross-unit step.  No CTA straddles two units, so a unit's last piece is not
// delayed behind another unit's piece, and the unit's partials sit in slots cb_v + j.
struct UnitSplit {
  int u, j, n;       // unit, index of this CTA within the unit, CTAs of the unit
  int lo, hi;        // token range within the unit's work list
  int dm;            // designated merger protocol (CTA j = 0 merges; its range is shorter)
};
// tokens the designated merger's range is shortened by (at most half its share): about
// the time of the other pieces' piece end and arrival, so it waits on none of them
constexpr int ATT_MERGER_SHORT = 192;

// floor(x / y) for 0 <= x < 2^31, 0 < y: fast reciprocal estimate (off by at most one
// below 2^22), then exact corrections with wide products
__device__ __forceinline__ int floor_div32(int x, int y) {
  int q = __float2int_rz(__fdividef(__int2float_rn(x), __int2float_rn(y)));
  while ((long long)q * y > x) --q;
  while ((long long)(q + 1) * y <= x) ++q;
  return q;
}

// The same split in 32-bit arithmetic for <= 32 units and (n + tail) units P < 2^31 (one
// warp pass, no 64-bit multiplies or divisions: the split sits between the dependency wait
// and the first tile).  With dm, CTA 0 of a unit of n >= 2 CTAs (the designated merger)
// gets ATT_MERGER_SHORT fewer tokens, the others share the rest equally.
template <bool DENSE>
__device__ __forceinline__ UnitSplit unit_split_fast(const AttnArgs& a, int cta, int P, bool dm) {
  const int U = a.units, lane = threadIdx.x & 31;
  const int tv = lane < U ? (DENSE ? a.n : __ldcg(a.seg_prefix + (size_t)lane * (a.C + 1) + a.C) + a.tail_len) : 0;
  int incl = tv;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  const int T = __shfl_sync(0xffffffffu, incl, 31);
  const bool uniform = T <= 0;  // degenerate: equal split by unit count
  const int Tt = uniform ? U : T;
  const int Sv = uniform ? lane : incl - tv, t1 = uniform ? 1 : tv;
  const int extra = P - U;
  // cb_v = v + floor(extra S_v / T), cb_{v+1} likewise (two independent divisions)
  const int cb = lane + floor_div32(extra * Sv, Tt);
  const int cbn = lane + 1 + floor_div32(extra * (Sv + t1), Tt);
  const unsigned hit = __ballot_sync(0xffffffffu, lane < U && cb <= cta && cta < cbn);
  const int l = hit ? __ffs(hit) - 1 : 0;
  UnitSplit r;
  r.u = l;
  r.j = cta - __shfl_sync(0xffffffffu, cb, l);
  r.n = __shfl_sync(0xffffffffu, cbn, l) - (cta - r.j);
  const int Tu = uniform ? 0 : __shfl_sync(0xffffffffu, tv, l);
  r.dm = dm;
  // lane 0: lo, lane 1: hi
  const int jj = r.j + (lane & 1);
  int bnd;
  if (dm && r.n > 1) {
    const int share = floor_div32(Tu, r.n);
    const int cut = ATT_MERGER_SHORT < share / 2 ? ATT_MERGER_SHORT : share / 2;
    const int h0 = share - cut;  // the merger's range [0, h0)
    bnd = jj == 0 ? 0 : h0 + floor_div32((Tu - h0) * (jj - 1), r.n - 1);
  } else {
    bnd = floor_div32(Tu * jj, r.n);
  }
  r.lo = __shfl_sync(0xffffffffu, bnd, 0);
  r.hi = __shfl_sync(0xffffffffu, bnd, 1);
  return r;
}
// floor(x / y) for 0 <= x, 0 < y, quotient below 2^24: an fp32 reciprocal estimate fixed
// up with exact 64-bit multiplies (a dependent 64-bit integer or fp64 division costs
// hundreds of cycles on the single warp that computes the split)
__device__ __forceinline__ long long floor_div(long long x, long long y) {
  long long q = (long long)((float)x * __frcp_rn((float)y));
  while (q > 0 && q * y > x) --q;
  while ((q + 1) * y <= x) ++q;
  return q;
}

template <bool DENSE>
__device__ __forceinline__ UnitSplit unit_split_of(const AttnArgs& a, int cta, int P, const int* pref) {
  const int U = a.units, lane = threadIdx.x & 31;
  auto tok = [&](int v) -> long long {
    if (v >= U) return 0;
    return DENSE ? (long long)a.n : (long long)pref[(size_t)v * (a.C + 1) + a.C] + a.tail_len;
  };
  long long T = 0;
  for (int v0 = 0; v0 < U; v0 += 32) T += tok(v0 + lane);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) T += __shfl_xor_sync(0xffffffffu, T, o);
  const bool uniform = T <= 0;  // degenerate: equal split by unit count
  const long long Tt = uniform ? U : T;
  const long long extra = P - U;
  long long S = 0;
  UnitSplit r = {0, 0, 1, 0, 0, 0};
  for (int v0 = 0; v0 < U; v0 += 32) {
    const int v = v0 + lane;
    const long long tv = uniform ? (v < U ? 1 : 0) : tok(v);
    long long incl = tv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    const long long Sv = S + incl - tv;
    // cb_v = v + floor(extra S_v / T); cb_{v+1} from the next lane (S_{v+1} = S_v + t_v)
    const long long cb = v + floor_div(extra * Sv, Tt);
    long long cbn = __shfl_down_sync(0xffffffffu, cb, 1);
    if (lane == 31) cbn = v + 1 + floor_div(extra * (Sv + tv), Tt);
    const unsigned hit = __ballot_sync(0xffffffffu, v < U && cb <= cta && cta < cbn);
    if (hit) {
      const int l = __ffs(hit) - 1;
      const int cbl = (int)__shfl_sync(0xffffffffu, cb, l);
      r.u = v0 + l;
      r.j = cta - cbl;
      r.n = (int)__shfl_sync(0xffffffffu, cbn, l) - cbl;
      const long long Tu = uniform ? 0 : __shfl_sync(0xffffffffu, tv, l);
      r.lo = (int)floor_div(Tu * r.j, r.n);
      r.hi = (int)floor_div(Tu * (r.j + 1), r.n);
      break;
    }
    S += __shfl_sync(0xffffffffu, incl, 31);
  }
  return r;
}

// S9 for one head g of unit u (global split): LSE-weighted merge of the partial slots
// c0 + i + soff, i < span (ranges that held no token of the unit are skipped), by one warp;
// lanes hold 4 dims.  Piece weights are computed 32 at a time (one per lane) and
// broadcast, so the o loads are independent; chunks of 32 pieces: the lane's piece lse and
// the chunk's first 16 partial rows are loaded together, the running max is rescaled
// online across chunks.
template <int G>
__device__ __forceinline__ void merge_head_global(const AttnArgs& a, int u, int g, int c0, int span, int soff,
                                               bool unit_mode, long long T, int P) {
  const int lane = threadIdx.x & 31;
  float mx = -INFINITY, sum = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i0 = 0; i0 < span; i0 += 32) {
    const int i = i0 + lane;
    const bool live = i < span && (unit_mode || T >= P ||
                                   range_start(c0 + i, T, P) != range_start(c0 + i + 1, T, P));
    const unsigned lmask = __ballot_sync(0xffffffffu, live);
    const int cnt = span - i0 < 32 ? span - i0 : 32;
    const float l = live ? __ldcg(a.part_lse + ((size_t)(c0 + i) + soff) * G + g) : -INFINITY;
    float4 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float4* src =
          reinterpret_cast<const float4*>(a.part_o + (((size_t)(c0 + i0 + k) + soff) * G + g) * 128) + lane;
      v[k] = (k < cnt && ((lmask >> k) & 1u)) ? __ldcg(src) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float nm = fmaxf(mx, warp_max(l));
    const float sc = mx == -INFINITY ? 0.f : __expf(mx - nm);
    acc.x *= sc; acc.y *= sc; acc.z *= sc; acc.w *= sc;
    sum *= sc;
    mx = nm;
    const float wl = (live && l > -INFINITY) ? __expf(l - mx) : 0.f;
    sum += warp_sum(wl);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float w = __shfl_sync(0xffffffffu, wl, k);
      acc.x = fmaf(w, v[k].x, acc.x);
      acc.y = fmaf(w, v[k].y, acc.y);
      acc.z = fmaf(w, v[k].z, acc.z);
      acc.w = fmaf(w, v[k].w, acc.w);
    }
    if (cnt > 16) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int j = 16 + k;
        const float4* src =
            reinterpret_cast<const float4*>(a.part_o + (((size_t)(c0 + i0 + j) + soff) * G + g) * 128) + lane;
        v[k] = (j < cnt && ((lmask >> j) & 1u)) ? __ldcg(src) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float w = __shfl_sync(0xffffffffu, wl, 16 + k);
        acc.x = fmaf(w, v[k].x, acc.x);
        acc.y = fmaf(w, v[k].y, acc.y);
        acc.z = fmaf(w, v[k].z, acc.z);
        acc.w = fmaf(w, v[k].w, acc.w);
      }
    }
  }
  const float inv = 1.f / sum;
  const size_t orow = ((size_t)u * G + g) * 128 + lane * 4;
  if (a.out) {
    __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(a.out + orow);
    ob[0] = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    ob[1] = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
  }
  if (a.out_f32)
    *reinterpret_cast<float4*>(a.out_f32 + orow) =
        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  if (a.lse && lane == 0) a.lse[(size_t)u * G + g] = mx + logf(sum);
}

// the unit-aligned split's merge stages the unit's contiguous partials in the idle stage
// buffers (a CTA of that split holds one piece, so no copy is in flight at its end)
template <int G>
__device__ __forceinline__ bool smem_merge_ok(bool unit_mode, int np) {
  return unit_mode && np * G * 4 + 16 <= 1024 &&
         (size_t)np * G * 512 + 1024 <= (size_t)ATT_LIST_STAGES * ATT_STAGE_BYTES;
}

// UNIT: the unit-aligned split (a.unit_split != 0) compiled apart from the global split,
// so each instantiation holds only its own prologue, piece-end and merge code (the kernel
// starts with a cold instruction cache every layer)
template <int G, bool DENSE, bool UNIT>
__global__ void __launch_bounds__(ATT_THREADS, 1)
    attention_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, long long dense_total) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* stages = smem;
  StageMeta* meta = (StageMeta*)(stages + ATT_BODY);
  uint64_t* full = (uint64_t*)(meta + ATT_STAGES);
  uint64_t* empty = full + ATT_STAGES;
  uint64_t* mbar = empty + ATT_STAGES;  // [0]: merge staging, [1]: lists, [2..5]: epilogue
  uint64_t* ep_full = mbar + 2;          // [2] piece handed to the epilogue warp (global split)
  uint64_t* ep_empty = mbar + 4;         // [2] epilogue buffer free again
  float* scratch = (float*)(empty + 3 * ATT_STAGES);
  int* s_list = (int*)(stages + ATT_LIST_STAGES * ATT_STAGE_BYTES);  // seg_row [C] | seg_prefix [C+1]
  // global split (no lists in smem): two piece buffers for the epilogue warp in the list area
  float* ep_buf = (float*)s_list;
  __shared__ int s_merge;
  __shared__ int ep_meta[2];  // unit of the piece in each epilogue buffer; -1: end of stream

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) tl_mark(a.tlog, 4, 0, blockIdx.x == 0);
  // zero the V halves of the stages once: a never-written V slot meets P = 0, and 0 * NaN
  // would poison O (a never-written K slot only feeds a logit that the mask replaces)
  const int nst = (!DENSE && UNIT) ? ATT_LIST_STAGES : ATT_STAGES;  // stages in use
  constexpr int HALF16 = ATT_STAGE_BYTES / 32;  // 16-byte words per K or V half
  for (int i = threadIdx.x; i < nst * HALF16; i += ATT_THREADS)
    reinterpret_cast<uint4*>(stages + (i / HALF16) * ATT_STAGE_BYTES + ATT_STAGE_BYTES / 2)[i % HALF16] =
        make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < ATT_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], ATT_CWARPS * 32);  // every consumer lane releases its own reads
    }
    mbar_init(mbar, 1);
    mbar_init(mbar + 1, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ep_full[i], ATT_CWARPS * 32);  // every writer lane publishes its own stores
      mbar_init(&ep_empty[i], 32);
    }
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (DENSE && threadIdx.x == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
  }
  pdl_wait();  // inputs (work list, q) are produced by the previous kernel

  const int P = gridDim.x, cta = blockIdx.x;
  // debug stamps of CTA 0 (tlog != nullptr): [0] after pdl_wait, [2+t] tile t issued,
  // [18+t] tile t consumed, [34] kernel end
  auto stamp = [&](int i) {
    if (a.tlog && cta == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      a.tlog[192 + i] = t_;
    }
  };
  if (threadIdx.x == 0) stamp(0);
  if (threadIdx.x == 0) tl_mark(a.tlog, 4, 1, blockIdx.x == 0);
  if (a.tlog && threadIdx.x == 0 && 2 * cta + 1 < 512) {  // per-CTA start / end (debug)
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    a.tlog[512 + 2 * cta] = t_;
  }
  int ntile_dbg = 0;
  // unit-aligned split: CTA cta works on one unit only (see UnitSplit); otherwise the
  // global token range split (needs unit_prefix)
  constexpr bool unit_mode = UNIT;
  // every unit's work list in smem (sparse, unit-aligned split, when it fits): rows then
  // prefixes, two bulk copies of 16-byte multiples (the arrays carry 4 ints of padding)
  const size_t rows_n = (size_t)a.units * a.C, pref_n = (size_t)a.units * (a.C + 1);
  const size_t rows_pad = (rows_n + 3) & ~(size_t)3, pref_pad = (pref_n + 3) & ~(size_t)3;
  const bool all_lists = !DENSE && unit_mode && rows_pad + pref_pad <= (size_t)LIST_INTS;
  const int* pref_src = a.seg_prefix;
  if (all_lists && threadIdx.x == 0) {
    fence_proxy_async_global();
    mbar_arrive_expect_tx(mbar + 1, (uint32_t)((rows_pad + pref_pad) * 4));
    bulk_g2s(s_list, a.seg_row, (uint32_t)(rows_pad * 4), mbar + 1);
    bulk_g2s(s_list + rows_pad, a.seg_prefix, (uint32_t)(pref_pad * 4), mbar + 1);
  }
  // the split needs only the per-unit totals: read them from L2 while the lists land
  UnitSplit us_ = {0, 0, 1, 0, 0, 0};
  if (unit_mode) {
    const bool s32 = a.units <= 32 && (long long)(a.n + a.tail_len) * a.units * P < (1LL << 31);
    us_ = s32 ? unit_split_fast<DENSE>(a, cta, P, !DENSE && a.mref != nullptr && a.dm_ok)
              : unit_split_of<DENSE>(a, cta, P, pref_src);
  }
  if (all_lists) {
    mbar_wait(mbar + 1, 0);
    if (threadIdx.x == 0) stamp(45);
  }
  if (threadIdx.x == 0) stamp(40);
  // sparse global split: every unit carries ATT_PIECE_TOKENS virtual tokens after its work
  // list, so the split prices the fixed cost of a piece (combine, arrival, merge); a CTA
  // whose range holds only virtual tokens of a unit contributes an empty piece
  const long long X = (!DENSE && !unit_mode) ? ATT_PIECE_TOKENS : 0;
  auto vpre = [&](int v) -> long long { return a.unit_prefix[v] + (long long)v * X; };
  const long long T = unit_mode ? 0 : (DENSE ? dense_total : vpre(a.units));
  // unit-aligned sparse split: the CTA's unit's whole work list into smem with one round
  // trip of independent loads (all threads), so the producer's segment search and run
  // walk never wait on L2
  const bool list_smem = !DENSE && unit_mode;
  if (list_smem && !all_lists) {
    const int* gr = a.seg_row + (size_t)us_.u * a.C;
    const int* gp = a.seg_prefix + (size_t)us_.u * (a.C + 1);
    constexpr int PER = 16;  // independent loads in flight per thread (2 C + 1 <= 2560: one batch)
    for (int i0 = 0; i0 < 2 * a.C + 1; i0 += PER * ATT_THREADS) {
      int v[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int i = i0 + k * ATT_THREADS + threadIdx.x;
        v[k] = i < a.C ? __ldcg(gr + i) : (i < 2 * a.C + 1 ? __ldcg(gp + (i - a.C)) : 0);
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int i = i0 + k * ATT_THREADS + threadIdx.x;
        if (i < 2 * a.C + 1) s_list[i] = v[k];
      }
    }
    if (threadIdx.x == 0) stamp(41);
    __syncthreads();
    if (threadIdx.x == 0) stamp(42);
  }

  if (warp == 0) {
    // ============================ producer (warp-uniform control flow) ============================
    const bool leader = lane == 0;
    // one run of consecutive layout rows into stage slots [slot, slot + len): the index
    // layout (rows < n) or the recent-token tail (rows n..)
    auto issue_run = [&](uint8_t* sK, uint8_t* sV, int slot, int row, int len, int u, uint64_t* bar) {
      const uint8_t* kb;
      const uint8_t* vb;
      const int ku = a.kv_div > 1 ? u / a.kv_div : u;  // the K/V unit (per-head ablation)
      if (row >= a.n) {
        const size_t o = ((size_t)ku * a.tail_cap + (row - a.n)) * 256;
        kb = (const uint8_t*)a.Kt + o;
        vb = (const uint8_t*)a.Vt + o;
      } else {
        const size_t o = ((size_t)ku * a.n + row) * 256;
        kb = (const uint8_t*)a.Kp + o;
        vb = (const uint8_t*)a.Vp + o;
      }
      bulk_g2s(sK + slot * 256, kb, (uint32_t)len * 256u, bar);
      bulk_g2s(sV + slot * 256, vb, (uint32_t)len * 256u, bar);
    };
    int stage = 0;
    uint32_t phase = 0;
    // the global split: CTA cta covers tokens [rs(cta), rs(cta + 1)) of the unit stream
    long long t = unit_mode ? 0 : range_start(cta, T, P);
    const long long t_end = unit_mode ? 0 : range_start(cta + 1, T, P);
    int u = us_.u;
    if (!unit_mode && t < t_end) {
      if (DENSE) {
        u = (int)(t / a.n);
      } else {  // largest u with unit_prefix[u] + u X <= t
        u = warp_floor_search_off(a.unit_prefix, a.units, t, X);
      }
    }
    bool more = unit_mode || t < t_end;
    bool pf_ok = false;
    int pf_row = 0, pf_end = 0, pf_tot = 0;
    while (more) {
      long long pend = 0;
      int lt, le;
      if (unit_mode) {
        lt = us_.lo;
        le = us_.hi;
      } else {
        const long long ubase = DENSE ? (long long)u * a.n : vpre(u);
        const long long uend = DENSE ? ubase + a.n : vpre(u + 1);
        pend = uend < t_end ? uend : t_end;
        lt = (int)(t - ubase);
        le = (int)(pend - ubase);
        if (X) {  // clip the virtual tokens
          const int real = (int)(a.unit_prefix[u + 1] - a.unit_prefix[u]);
          lt = lt < real ? lt : real;
          le = le < real ? le : real;
        }
      }
      if (lt >= le) {  // empty piece (T_v < n_v, or virtual tokens only): no tokens
        mbar_wait(&empty[stage], phase ^ 1);
        if (leader) {
          meta[stage].mask = 0;
          meta[stage].unit = u;
          meta[stage].flags = FLAG_FIRST | FLAG_LAST;
          mbar_arrive(&full[stage]);
        }
        if (++stage == nst) { stage = 0; phase ^= 1; }
        if (unit_mode) break;
        t = pend;
        ++u;
        more = t < t_end;
        pf_ok = false;
        continue;
      }
      // sparse: run table window of 32 segments (lane i holds segment k0 + i)
      const int* seg_row = all_lists ? s_list + (size_t)u * a.C
                           : list_smem ? s_list : a.seg_row + (size_t)u * a.C;
      const int* seg_pref = all_lists ? s_list + rows_pad + (size_t)u * (a.C + 1)
                            : list_smem ? s_list + a.C : a.seg_prefix + (size_t)u * (a.C + 1);
      int k = 0, k0 = 0, row = 0, left = 0, w_row = 0, w_end = 0;
      // the unit's list tokens; tokens past them are the recent-token tail (rows n..)
      const bool use_pf = !DENSE && pf_ok;  // this unit's head window was prefetched (lt = 0)
      const int ltot = DENSE ? 0 : (use_pf ? pf_tot : seg_pref[a.C]);
      if (!DENSE && lt >= ltot) {
        row = a.n + (lt - ltot);
        left = ltot + a.tail_len - lt;
      } else if (use_pf) {  // lt = 0: window at segment 0 (empty segments are stepped over)
        w_row = pf_row;
        w_end = pf_end;
        row = __shfl_sync(0xffffffffu, w_row, 0);
        left = __shfl_sync(0xffffffffu, w_end, 0);
      } else if (!DENSE) {
        if (leader) stamp(43);
        k = k0 = warp_floor_search<int>(seg_pref, a.C, lt);  // largest k with seg_pref[k] <= lt
        w_row = (k0 + lane < a.C) ? seg_row[k0 + lane] : 0;
        w_end = (k0 + lane < a.C) ? seg_pref[k0 + lane + 1] : 0;
        const int sp = seg_pref[k];
        row = __shfl_sync(0xffffffffu, w_row, 0) + (lt - sp);
        left = __shfl_sync(0xffffffffu, w_end, 0) - lt;
        if (leader) stamp(44);
      }
      // global split: when the range runs on into unit u + 1, load that unit's head window
      // now, so the unit switch does not wait on L2 (consumed in the next iteration)
      pf_ok = false;
      if (!DENSE && !unit_mode && pend < t_end && u + 1 < a.units) {
        const int* nr = a.seg_row + (size_t)(u + 1) * a.C;
        const int* npf = a.seg_prefix + (size_t)(u + 1) * (a.C + 1);
        pf_row = lane < a.C ? __ldcg(nr + lane) : 0;
        pf_end = lane < a.C ? __ldcg(npf + lane + 1) : 0;
        pf_tot = __ldcg(npf + a.C);
        pf_ok = true;
      }
      bool first = true;
      while (lt < le) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sK = stages + stage * ATT_STAGE_BYTES;
        uint8_t* sV = sK + ATT_STAGE_BYTES / 2;
        unsigned long long mask = 0;
        if (DENSE) {
          const int cnt = (le - lt) < ATT_TILE ? (le - lt) : ATT_TILE;
          mask = cnt == 64 ? ~0ull : ((1ull << cnt) - 1ull);
          if (leader) {
            meta[stage].mask = mask;
            meta[stage].unit = u;
            meta[stage].flags = (first ? FLAG_FIRST : 0) | (lt + cnt >= le ? FLAG_LAST : 0);
            mbar_arrive_expect_tx(&full[stage], ATT_STAGE_BYTES);
            const int b = u / a.Hkv, h = u % a.Hkv;
            tma_load_4d(sK, &tmK, 0, lt, h, b, &full[stage]);
            tma_load_4d(sK + 8192, &tmK, 64, lt, h, b, &full[stage]);
            tma_load_4d(sV, &tmV, 0, lt, h, b, &full[stage]);
            tma_load_4d(sV + 8192, &tmV, 64, lt, h, b, &full[stage]);
          }
          lt += cnt;
        } else {
          uint32_t bytes = 0;
          int s = 0;
          int r_slot = -1, r_row = 0, r_len = 0;  // pending run (merged while contiguous)
          (void)0;
          while (s < ATT_TILE && lt < le) {
            const int avail = left < (le - lt) ? left : (le - lt);
            const int s0 = s + ((row - s) & 7);
            if (s0 >= ATT_TILE) break;
            const int L = avail < (ATT_TILE - s0) ? avail : (ATT_TILE - s0);
            if (r_slot >= 0 && r_slot + r_len == s0 && r_row + r_len == row && (r_row >= a.n) == (row >= a.n)) {
              r_len += L;
            } else {
              if (r_slot >= 0 && leader) issue_run(sK, sV, r_slot, r_row, r_len, u, &full[stage]);
              r_slot = s0; r_row = row; r_len = L;
            }
            mask |= (L == 64 ? ~0ull : ((1ull << L) - 1ull)) << s0;
            bytes += (uint32_t)L * 512u;
            s = s0 + L;
            row += L;
            lt += L;
            left -= L;
            if (left == 0 && lt < le && lt >= ltot) {  // into the tail
              row = a.n + (lt - ltot);
              left = ltot + a.tail_len - lt;
            } else if (left == 0 && lt < le) {
              ++k;
              if (k - k0 == 32) {
                k0 = k;
                w_row = (k0 + lane < a.C) ? seg_row[k0 + lane] : 0;
                w_end = (k0 + lane < a.C) ? seg_pref[k0 + lane + 1] : 0;
              }
              row = __shfl_sync(0xffffffffu, w_row, k - k0);
              left = __shfl_sync(0xffffffffu, w_end, k - k0) - lt;
            }
          }
          if (leader) {
            issue_run(sK, sV, r_slot, r_row, r_len, u, &full[stage]);
            meta[stage].mask = mask;
            meta[stage].unit = u;
            meta[stage].flags = (first ? FLAG_FIRST : 0) | (lt >= le ? FLAG_LAST : 0);
            mbar_arrive_expect_tx(&full[stage], bytes);
          }
        }
        first = false;
        if (leader && ntile_dbg < 16) stamp(2 + ntile_dbg);
        ++ntile_dbg;
        if (++stage == nst) { stage = 0; phase ^= 1; }
      }
      if (unit_mode) break;
      t = pend;
      ++u;
      more = t < t_end;
    }
    // end marker
    mbar_wait(&empty[stage], phase ^ 1);
    if (leader) {
      meta[stage].flags = FLAG_END;
      meta[stage].mask = 0;
      meta[stage].unit = -1;
      mbar_arrive(&full[stage]);
    }
    return;
  }

  if (warp == ATT_EPI_WARP) {
    // ============================ piece epilogue (global split) ============================
    // The consumers hand each finished piece (per-warp m, l, o) over in one of two smem
    // buffers and go on streaming; this warp combines it across the consumer warps, writes
    // the partial, counts the unit's arrival and, for the unit's last piece, merges (S9).
    if (unit_mode) return;  // one piece per CTA: the consumers finish it themselves
    for (int ne = 0;; ++ne) {
      const int b = ne & 1;
      mbar_wait(&ep_full[b], (uint32_t)((ne >> 1) & 1));
      const int u = ep_meta[b];
      if (u < 0) break;
      const size_t slot = (size_t)cta + u;  // cta + unit: unique per piece (ranges are contiguous)
      const float* base = ep_buf + b * SCRATCH_FLOATS;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float mw[ATT_CWARPS], mf = -INFINITY;
#pragma unroll
        for (int w = 0; w < ATT_CWARPS; ++w) {
          mw[w] = base[w * (8 * 128 + 16) + 8 * 128 + g];
          mf = fmaxf(mf, mw[w]);
        }
        const bool none = mf == -INFINITY;  // empty piece: zero weight in the merge
        float lf = 0.f;
        float4 of = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < ATT_CWARPS; ++w) {
          const float* sww = base + w * (8 * 128 + 16);
          const float e = none ? 0.f : exp2f(mw[w] - mf);
          lf += sww[8 * 128 + 8 + g] * e;
          const float4 v = reinterpret_cast<const float4*>(sww + g * 128)[lane];
          of.x = fmaf(v.x, e, of.x);
          of.y = fmaf(v.y, e, of.y);
          of.z = fmaf(v.z, e, of.z);
          of.w = fmaf(v.w, e, of.w);
        }
        const float il = none ? 0.f : 1.f / lf;
        reinterpret_cast<float4*>(a.part_o + (slot * G + g) * 128)[lane] =
            make_float4(of.x * il, of.y * il, of.z * il, of.w * il);
        if (lane == 0) a.part_lse[slot * G + g] = none ? -INFINITY : (mf + log2f(lf)) * 0.6931471805599453f;
      }
      mbar_arrive(&ep_empty[b]);
      // arrival: __syncwarp orders the lanes' partial stores before lane 0's gpu-scope
      // release; the last arrival acquires, and __syncwarp passes that on to the lanes
      const long long us = DENSE ? (long long)u * a.n : vpre(u);
      const long long ue = DENSE ? us + a.n : vpre(u + 1);
      int c0 = 0;
      const int np = pieces_of_unit(us, ue, T, P, &c0);
      int last = 0;
      if (lane == 0) last = atom_add_acq_rel_gpu(&a.unit_cnt[u], 1) == np - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      __syncwarp();
      if (last) {
        const int span = cta_of(ue - 1, T, P) - c0 + 1;
        for (int g = 0; g < G; ++g) merge_head_global<G>(a, u, g, c0, span, u, false, T, P);
        if (lane == 0) a.unit_cnt[u] = 0;  // self-reset for the next call
      }
    }
    return;
  }

  // ============================ consumers ============================
  const int cw = warp - 1;
  const int ct = threadIdx.x - 32;          // 0..127 consumer thread index
  const int h0 = 2 * (lane & 3);            // heads held by this lane in C fragments
  const int r0 = lane >> 2;                 // token row (S^T) / dim row (O^T) in fragment
  const float scale_log2 = 1.4426950408889634f * 0.08838834764831845f;  // log2(e)/sqrt(128)
  uint32_t qb[8][2];
  float mr[G];  // reference shift of the piece's unit (reference-shift merge)
  float own_o[G], own_l[1];  // this CTA's scaled share, head-major (designated merger keeps it)
  int own_flag = 0;
  const bool dm = us_.dm != 0;
  float o[8][4];
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  int cur_unit = -1;
  int ep_n = 0;  // pieces handed to the epilogue warp
  int stage = 0;
  uint32_t phase = 0;

  const uint32_t sbase = smem_u32(stages);
  const int a_slot = cw * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;  // K, ldmatrix non-trans
  const int a_chi = lane >> 4;
  const int v_slot = cw * 16 + (lane & 7) + (lane >> 4) * 8;         // V, ldmatrix trans
  const int v_chi = (lane >> 3) & 1;

  while (true) {
    mbar_wait(&full[stage], phase);
    const StageMeta md = meta[stage];
    if (ct == 0 && ntile_dbg < 16) stamp(18 + ntile_dbg);
    ++ntile_dbg;
    if (md.flags & FLAG_END) break;
    if (md.flags & FLAG_FIRST) {
      if (md.unit != cur_unit) {
        cur_unit = md.unit;
        const __nv_bfloat16* qu = a.q + (size_t)cur_unit * G * 128;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          if (r0 < G) {  // B fragment: n = lane/4 (head), k = 2*(lane%4)
            const uint32_t* qrow = reinterpret_cast<const uint32_t*>(qu + r0 * 128);
            qb[ks][0] = qrow[(ks * 16 + h0) >> 1];
            qb[ks][1] = qrow[(ks * 16 + 8 + h0) >> 1];
          } else {
            qb[ks][0] = 0u;
            qb[ks][1] = 0u;
          }
        }
        if (a.mref) {
#pragma unroll
          for (int g = 0; g < G; ++g) mr[g] = __ldg(a.mref + (size_t)cur_unit * G + g);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
    }
    const uint32_t mym = (uint32_t)((md.mask >> (cw * 16)) & 0xFFFFull);
    if (mym) {
      const uint32_t sK = sbase + stage * ATT_STAGE_BYTES;
      const uint32_t sV = sK + ATT_STAGE_BYTES / 2;
      float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t af[4];
        ldsm_x4(af[0], af[1], af[2], af[3], sK + tile_off<DENSE>(a_slot, 2 * ks + a_chi));
        mma_bf16_16816(s, af, qb[ks][0], qb[ks][1]);
      }
      // s[0],s[1]: token r0, heads h0,h0+1 ; s[2],s[3]: token r0+8
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
      const float c0 = exp2f(m0 - mn0), c1 = exp2f(m1 - mn1);  // m = -inf -> 0
      m0 = mn0;
      m1 = mn1;
      const float p0 = exp2f(x0 - mn0), p1 = exp2f(x1 - mn1);
      const float p2 = exp2f(x2 - mn0), p3 = exp2f(x3 - mn1);
      l0 = l0 * c0 + p0 + p2;
      l1 = l1 * c1 + p1 + p3;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        o[i][0] *= c0; o[i][1] *= c1; o[i][2] *= c0; o[i][3] *= c1;
      }
      const uint32_t b0 = movmatrix_t(pack_bf16(p0, p1));
      const uint32_t b1 = movmatrix_t(pack_bf16(p2, p3));
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t af[4];
        ldsm_x4_t(af[0], af[1], af[2], af[3], sV + tile_off<DENSE>(v_slot, 2 * mt + v_chi));
        mma_bf16_16816(o[mt], af, b0, b1);
      }
    }
    mbar_arrive(&empty[stage]);
    if (++stage == nst) { stage = 0; phase ^= 1; }

    if (md.flags & FLAG_LAST) {
      unsigned long long t_last0 = 0;
      if (a.tlog && ct == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_last0));
      // ---- cross-warp combine of this piece -> partial slot (cta + unit)
      float L0 = l0, L1 = l1;
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        L0 += __shfl_xor_sync(0xffffffffu, L0, off);
        L1 += __shfl_xor_sync(0xffffffffu, L1, off);
      }
      int ep_b = 0;
      if (!unit_mode) {  // hand the piece to the epilogue warp (buffer ep_n & 1)
        ep_b = ep_n & 1;
        mbar_wait(&ep_empty[ep_b], (uint32_t)(((ep_n >> 1) & 1) ^ 1));
      }
      float* sw = (unit_mode ? scratch : ep_buf + ep_b * SCRATCH_FLOATS) + cw * (8 * 128 + 16);
      if (lane < 4) {
        sw[8 * 128 + h0] = m0;
        sw[8 * 128 + h0 + 1] = m1;
        sw[8 * 128 + 8 + h0] = L0;
        sw[8 * 128 + 8 + h0 + 1] = L1;
      }
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        const int d0 = mt * 16 + r0;
        sw[h0 * 128 + d0] = o[mt][0];
        sw[(h0 + 1) * 128 + d0] = o[mt][1];
        sw[h0 * 128 + d0 + 8] = o[mt][2];
        sw[(h0 + 1) * 128 + d0 + 8] = o[mt][3];
      }
      if (!unit_mode) {
        if (ct == 0) ep_meta[ep_b] = md.unit;
        mbar_arrive(&ep_full[ep_b]);
        ++ep_n;
      }
     if (unit_mode) {
      asm volatile("bar.sync 1, %0;" ::"n"(ATT_CWARPS * 32));
      const int u = md.unit;
      // partial slot: the CTA index (unit-aligned split: one piece per CTA) or cta + unit
      // (global split: a CTA may hold pieces of several units; c + u is unique)
      const size_t slot = unit_mode ? (size_t)cta : (size_t)cta + u;
      if (a.mref) {
        // reference-shift merge, head-major: thread ct combines head gh = ct / TPH, dims
        // [d0, d0 + G) (G values per thread, so the accumulator adds are G-wide vectors).
        // The piece's 2^(mf - mref) (o, l): a shift outside the window (the fp32 range of
        // the scaled sums) flags the head, and the merger then merges the partials
        // instead.  The designated merger keeps its own share in registers; every other
        // piece adds it into the unit's accumulators.
        constexpr int TPH = 128 / G;
        const int gh = ct / TPH, d0 = (ct % TPH) * G;
        float mf = -INFINITY;
#pragma unroll
        for (int w = 0; w < ATT_CWARPS; ++w) mf = fmaxf(mf, scratch[w * (8 * 128 + 16) + 8 * 128 + gh]);
        const bool none = mf == -INFINITY;  // empty piece: zero weight in the merge
        float lf = 0.f, of[G];
#pragma unroll
        for (int i = 0; i < G; ++i) of[i] = 0.f;
#pragma unroll
        for (int w = 0; w < ATT_CWARPS; ++w) {
          const float* sww = scratch + w * (8 * 128 + 16);
          const float e = none ? 0.f : exp2f(sww[8 * 128 + gh] - mf);
          lf += sww[8 * 128 + 8 + gh] * e;
#pragma unroll
          for (int i = 0; i < G; ++i) of[i] += sww[gh * 128 + d0 + i] * e;
        }
        const float il = none ? 0.f : 1.f / lf;
#pragma unroll
        for (int i = 0; i < G; ++i) a.part_o[(slot * G + gh) * 128 + d0 + i] = of[i] * il;
        if (ct % TPH == 0) a.part_lse[slot * G + gh] = none ? -INFINITY : (mf + log2f(lf)) * 0.6931471805599453f;
        const float d = mf - mr[gh];
        const bool inw = d >= -ACC_DMIN && d <= ACC_DMAX;
        const float sc = (none || !inw) ? 0.f : exp2f(d);
#pragma unroll
        for (int i = 0; i < G; ++i) own_o[i] = of[i] * sc;
        own_l[0] = lf * sc;
        if (!none && !inw) own_flag = 1;
        if (!(dm && us_.j == 0)) {
          float* acc = a.acc + ((size_t)u * G + gh) * ATT_ACC_ROW;
          if (!none && inw) {
            red_add_f32xG<G>(acc + d0, own_o);
            if (ct % TPH == 0) atomicAdd(acc + 128, own_l[0]);
          } else if (!none && ct % TPH == 0) {
            a.acc_flag[(size_t)u * G + gh] = 1;
          }
        }
      } else {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float mf = -INFINITY;
#pragma unroll
        for (int w = 0; w < ATT_CWARPS; ++w) mf = fmaxf(mf, scratch[w * (8 * 128 + 16) + 8 * 128 + g]);
        float lf = 0.f, of = 0.f;
#pragma unroll
        for (int w = 0; w < ATT_CWARPS; ++w) {
          const float* sww = scratch + w * (8 * 128 + 16);
          const float e = exp2f(sww[8 * 128 + g] - mf);
          lf += sww[8 * 128 + 8 + g] * e;
          of += sww[g * 128 + ct] * e;
        }
        const bool none = mf == -INFINITY;  // empty piece: zero weight in the merge
        a.part_o[(slot * G + g) * 128 + ct] = none ? 0.f : of / lf;
        if (ct == 0) a.part_lse[slot * G + g] = none ? -INFINITY : (mf + log2f(lf)) * 0.6931471805599453f;
      }
      }
      // ---- arrival.  The barrier orders every consumer thread's partial stores (and
      // accumulator adds) before thread 0's gpu-scope release (fences are cumulative).
      // Designated merger (reference shift, 32-bit split): CTA j = 0 of the unit (given a
      // shorter range) waits for the other n - 1 arrivals; the others release and leave.
      // Otherwise the last CTA to arrive (acq_rel atomic) merges.
      asm volatile("bar.sync 1, %0;" ::"n"(ATT_CWARPS * 32));
      long long ue = 0;
      int c0 = cta - us_.j, np = us_.n;
      if (!unit_mode) {
        const long long us = DENSE ? (long long)u * a.n : vpre(u);
        ue = DENSE ? us + a.n : vpre(u + 1);
        np = pieces_of_unit(us, ue, T, P, &c0);
      }
      if (ct == 0) {
        if (dm) {
          if (us_.j != 0) {
            red_release_gpu(&a.unit_cnt[u], 1);
            s_merge = 0;
          } else {
            while (ld_acquire_gpu(&a.unit_cnt[u]) < np - 1) {
            }
            s_merge = 1;
          }
        } else {
          const int prev = atom_add_acq_rel_gpu(&a.unit_cnt[u], 1);
          s_merge = (prev == np - 1);
        }
        if (s_merge && !a.mref && smem_merge_ok<G>(unit_mode, np)) {
          // the unit's partials are contiguous slots [c0, c0 + np): one bulk copy of the
          // o rows and one of the lse values into the (now idle) stage buffers
          fence_proxy_async_global();
          // (lse: from the 16-byte aligned slot at or below c0 G; the merge skips the head)
          const int l0 = (c0 * G) & 3;
          const uint32_t ob = (uint32_t)(np * G * 128 * 4), lb = (uint32_t)(((l0 + np * G) * 4 + 15) & ~15);
          mbar_arrive_expect_tx(mbar, ob + lb);
          bulk_g2s(stages + 1024, a.part_o + (size_t)c0 * G * 128, ob, mbar);
          bulk_g2s(stages, a.part_lse + ((size_t)c0 * G - l0), lb, mbar);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(ATT_CWARPS * 32));
      if (a.tlog && ct == 0 && cta < 512) {  // debug: the CTA's unit, index, CTAs of the unit; release time
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        a.tlog[3600 + cta] = (unsigned long long)u | ((unsigned long long)us_.j << 16) | ((unsigned long long)us_.n << 32);
        a.tlog[3800 + cta] = t_;  // after the arrival (release / poll)
        a.tlog[5200 + cta] = (unsigned long long)(us_.hi - us_.lo);  // the CTA's tokens
      }
      if (s_merge && a.tlog && ct == 0 && u < 8) {  // debug: merge start
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        a.tlog[964 + 2 * u] = t_;
      }
      bool merged = false;
      if (s_merge && a.mref) {
        // ---- S9 by the reference shift: the accumulators hold sum_c 2^(m_c - mref) (o_c, l_c)
        // over every piece (the arrival's acquire orders them); thread ct reads dim ct of
        // every head, then resets the accumulators for the next call
        constexpr int TPH = 128 / G;
        const int gh = ct / TPH, d0 = (ct % TPH) * G;
        float* acc = a.acc + ((size_t)u * G + gh) * ATT_ACC_ROW;
        float ov[G];
        ld_cg_f32xG<G>(acc + d0, ov);
        float lv = __ldcg(acc + 128);
        int fl = own_flag;
#pragma unroll
        for (int g = 0; g < G; ++g) fl |= __ldcg(a.acc_flag + (size_t)u * G + g);
        if (dm && us_.j == 0) {  // the merger's own share (not in the accumulators)
#pragma unroll
          for (int i = 0; i < G; ++i) ov[i] += own_o[i];
          lv += own_l[0];
        }
        fl |= lv > 0.f ? 0 : 1;
        // every read before the resets; the OR over the CTA's threads makes the choice of
        // merge uniform (a flag or an empty head anywhere -> the partial merge)
        fl = bar_red_or(fl);
#pragma unroll
        for (int i = 0; i < G; ++i) acc[d0 + i] = 0.f;
        if (ct % TPH == 0) {
          acc[128] = 0.f;
          a.acc_flag[(size_t)u * G + gh] = 0;
        }
        if (dm && ct == 0) a.unit_cnt[u] = 0;
        if (!fl) {
          const float inv = 1.f / lv;
          const size_t orow = ((size_t)u * G + gh) * 128 + d0;
          if (a.out) {
#pragma unroll
            for (int i = 0; i < G; i += 2) {
              if (G == 1) a.out[orow] = __float2bfloat16_rn(ov[0] * inv);
              else *reinterpret_cast<__nv_bfloat162*>(a.out + orow + i) = __floats2bfloat162_rn(ov[i] * inv, ov[i + (G > 1)] * inv);
            }
          }
          if (a.out_f32) {
#pragma unroll
            for (int i = 0; i < G; ++i) a.out_f32[orow + i] = ov[i] * inv;
          }
          if (a.lse && ct % TPH == 0) a.lse[(size_t)u * G + gh] = (mr[gh] + log2f(lv)) * 0.6931471805599453f;
          if (ct == 0) a.unit_cnt[u] = 0;  // self-reset for the next call
          merged = true;
        }
      }
      if (merged) {
      } else if (s_merge && !a.mref && smem_merge_ok<G>(unit_mode, np)) {
        // ---- S9 (unit-aligned split): merge the staged pieces from shared memory
        mbar_wait(mbar, 0);
        if (a.tlog && ct == 0 && u < 8) {  // debug: pieces staged
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          a.tlog[980 + u] = t_;
          a.tlog[990 + u] = (unsigned long long)np;
        }
        float* sl = reinterpret_cast<float*>(stages) + ((c0 * G) & 3);
        const float4* so = reinterpret_cast<const float4*>(stages + 1024);
        for (int g = cw; g < G; g += ATT_CWARPS) {
          float mx = -INFINITY;
          for (int i = lane; i < np; i += 32) mx = fmaxf(mx, sl[i * G + g]);
          mx = warp_max(mx);
          // piece weights one per lane, written over the lse they come from (each element
          // is read and written by the same lane), then the o rows in two FMA chains
          float sum = 0.f;
          for (int i = lane; i < np; i += 32) {
            const float l = sl[i * G + g];
            const float w = l > -INFINITY ? __expf(l - mx) : 0.f;
            sl[i * G + g] = w;
            sum += w;
          }
          sum = warp_sum(sum);
          __syncwarp();
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f), acc1 = make_float4(0.f, 0.f, 0.f, 0.f);
          int i = 0;
#pragma unroll 2
          for (; i + 1 < np; i += 2) {
            const float w0 = sl[i * G + g], w1 = sl[(i + 1) * G + g];
            const float4 v0 = so[((size_t)i * G + g) * 32 + lane];
            const float4 v1 = so[((size_t)(i + 1) * G + g) * 32 + lane];
            acc.x = fmaf(w0, v0.x, acc.x);
            acc.y = fmaf(w0, v0.y, acc.y);
            acc.z = fmaf(w0, v0.z, acc.z);
            acc.w = fmaf(w0, v0.w, acc.w);
            acc1.x = fmaf(w1, v1.x, acc1.x);
            acc1.y = fmaf(w1, v1.y, acc1.y);
            acc1.z = fmaf(w1, v1.z, acc1.z);
            acc1.w = fmaf(w1, v1.w, acc1.w);
          }
          if (i < np) {
            const float w0 = sl[i * G + g];
            const float4 v0 = so[((size_t)i * G + g) * 32 + lane];
            acc.x = fmaf(w0, v0.x, acc.x);
            acc.y = fmaf(w0, v0.y, acc.y);
            acc.z = fmaf(w0, v0.z, acc.z);
            acc.w = fmaf(w0, v0.w, acc.w);
          }
          acc.x += acc1.x;
          acc.y += acc1.y;
          acc.z += acc1.z;
          acc.w += acc1.w;
          const float inv = 1.f / sum;
          const size_t orow = ((size_t)u * G + g) * 128 + lane * 4;
          if (a.out) {
            __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(a.out + orow);
            ob[0] = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
            ob[1] = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
          }
          if (a.out_f32)
            *reinterpret_cast<float4*>(a.out_f32 + orow) =
                make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
          if (a.lse && lane == 0) a.lse[(size_t)u * G + g] = mx + logf(sum);
        }
        if (ct == 0) a.unit_cnt[u] = 0;  // self-reset for the next call
        if (a.tlog && ct == 0 && u < 8) {
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          a.tlog[965 + 2 * u] = t_;
        }
      } else if (s_merge) {
        // ---- S9: merge this unit's pieces (slots c + u), LSE-weighted
        // warp w merges heads w, w+4, ...; lanes hold 4 dims; piece weights are computed
        // 32 at a time (one per lane) and broadcast, so the o loads are independent.
        const int span = unit_mode ? np : cta_of(ue - 1, T, P) - c0 + 1;
        const int soff = unit_mode ? 0 : u;  // slot = c + soff
        for (int g = cw; g < G; g += ATT_CWARPS) merge_head_global<G>(a, u, g, c0, span, soff, unit_mode, T, P);
        if (ct == 0) a.unit_cnt[u] = 0;  // self-reset for the next call
        if (a.tlog && ct == 0 && u < 8) {
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          a.tlog[965 + 2 * u] = t_;
        }
      }
     }
      if (a.tlog && ct == 0 && cta < 148) {  // debug: time in piece ends / merges, merge count
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        a.tlog[2100 + cta] += t_ - t_last0;
        a.tlog[2300 + cta] += (unit_mode && s_merge) ? 1ull : 0ull;
        a.tlog[2500 + cta] += 1ull;
      }
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    }
  }
  if (!unit_mode) {  // end marker for the epilogue warp
    const int b = ep_n & 1;
    mbar_wait(&ep_empty[b], (uint32_t)(((ep_n >> 1) & 1) ^ 1));
    if (ct == 0) ep_meta[b] = -1;
    mbar_arrive(&ep_full[b]);
  }
  if (ct == 0) stamp(34);
  if (a.tlog && ct == 0 && 2 * cta + 1 < 512) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    a.tlog[512 + 2 * cta + 1] = t_;
    a.tlog[816 + cta] = (unsigned long long)ntile_dbg;
  }
  if (ct == 0) tl_mark(a.tlog, 4, 2, cta == 0);
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------- plain merge
__global__ void lse_merge_plain_kernel(const float* __restrict__ o_parts, const float* __restrict__ lse_parts,
                                       int n_parts, int n_rows, __nv_bfloat16* __restrict__ out,
                                       float* __restrict__ lse_out) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  float mx = -INFINITY, sum = 0.f;
  for (int s = 0; s < n_parts; ++s) {
    const float l = lse_parts[(size_t)s * n_rows + row];
    if (l == -INFINITY) continue;
    const float4 ov = *reinterpret_cast<const float4*>(o_parts + ((size_t)s * n_rows + row) * 128 + lane * 4);
    const float mn = fmaxf(mx, l);
    const float sc = expf(mx - mn), w = expf(l - mn);
    acc[0] = acc[0] * sc + w * ov.x;
    acc[1] = acc[1] * sc + w * ov.y;
    acc[2] = acc[2] * sc + w * ov.z;
    acc[3] = acc[3] * sc + w * ov.w;
    sum = sum * sc + w;
    mx = mn;
  }
  const float inv = sum > 0.f ? 1.f / sum : 0.f;
  __nv_bfloat162* orow = reinterpret_cast<__nv_bfloat162*>(out + (size_t)row * 128 + lane * 4);
  orow[0] = __floats2bfloat162_rn(acc[0] * inv, acc[1] * inv);
  orow[1] = __floats2bfloat162_rn(acc[2] * inv, acc[3] * inv);
  if (lse_out && lane == 0) lse_out[row] = sum > 0.f ? mx + logf(sum) : -INFINITY;
}

// ---------------------------------------------------------------------------- launchers
template <int G, bool DENSE>
static cudaError_t launch_attn_t(const AttnArgs& a, const CUtensorMap* tmK, const CUtensorMap* tmV,
                                 long long dense_total, int num_ctas, cudaStream_t s, bool pdl) {
  auto kern = a.unit_split ? attention_kernel<G, DENSE, true> : attention_kernel<G, DENSE, false>;
  cudaError_t e = func_smem_optin((const void*)kern, ATT_SMEM);
  if (e != cudaSuccess) return e;
  CUtensorMap dummy;
  memset(&dummy, 0, sizeof(dummy));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_ctas);
  cfg.blockDim = dim3(ATT_THREADS);
  cfg.dynamicSmemBytes = ATT_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a, tmK ? *tmK : dummy, tmV ? *tmV : dummy, dense_total);
}

template <bool DENSE>
static cudaError_t launch_attn_g(const AttnArgs& a, const CUtensorMap* tmK, const CUtensorMap* tmV, int G,
                                 int num_ctas, cudaStream_t s, bool pdl) {
  const long long dt = (long long)a.units * a.n;
  switch (G) {
    case 1: return launch_attn_t<1, DENSE>(a, tmK, tmV, dt, num_ctas, s, pdl);
    case 2: return launch_attn_t<2, DENSE>(a, tmK, tmV, dt, num_ctas, s, pdl);
    case 4: return launch_attn_t<4, DENSE>(a, tmK, tmV, dt, num_ctas, s, pdl);
    case 8: return launch_attn_t<8, DENSE>(a, tmK, tmV, dt, num_ctas, s, pdl);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_attention_sparse(const AttnArgs& a, int G, int num_ctas, cudaStream_t s, bool pdl) {
  return launch_attn_g<false>(a, nullptr, nullptr, G, num_ctas, s, pdl);
}
cudaError_t launch_attention_dense(const AttnArgs& a, const CUtensorMap* tmK, const CUtensorMap* tmV, int G,
                                   int num_ctas, cudaStream_t s, bool pdl) {
  return launch_attn_g<true>(a, tmK, tmV, G, num_ctas, s, pdl);
}

cudaError_t launch_lse_merge_plain(const float* o_parts, const float* lse_parts, int n_parts, int n_rows,
                                   __nv_bfloat16* out, float* lse, cudaStream_t s) {
  lse_merge_plain_kernel<<<(n_rows + 7) / 8, 256, 0, s>>>(o_parts, lse_parts, n_parts, n_rows, out, lse);
  return cudaGetLastError();
}

}  // namespace tactic
