// internal.h -- index structure and kernel launchers shared by the libtactic sources.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <string>

#include "../../include/tactic.h"

namespace tactic {

constexpr int D = 128;

// Sample constants of Alg. 1 (readings 8-10): exact head N, window centres x1, x2,
// half-width w, exact fallback for tiny n.  Integer formulas so every party agrees.
struct SampleConsts {
  int N, x1, x2, w;
  bool fallback;
  int slots;  // logits computed per head: N + 2(2w+1), or n in fallback
};
// n tokens, fractions from params (nullable: defaults); false on out-of-range fractions
bool sample_consts(int n, const tactic_params_t* params, SampleConsts* out);
// programmatic dependent launch between the decode kernels (TACTIC_NO_PDL=1 disables)
bool pdl_enabled();
// Dynamic shared-memory opt-in of kernel `fn` for at least `bytes` on the CURRENT device
// (function attributes are per device; cached per (fn, device), thread-safe);
// nonportable_cluster also allows clusters of more than 8 CTAs.
cudaError_t func_smem_optin(const void* fn, size_t bytes, bool nonportable_cluster = false);

// Unit-aligned attention split applies when every unit can get >= 2 CTAs; otherwise the
// attention kernel cuts the global token list (and the fit kernel computes unit_prefix).
inline bool unit_split_ok(int units, int ctas) { return 2 * units <= ctas; }

// debug timestamps (TACTIC_TLOG=1): per-kernel-specific slots below 1536, then a
// timeline of the decode kernels at TL_BASE + 4k: first CTA start, first CTA past
// griddepcontrol.wait, last CTA end (atomicMax); k = 0 score, 1 rank, 2 sample, 3 fit,
// 4 attention
constexpr int TL_BASE = 1536;
inline size_t tlog_entries(int units) { return (size_t)(units * 128 > 8192 ? units * 128 : 8192); }
#ifdef __CUDACC__
// what: 0 start, 1 past the wait (first CTA only), 2 end (every CTA; the max survives).
// Called by one thread per CTA.
__device__ __forceinline__ void tl_mark(unsigned long long* tl, int k, int what, bool first_cta) {
  if (!tl) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (what < 2) {
    if (first_cta) tl[TL_BASE + 4 * k + what] = t;
  } else {
    atomicMax(&tl[TL_BASE + 4 * k + 2], t);
  }
}
#endif

// Token-range split of a global work list over P CTAs: CTA c owns [rs(c), rs(c+1)).
__host__ __device__ inline long long range_start(int c, long long T, int P) {
  return (long long)c * T / P;
}
// CTA whose range contains token t (0 <= t < T): largest c with rs(c) <= t.
__host__ __device__ inline int cta_of(long long t, long long T, int P) {
  long long c = ((t + 1) * (long long)P - 1) / T;
  return (int)(c < P - 1 ? c : P - 1);
}

}  // namespace tactic

struct tactic_index_s {
  int device = 0;
  int B = 0, Hkv = 0, G = 0, n = 0, C = 0, units = 0, iters_req = 0;
  int num_ctas = 0, num_sms = 0;
  tactic::SampleConsts sc{};
  // index data
  __nv_bfloat16* Kp = nullptr;   // [units][n][128] cluster-contiguous, rows chunk-swizzled
  __nv_bfloat16* Vp = nullptr;
  float* cent = nullptr;         // [units][C][128] float32 centroids (storage format)
  int* offsets = nullptr;        // [units][C+1]
  int* perm = nullptr;           // [units][n] original token ids in layout order
  int* assign = nullptr;         // [units][n]
  int* iters_run = nullptr;      // [units]
  int* all_list = nullptr;       // [units][C]  rows of non-empty clusters (p >= 1 work list)
  int* unit_cnt = nullptr;       // [units] attention arrival counters
  int* all_prefix = nullptr;     // [units][C+1]
  long long* all_unit_prefix = nullptr;  // [units+1]
  // recent-token tail: tokens appended after the build,
  // attended in full by every decode; rows n .. n+tail_len-1 of each unit, stored in
  // separate [units][tail_cap][128] buffers with the same row swizzle as Kp/Vp
  __nv_bfloat16* Kt = nullptr;
  __nv_bfloat16* Vt = nullptr;
  int tail_len = 0, tail_cap = 0;
  // decode workspace
  double* crit = nullptr;        // [units][G][C]
  int* order = nullptr;          // [units][G][C]
  int* ends = nullptr;           // [units][G][C]
  int* rowmap = nullptr;         // [units][G][slots] layout row of every sampled slot
  float* summ = nullptr;         // [units][G][nb][4] per-sample-block fit summaries
  int* head_list = nullptr;      // [units*G][C]   per-head work lists (NEXT 2 ablation)
  int* head_prefix = nullptr;    // [units*G][C+1]
  int* head_cnt2 = nullptr;      // [units*G] attention arrival counters of the ablation
  int fixed_budget = 0;          // > 0 during tactic_decode_fixed_budget (NEXT 4 baseline)
  uint32_t options = 0;          // TACTIC_OPT_* (tactic_index_set_options)
  float* logits = nullptr;       // [units][G][slots]
  double* fit = nullptr;         // [units][G][6]
  int* J = nullptr;              // [units][G]
  uint8_t* umask = nullptr;      // [units][C]
  int* union_list = nullptr;     // [units][C] first layout row of each union segment
  int* union_prefix = nullptr;   // [units][C+1]
  long long* unit_prefix = nullptr;  // [units+1]
  unsigned int* counter = nullptr;   // last-block counter (self-resetting)
  float* part_o = nullptr;       // [num_ctas + units][G][128]
  float* part_lse = nullptr;     // [num_ctas + units][G]
  // reference-shift merge (attention.cu): per-head shift written by the fit, the fp32
  // accumulators the pieces add into, and the per-head out-of-window flags (all zero
  // between calls: the merging CTA resets them)
  float* mref = nullptr;         // [units][G] log2-domain shift (the fit's sampled max m)
  float* acc = nullptr;          // [units][G][132]: sum of 2^(m_c - mref) (o_c, l_c)
  int* acc_flag = nullptr;       // [units][G]
  double* stage = nullptr;       // sharded stage 1 -> 1b: [units][G][2] (E_N, 0)
  __nv_bfloat16* q_stage = nullptr;  // [units][G][128] (host-buffer decode)
  __nv_bfloat16* o_stage = nullptr;
  long long device_bytes = 0;
  cudaEvent_t ev_build[2] = {nullptr, nullptr};  // around the build's kernels (info.build_gpu_ms)
  int fz_checked_m = 0;           // one-launch decode: 0 unchecked, -1 no cluster shape fits, else M
  bool lists_valid = false;      // a p < 1 selection has been enqueued (attention-only needs its lists)
  // tactic_decode_host: the H2D copy, the decode and the D2H copy captured as one CUDA graph,
  // re-captured when its key (host buffers, p, tail length, options) changes
  cudaGraphExec_t hg_exec = nullptr;
  cudaStream_t hg_stream = nullptr;
  const void* hg_q = nullptr;
  void* hg_o = nullptr;
  float hg_p = 0.f;
  int hg_tail = -1;
  uint32_t hg_opts = 0;
  bool hg_failed = false;        // capture not possible for this key (e.g. pageable host memory)
  unsigned long long* tlog = nullptr;  // [units][16][8] phase timestamps (TACTIC_TLOG=1)
};

namespace tactic {


// ---- attention (attention.cu)
// sparse global split: virtual tokens per unit that stand for a piece's fixed cost
// (the epilogue warp takes the combine, arrival and merge off the consumers; what is left
// is the pipeline bubble at a unit switch and the epilogue backlog of short pieces)
constexpr int ATT_PIECE_TOKENS = 128;
struct AttnArgs {
  const __nv_bfloat16* q;          // [units][G][128]
  const __nv_bfloat16* Kp;         // sparse mode: swizzled [units][n][128]
  const __nv_bfloat16* Vp;
  const int* seg_row;              // [units][C] first layout row of each work-list segment
  const int* seg_prefix;           // [units][C+1] token prefix over the segments
  const long long* unit_prefix;    // [units+1] (sparse)
  int n, C, units, Hkv;
  float* part_o;                   // [num_ctas + units][G][128]
  float* part_lse;                 // [num_ctas + units][G]
  int* unit_cnt;                   // [units] arrival counters, zero between calls
  // reference-shift merge (unit-aligned split only; nullptr: the partial merge)
  const float* mref;               // [units][G] log2-domain shift per head
  float* acc;                      // [units][G][132] (o[128], l), zero between calls
  int* acc_flag;                   // [units][G] a piece fell outside the shift window
  __nv_bfloat16* out;              // nullable [units][G][128]
  float* out_f32;                  // nullable
  float* lse;                      // nullable [units][G]
  unsigned long long* tlog;        // nullable debug timestamps (CTA 0)
  int unit_split;                  // 1: unit-aligned split from seg_prefix totals (units <= CTAs/2)
  // recent-token tail (sparse): tail_len tokens per unit after each unit's work list,
  // rows n.. of Kt/Vt ([units][tail_cap][128])
  const __nv_bfloat16* Kt;
  const __nv_bfloat16* Vt;
  int tail_len, tail_cap;
  // per-head loading ablation (NEXT 2): work-list units are (unit, head) pairs with G = 1,
  // reading the K/V of unit u / kv_div (0 or 1: units are KV units)
  int kv_div;
  // the designated-merger protocol (a unit's CTA 0 polls for the others' arrivals) only when
  // the whole grid fits on the device at once (num_ctas <= SMs), so a polling CTA never
  // holds an SM that one of the CTAs it waits for needs
  int dm_ok;
};
cudaError_t launch_attention_sparse(const AttnArgs& a, int G, int num_ctas, cudaStream_t s, bool pdl);
cudaError_t launch_attention_dense(const AttnArgs& a, const CUtensorMap* tmK, const CUtensorMap* tmV, int G,
                                   int num_ctas, cudaStream_t s, bool pdl);
cudaError_t launch_lse_merge_plain(const float* o_parts, const float* lse_parts, int n_parts, int n_rows,
                                   __nv_bfloat16* out, float* lse, cudaStream_t s);
size_t attention_smem_bytes();

// ---- recent-token tail and new-token assignment (tail.cu)
cudaError_t launch_tail_append(const __nv_bfloat16* k_new, const __nv_bfloat16* v_new, int t, tactic_index_s* x,
                               cudaStream_t s);
cudaError_t launch_assign(const __nv_bfloat16* k, int t, const tactic_index_s* x, int* assign, cudaStream_t s);
cudaError_t launch_unit_prefix_fill(long long* up, int units, long long per_unit, cudaStream_t s);
// per-head work lists order[0..J_g) of every (unit, head) (NEXT 2 ablation)
cudaError_t launch_head_lists(const tactic_index_s* x, cudaStream_t s);
// ---- Table-1 diagnostics (diag.cu)
cudaError_t launch_exact_logits(const __nv_bfloat16* q, const tactic_index_s* x, float* logits, cudaStream_t s);

// ---- selection (select.cu)
struct SelArgs {
  const __nv_bfloat16* q;
  tactic_index_s* idx;
  double p;
  int mode;                        // 0 = Alg. 1, 1 = sharded stage 2 (theta*), 2 = sharded stage 1
  const double* gmax;              // [units][G][2] (stage 2 / 1b)
  const double* gmass;             // [units][G][1+T]
  double* mass_out;                // stage 1b
  double* local_max;               // stage 1
};
cudaError_t launch_score(const SelArgs& a, cudaStream_t s, bool pdl);
// S1 for every (unit, head) into x->crit (score_kernel), q: [units][G][128]
cudaError_t launch_score_all(const __nv_bfloat16* q, tactic_index_s* x, cudaStream_t s, bool pdl);
// S1 + S2 + S3 (rank_cluster.cu): crit, order, ends, sampled-slot row map
// q_copy (nullable): CTA 0 of every (unit, head) stores q there (q in mapped host memory)
cudaError_t launch_score_rank(const __nv_bfloat16* q, tactic_index_s* x, cudaStream_t s, bool pdl,
                              __nv_bfloat16* q_copy = nullptr);
bool score_rank_prescored(const tactic_index_s* x);  // S1 runs in score_kernel first (C3)
cudaError_t launch_sample(const SelArgs& a, cudaStream_t s, bool pdl);
cudaError_t launch_fit(const SelArgs& a, cudaStream_t s, bool pdl);
int sample_blocks(int slots);
// dynamic shared memory of the fit kernel (every decode with p < 1) and of the sharded
// stages' select kernel; checked against the device's opt-in limit at build / import
size_t fit_smem_bytes(const tactic_index_s* x, bool windows_exact);
size_t stage1b_smem_bytes(const tactic_index_s* x);
cudaError_t launch_stage1b(const SelArgs& a, cudaStream_t s);
// ---- the whole decode step in one cluster launch (decode_fused.cu)
struct FusedArgs {
  const __nv_bfloat16* q;          // [units][G][128]
  const float* cent;               // [units][C][128]
  const int* offsets;              // [units][C+1]
  const __nv_bfloat16* Kp;         // [units][n][128] cluster-contiguous, rows swizzled
  const __nv_bfloat16* Vp;
  const __nv_bfloat16* Kt;         // recent-token tail [units][tail_cap][128] (nullable)
  const __nv_bfloat16* Vt;
  int n, C, units, tail_len, tail_cap;
  SampleConsts sc;
  float p;                         // target fraction, < 1
  int fixed_budget;                // > 0: Quest-like token budget per head (NEXT 4)
  // selection outputs (the multi-kernel path's layout)
  double* crit;                    // [units][G][C]
  int* order;                      // [units][G][C]
  int* ends;                       // [units][G][C]
  float* logits;                   // [units][G][slots]
  double* fit;                     // [units][G][6]
  int* J;                          // [units][G]
  uint8_t* umask;                  // [units][C]
  int* ulist;                      // [units][C]
  int* uprefix;                    // [units][C+1]
  long long* unit_prefix;          // nullable [units+1] (global attention split consumers)
  unsigned int* unit_cnt;          // arrival counter for unit_prefix (zero between calls)
  __nv_bfloat16* out;              // nullable [units][G][128]
  float* out_f32;                  // nullable
  float* lse;                      // nullable [units][G]
  unsigned long long* tlog;        // nullable debug stamps
  int dbg_stop;                    // debug: leave after this phase (0 = run to the end)
};
// M clusters per CTA (64 or 128), R = ceil(C / M) CTAs per cluster (<= 16)
cudaError_t launch_decode_fused(const FusedArgs& a, int G, int M, int R, cudaStream_t s);
int fused_max_active_clusters(int G, int M, int R);
size_t fused_smem_bytes(int M);

// ---- k-means / layout (kmeans.cu)
struct KmArgs {
  const __nv_bfloat16* K;
  const __nv_bfloat16* V;
  long long sb, sh, sn;            // strides in elements
  int B, Hkv, n, C, Cpad, units, nblk, iters_req;
  // index buffers (device pointers)
  float* cent;
  int* offsets;
  int* perm;
  int* assign;
  int* iters_run;
  int* all_list;
  int* all_prefix;
  __nv_bfloat16* Kp;
  __nv_bfloat16* Vp;
  // scratch
  uint8_t* bimg;                   // [units][Cpad/128][64 KB]
  float* cnorm;                    // [units][Cpad]
  int* blk_counts;                 // [units][nblk][C]
  int* col_tot;                    // [units][C] cluster sizes (km_scan -> km_scatter)
  int* changed;                    // [units]
  int* converged;                  // [units]
  double* acc;                     // nullable [units][C][128]: B3 member sums (zero between uses)
};
cudaError_t km_init_centroids(const KmArgs& a, const int* init_dev, cudaStream_t s);
// tmK: 4-D map of the caller's K ([B][Hkv][n][128], box 64 dims x 128 rows, SWIZZLE_128B)
cudaError_t km_assign(const KmArgs& a, const CUtensorMap* tmK, int iter, bool simt, cudaStream_t s);
cudaError_t km_count_scan_scatter(const KmArgs& a, int iter, cudaStream_t s);
cudaError_t km_update(const KmArgs& a, int iter, cudaStream_t s);
cudaError_t km_finalize(const KmArgs& a, cudaStream_t s);
cudaError_t km_inertia(const KmArgs& a, double* part /* [units][C] */, cudaStream_t s);
cudaError_t km_check_finite(const KmArgs& a, int* flag, cudaStream_t s);

}  // namespace tactic
