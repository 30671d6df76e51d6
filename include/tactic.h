/*
 * tactic.h -- C ABI of the B200-native Tactic decode-time sparse attention library
 * (libtactic.so, hand-written sm_100a CUDA).
 *
 * Method: "Tactic: Adaptive Sparse Attention with Clustering and Distribution
 * Fitting for Long-Context LLMs" (arXiv 2502.12216).  Citations `P:n` are lines of
 * PAPER.md; "reading k" refers to the numbered readings in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Head dimension d is fixed at 128.  bf16 tensors are IEEE bfloat16 bit patterns.
 *  - A *unit* is one (sequence b, KV head h), numbered u = b * num_kv_heads + h.  Its G
 *    query heads are q-heads h*G .. h*G+G-1 of sequence b (GQA), so every
 *    q / out tensor is laid out [B][Hq = Hkv*G][128] == [units][G][128].
 *  - Unless stated otherwise pointers are CUDA device pointers on the current device and
 *    calls are asynchronous and stream-ordered on `stream` (a cudaStream_t, passed as
 *    void* so this header needs no CUDA include).  No entry point synchronises the device
 *    except where it says "host outputs".
 *  - Every call returns a tactic_status_t; no exception crosses the ABI.  A human-readable
 *    detail of the last failure on the calling thread is returned by tactic_last_error().
 *    Asynchronous kernel faults surface as TACTIC_ERR_CUDA at a later call.
 *  - Decode calls on one index share that index's device workspace: serialise them on one
 *    stream (the workspace makes the call CUDA-graph capturable: no allocation, no sync).
 */
#ifndef TACTIC_H_
#define TACTIC_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TACTIC_HEAD_DIM 128
#define TACTIC_MAX_CLUSTERS 4096      /* per unit (sort / selection kernels keep C in smem) */
#define TACTIC_MAX_SEQ_LEN 1048576    /* per unit (exact-head prefix of Alg. 1 kept in smem) */
#define TACTIC_SHARD_GRID_T 512       /* sequence-sharded mode: criticality grid points   */
#define TACTIC_SHARD_GRID_STEP 0.0625 /* grid step in logit units (1/16), reading 23      */
#define TACTIC_TAIL_CAPACITY 2048     /* default recent-token tail per unit (re-cluster
                                         every 2048 generated tokens)                      */

typedef enum {
  TACTIC_OK = 0,
  TACTIC_ERR_INVALID_ARGUMENT = 1, /* bad scalar (C, iters, p, G ...) or null pointer      */
  TACTIC_ERR_SHAPE = 2,            /* tensor shapes / strides inconsistent with the index  */
  TACTIC_ERR_OOM = 3,              /* device allocation failed                            */
  TACTIC_ERR_CUDA = 4,             /* CUDA runtime / kernel error                         */
  TACTIC_ERR_NOT_FINITE = 5,       /* TACTIC_FLAG_VALIDATE found NaN/Inf in K or V        */
  TACTIC_ERR_UNSUPPORTED = 6       /* device is not sm_100 or a size limit is exceeded    */
} tactic_status_t;

typedef struct tactic_index_s* tactic_index_t; /* opaque; owns every device buffer it allocates */

/* KV-cache descriptor.  Strides are in elements; 0 means the contiguous default
 * [B][Hkv][n][128] (stride_n = 128, stride_h = n*128, stride_b = Hkv*n*128).
 * stride_n must be a multiple of 8 (16-byte rows) and the last dimension contiguous. */
typedef struct {
  int32_t batch;
  int32_t num_kv_heads;
  int32_t group_size;   /* G: query heads per KV head, one of 1, 2, 4, 8            */
  int32_t seq_len;      /* n, tokens per unit (>= 1, <= TACTIC_MAX_SEQ_LEN)           */
  int32_t head_dim;     /* must be 128                                               */
  int64_t stride_b, stride_h, stride_n;
} tactic_kv_desc_t;

#define TACTIC_FLAG_VALIDATE     1u  /* build/import: scan K,V for NaN/Inf first   */
#define TACTIC_FLAG_KMEANS_SIMT  2u  /* build: CUDA-core assignment kernel instead of the
                                        tcgen05 one (debug / cross-check only)             */

typedef struct {
  uint64_t seed;                /* k-means init sampler seed (reading 3)                 */
  const int32_t* init_indices;  /* nullable HOST pointer [units][C]: caller-chosen init
                                   token indices; NULL = SplitMix64 + Fisher-Yates
                                   sampler seeded with seed + (u+1)*0x9E3779B97F4A7C15   */
  uint32_t flags;               /* TACTIC_FLAG_*                                          */
  int32_t num_ctas;             /* attention grid size; 0 = number of SMs                 */
  /* Alg. 1 sampling fractions (0 = the default in brackets):
   *   exact_frac        share of the sorted tokens whose weights are exact ("1-2% of
   *                     total tokens"; reading 10: [0.02])
   *   p1, p2            window centres as shares of n ("e.g., 10% and 60%";
   *                     [0.10], [0.60]), 0 < p1 < p2 < 1
   *   window_half_frac  window half-width as a share of n (reading 8: [0.0025])
   * Each fraction is quantised to parts per million, f -> round(f * 1e6), and the index
   * derives (integer arithmetic, identical in the oracle):
   *   N = ceil(e n / 1e6),  x_k = round_half_up(p_k n / 1e6),  w = max(1, round_half_up(h n / 1e6));
   * the windows [x_k - w, x_k + w] must not collide with the head, each other or the end,
   * else every rank is exact (tiny n).  Fixed at build / import; see
   * tactic_sample_constants.  Out of range: TACTIC_ERR_INVALID_ARGUMENT.               */
  float exact_frac, p1, p2, window_half_frac;
  /* global number of this index's unit 0 for the init sampler's seeding (default 0): a
   * rank that holds units [u0, u1) of a batch x KV-head sharded layer passes u0 and draws
   * the same initial centroids as a single index over all units would. */
  int32_t unit_offset;
} tactic_params_t;

/* The integer constants of Alg. 1's sampling for sequence length n (see tactic_params_t):
 * exact head N, window centres x1 < x2, half-width w, fallback = 1 when every rank is
 * exact (windows collide), slots = logits computed per head (N + 2(2w + 1), or n).     */
typedef struct {
  int32_t N, x1, x2, w, fallback, slots;
} tactic_sample_constants_t;

typedef struct {
  int32_t units, batch, num_kv_heads, group_size, seq_len, n_clusters;
  int32_t iters_requested;
  int32_t select_cluster_size;  /* CTAs per thread-block cluster of the one-launch decode
                                   (TACTIC_OPT_CLUSTER_DECODE, see tactic_decode); 0 = this
                                   index decodes through the multi-kernel chain          */
  int64_t device_bytes;         /* bytes the index holds on the device                   */
  float build_gpu_ms;           /* device time of the build's kernels (first k-means launch
                                   to the end of the layout), from CUDA events the library
                                   records on the build stream -- host work (allocation,
                                   launch) excluded; waits for the build to finish; -1 if
                                   unavailable                                           */
} tactic_index_info_t;

/* ---------------------------------------------------------------------------------------
 * Index build (after prefill).  P:363-364 (§4.2): per unit, k-means over the keys --
 * init by sampling C tokens uniformly without replacement (no k-means++, P:364 footnote),
 * then Lloyd iterations (assign every key to the nearest centroid by squared Euclidean
 * distance, reading 4; centroids := member means; an empty cluster keeps its centroid,
 * reading 6) until the assignment is unchanged or `iters` iterations (P:364, P:402:
 * 10).  The keys and values are then copied into a cluster-contiguous layout (clusters in
 * id order, tokens of a cluster in ascending position; "non-contiguous KV access").
 *
 *   K, V      device bf16, layout per `kv`.  Only read; the caller may free / overwrite
 *             them once the stream has passed this call.
 *   n_clusters C, 1 <= C <= min(seq_len, TACTIC_MAX_CLUSTERS)   (else INVALID_ARGUMENT)
 *   iters     >= 1
 *   params    nullable (defaults: seed 0, sampler init, no flags, default sampling)
 *   out       receives the new index (NULL on failure).
 * TACTIC_ERR_UNSUPPORTED when the per-unit selection state (G x C order and end ranks,
 * the sampled-slot summaries) exceeds one CTA's shared memory, e.g. G = 8 with C > ~3000
 * (tactic_index_set_options checks the windows-exact variant the same way).
 * The assignment GEMM runs on tcgen05 tensor cores (bf16 keys x split-bf16 centroids,
 * fp32 accumulate, fused argmin epilogue).  The call enqueues work only; it allocates
 * device memory (not capturable).                                                     */
tactic_status_t tactic_build_index(const void* K, const void* V, const tactic_kv_desc_t* kv,
                                   int32_t n_clusters, int32_t iters,
                                   const tactic_params_t* params, void* stream,
                                   tactic_index_t* out);

/* Index from a caller-supplied clustering (parity feeding, checkpoint restore).
 *   centroids HOST float32 [units][C][128]; assign HOST int32 [units][n] in [0, C).
 * Centroids are stored as given (float32 is the index storage format, reading 18).
 * Synchronises the stream before returning (host inputs are staged).                 */
tactic_status_t tactic_index_import(const void* K, const void* V, const tactic_kv_desc_t* kv,
                                    int32_t n_clusters, const float* centroids,
                                    const int32_t* assign, const tactic_params_t* params,
                                    void* stream, tactic_index_t* out);

/* Host outputs (each nullable): centroids float32 [units][C][128], assign int32
 * [units][n], inertia float64 [units] (sum_i |K_i - c_a(i)|^2, fp64 accumulation),
 * iters_run int32 [units].  Synchronises the stream.                                  */
tactic_status_t tactic_index_export(tactic_index_t idx, float* centroids, int32_t* assign,
                                    double* inertia, int32_t* iters_run, void* stream);

tactic_status_t tactic_index_info(tactic_index_t idx, tactic_index_info_t* info);
/* Host-only (no device work): the sampling constants for n tokens under `params`
 * (nullable = defaults), or those an index uses.  INVALID_ARGUMENT on bad fractions or
 * n < 1.                                                                               */
tactic_status_t tactic_sample_constants(int32_t n, const tactic_params_t* params, tactic_sample_constants_t* out);
tactic_status_t tactic_index_sample_constants(tactic_index_t idx, tactic_sample_constants_t* out);
/* Debug: the %globaltimer / clock stamps the decode kernels leave in the index's timing
 * log (kernel timeline, per-phase stamps of CTA 0 of each kernel; tools/phase_timing.py
 * decodes them), host uint64 [count].  Only for indices created with the environment
 * variable TACTIC_TLOG=1; synchronises the device.                                   */
tactic_status_t tactic_index_debug_timing(tactic_index_t idx, uint64_t* host, int32_t count);
void tactic_index_destroy(tactic_index_t idx);

/* ---------------------------------------------------------------------------------------
 * Decode step (per layer-step, all units).  For every unit and each of its G query heads
 * (Alg. 1 is per query; reading 16):
 *  S1 criticality crit_j = q . c_j (float64),  S2 sort clusters by (-crit, j),
 *  S3 token ranks of the partially sorted list,  S4 exact logits q.k/sqrt(d) of the first
 *  N = ceil(0.02 n) ranks and of two windows of 2w+1 ranks around x1 = 10% and x2 = 60%
 *  (readings 8-10),  S5 fit y = a/x + b through the window means,
 *  S6 select clusters in order until the estimated cumulative mass reaches p of the
 *  estimated total (Alg. 1 l.10, cluster granularity reading 14; p >= 1 selects
 *  every cluster, reading 15),  S7 union over the G heads turned into a balanced
 *  token work list over all units (sub-requests),  S8 split-KV flash-decode
 *  of every head over the union (reading 17),  S9 log-sum-exp merge (by default every
 *  piece's share is expressed against the fit's sampled maximum logit and added into fp32
 *  accumulators -- see TACTIC_OPT_DETERMINISTIC for the bit-reproducible piece-order merge).
 * Execution: a chain of kernels (score/rank, sample, fit, attention; the later ones
 * overlap their prologues with programmatic dependent launch).  With
 * TACTIC_OPT_CLUSTER_DECODE (and G in {1,2,4,8}, C <= 2048, C x G <= 4096, default
 * selection rules) S1-S9 of every unit run in ONE launch instead, one thread-block
 * cluster of ceil(C / M) CTAs per unit (M = 64 or 128 clusters per CTA) exchanging
 * through distributed shared memory.  Both compute the same selection (parity-tested
 * against each other and the oracle); the selection outputs of tactic_decode_debug are
 * written by either.
 *   q    device bf16 [B][Hq][128]          p   0 < p <= 1  (else INVALID_ARGUMENT)
 *   out  device bf16 [B][Hq][128]          lse nullable device float32 [B][Hq] (natural log)
 */
tactic_status_t tactic_decode(const void* q, tactic_index_t idx, float p, void* out,
                              void* stream);
tactic_status_t tactic_decode_ex(const void* q, tactic_index_t idx, float p, void* out,
                                 float* lse, void* stream);

/* Same computation through HOST buffers: q_host bf16 [B][Hq][128] in, out_host bf16
 * [B][Hq][128] out; synchronises the stream (end-to-end user call).  With page-locked,
 * mapped buffers (cudaHostAlloc / torch pin_memory on a UVA system) and the multi-kernel
 * path (p < 1, no cluster decode, no prescoring) the transfers are zero-copy: the entry
 * kernel reads q over the bus (staging it for the later kernels) and the S9 merge writes
 * the output into out_host; otherwise q is copied in and the output copied back.  Either
 * way the call is captured once as one CUDA graph per (q_host, out_host, p, tail length,
 * options) and replayed by later calls with the same key (one launch per call); with
 * pageable buffers the capture is refused and the call falls back to stream-ordered
 * copies and launches.  TACTIC_HOST_COPIES=1 forces the copies.                      */
tactic_status_t tactic_decode_host(const void* q_host, tactic_index_t idx, float p,
                                   void* out_host, void* stream);

/* Decode with selection introspection (HOST outputs, each nullable; synchronises):
 *   order      int32 [units][G][C]   cluster ids in rank order (S2)
 *   J          int32 [units][G]      selected prefix length of `order` (S6)
 *   fit        float64 [units][G][6] (a, b, m, W, mu1, mu2)  (S4-S6)
 *   union_mask uint8 [units][C]      1 = cluster in the GQA union (S7)            */
tactic_status_t tactic_decode_debug(const void* q, tactic_index_t idx, float p, void* out,
                                    float* lse, int32_t* order, int32_t* J, double* fit,
                                    uint8_t* union_mask, void* stream);

/* Per-stage timing (Fig. 9-style breakdown): same work as tactic_decode_ex, but
 * records the caller's CUDA events (cudaEvent_t passed as void*) on `stream`:
 *   events[0] before S1, events[1] after S7 (selection), events[2] after S8 + S9 (the
 *   merge is fused into the attention kernel), events[3] right after events[2].
 *   n_events must be 4.  Stage boundaries are serialised.  */
tactic_status_t tactic_decode_profiled(const void* q, tactic_index_t idx, float p, void* out,
                                       void* const* events, int32_t n_events, void* stream);

/* Measurement aid: S8 + S9 alone (the sparse split-KV attention kernel with its fused
 * merge), over the work lists the last selection on this index left on the device (call
 * tactic_decode / tactic_decode_ex first with the same q; p < 1).  q, out: as in
 * tactic_decode.  Launched without a programmatic dependency, so back-to-back calls on
 * one stream time the kernel's launch duration.  Errors: TACTIC_ERR_INVALID_ARGUMENT on
 * NULL arguments or before the index's first p < 1 selection has been enqueued.        */
tactic_status_t tactic_decode_attention_only(const void* q, tactic_index_t idx, void* out, void* stream);

/* ---------------------------------------------------------------------------------------
 * The library's own dense baseline (full attention, Eq. 1-2):
 * split-KV flash-decode over all n tokens of every unit of the caller's K/V, then LSE
 * merge.  Needs a caller workspace of tactic_dense_workspace_size() bytes, zero-filled
 * once when allocated (it holds self-resetting arrival counters; the library leaves it
 * zeroed after every call).                                                           */
tactic_status_t tactic_dense_workspace_size(const tactic_kv_desc_t* kv, int32_t num_ctas,
                                            size_t* bytes);
tactic_status_t tactic_dense_decode(const void* q, const void* K, const void* V,
                                    const tactic_kv_desc_t* kv, void* out, float* lse,
                                    void* workspace, size_t workspace_bytes,
                                    int32_t num_ctas, void* stream);

/* S9 alone: o_parts float32 [n_parts][n_rows][128], lse_parts float32 [n_parts][n_rows]
 * (natural log; -inf marks an empty part) -> out bf16 [n_rows][128], lse nullable f32. */
tactic_status_t tactic_lse_merge(const float* o_parts, const float* lse_parts,
                                 int32_t n_parts, int32_t n_rows, void* out, float* lse,
                                 void* stream);

/* ---------------------------------------------------------------------------------------
 * Sequence-sharded mode (1M-token contexts; reading 23).  Each rank holds an index over
 * its token shard.  Per decode step:
 *   stage1  : local S1-S5; writes local_max float64 [units][G][2] = (m_s, theta_max_s),
 *             theta = crit/sqrt(d).                      -> caller all-reduces MAX
 *   stage1b : re-expresses the local fit in the global exponent frame; writes
 *             mass float64 [units][G][1+T] = (W_s, M_s(theta_t), t=1..T) on the grid
 *             theta_t = theta_max - t*STEP.               -> caller all-reduces SUM
 *   stage2  : theta* = largest theta_t with sum M >= p * sum W (none: select all);
 *             selects local clusters with theta >= theta*, S7-S9 locally; writes
 *             o_part float32 [units][G][128], lse_part float32 [units][G].
 *                                                         -> caller all-gathers, then
 *   tactic_lse_merge over the shards.                                                  */
tactic_status_t tactic_decode_stage1(const void* q, tactic_index_t idx, double* local_max,
                                     void* stream);
tactic_status_t tactic_decode_stage1b(tactic_index_t idx, const double* global_max,
                                      double* mass, void* stream);
tactic_status_t tactic_decode_stage2(const void* q, tactic_index_t idx, float p,
                                     const double* global_max, const double* global_mass,
                                     float* o_part, float* lse_part, void* stream);

/* ---------------------------------------------------------------------------------------
 * Multi-step generation.  P:112 (§1): Tactic "performs full
 * attention on newly generated tokens" and re-clusters periodically ("every ... 2048
 * tokens").  Tokens generated after the build are appended to a per-unit dense tail
 * that every later decode attends in full, after the selected clusters (the selection
 * S1-S7 still ranks only the clustered tokens; with p >= 1 the decode equals full
 * attention over the n + tail tokens).  When the tail is full the caller re-clusters:
 * builds a new index over the clustered + tail tokens (the Python DecodeSession policy).
 *
 * tactic_set_tail_capacity: (re)allocates room for `capacity` tail tokens per unit;
 *   only while the tail is empty (else INVALID_ARGUMENT).  0 frees it.  Not capturable.
 * tactic_append: appends t >= 0 tokens per unit.  k_new, v_new device bf16 [units][t][128]
 *   (unit u = b * Hkv + h, as for q).  Allocates the default capacity
 *   (TACTIC_TAIL_CAPACITY) on first use; SHAPE if the tail would overflow.  Decodes
 *   enqueued after it on the same stream see the tokens.  A CUDA graph captured before an
 *   append keeps the tail length of its capture: re-capture after appending.
 *   Sequence-sharded mode: append to ONE shard's index (the tail is attended by the shard
 *   that holds it, like any of its tokens; appending everywhere would count it per shard).
 * tactic_index_tail: host outputs (nullable) tail length / capacity.
 * tactic_assign_tokens: SPEC assign_token: for t new keys per unit
 *   (device bf16 [units][t][128]) the nearest centroid by squared Euclidean distance in
 *   float64, ties to the lowest id (readings 4, 7); device int32 [units][t].          */
tactic_status_t tactic_set_tail_capacity(tactic_index_t idx, int32_t capacity);
tactic_status_t tactic_append(tactic_index_t idx, const void* k_new, const void* v_new, int32_t t,
                              void* stream);
tactic_status_t tactic_index_tail(tactic_index_t idx, int32_t* len, int32_t* capacity);
tactic_status_t tactic_assign_tokens(tactic_index_t idx, const void* k, int32_t t, int32_t* assign,
                                     void* stream);

/* ---------------------------------------------------------------------------------------
 * Per-head loading ablation (SPEC's own-set
 * normalisation): the same selection as tactic_decode, but every query head
 * attends only ITS OWN selected clusters S_g (each KV token is loaded once per head that
 * selected it instead of once per KV head).  Same q / out layout as tactic_decode;
 * 0 < p < 1; needs units x G <= CTAs / 2 (else UNSUPPORTED).  Measurement of the GQA
 * union's benefit, not the method's output (which attends the union, reading 17).   */
tactic_status_t tactic_decode_per_head(const void* q, tactic_index_t idx, float p, void* out, void* stream);

/* Quest-like fixed-budget baseline ("uniformly chooses tokens
 * across attention heads", SPEC fixed_budget_select S:465): every head takes clusters in
 * criticality order until it holds `budget` tokens (rounded up to the cluster end, as
 * reading 14), 1 <= budget <= n; then the GQA-union attention (per_head = 0) or each
 * head over its own clusters (per_head = 1, same constraint as tactic_decode_per_head).
 * J: nullable HOST int32 [units][G] selected prefix lengths (synchronises if given).  */
tactic_status_t tactic_decode_fixed_budget(const void* q, tactic_index_t idx, int32_t budget, int32_t per_head,
                                           void* out, int32_t* J, void* stream);

/* Selection variants of later decodes on this index:
 *   TACTIC_OPT_WINDOWS_EXACT  SPEC's reading: the sampled window ranks
 *     [x_k - w, x_k + w] keep their exact weights in the estimated cumulative mass and in
 *     W (exact values take precedence over the fit, as for ranks <= N); the default is
 *     reading 11 (only ranks <= N exact).  0 restores the default.                     */
#define TACTIC_OPT_WINDOWS_EXACT 1u
/*   TACTIC_OPT_CLUSTER_DECODE  decode S1-S9 in one launch of per-unit thread-block
 *     clusters when the index qualifies (see tactic_decode).  Off by default: one unit's
 *     cluster streams at most ~60 GB/s per SM, so with few units (batch 1) the
 *     HBM-bound phases cannot spread over the whole chip.               */
#define TACTIC_OPT_CLUSTER_DECODE 2u
/*   TACTIC_OPT_DETERMINISTIC  S9 merges the unit's partials in piece order (bit-identical
 *     outputs from call to call).  The default merge adds every piece's share, shifted by
 *     the fit's sampled maximum logit (2^(m_c - m) (o_c, l_c)), into fp32 accumulators with
 *     atomic adds: ~1.5 us faster at C2, the output varies with the order of those adds
 *     within fp32 rounding (at most one bf16 rounding step).              */
#define TACTIC_OPT_DETERMINISTIC 4u
tactic_status_t tactic_index_set_options(tactic_index_t idx, uint32_t options);

/* ---------------------------------------------------------------------------------------
 * Table-1 diagnostics: the exact logit of every
 * clustered token for every query head, l = q . k / sqrt(d), in the index's LAYOUT order
 * (clusters in id order, tokens of a cluster ascending; cluster j occupies layout rows
 * [off_j, off_{j+1}) with off from the exported assignment's cluster sizes).
 *   q device bf16 [B][Hq][128];  logits device float32 [units][G][n].
 * Measurement tooling (Optimal / Cluster-Optimal budgets, achieved cumulative score),
 * not part of the decode path.                                                          */
tactic_status_t tactic_exact_logits(const void* q, tactic_index_t idx, float* logits, void* stream);

/* ---------------------------------------------------------------------------------------
 * Misc. */
const char* tactic_status_string(tactic_status_t s);
const char* tactic_last_error(void);             /* thread-local, never NULL            */
const char* tactic_version(void);
/* TACTIC_OK iff the current device is sm_100 (B200); fills SM count if non-NULL.     */
tactic_status_t tactic_device_check(int32_t* num_sms);

#ifdef __cplusplus
}
#endif
#endif /* TACTIC_H_ */
