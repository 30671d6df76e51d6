// tactic_api.cu -- the C ABI (include/tactic.h): argument validation, index ownership,
// host-side sampler, and the stream-ordered launch sequences of build and decode.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

using namespace tactic;

namespace {

thread_local std::string g_err = "";

tactic_status_t fail(tactic_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

tactic_status_t cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? TACTIC_ERR_OOM : TACTIC_ERR_CUDA, "%s: %s (%s)", where,
              cudaGetErrorString(e), cudaGetErrorName(e));
}

#define CK(expr)                                       \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

struct Resolved {
  int B, Hkv, G, n;
  long long sb, sh, sn;
};

tactic_status_t resolve_kv(const tactic_kv_desc_t* kv, Resolved* r) {
  if (!kv) return fail(TACTIC_ERR_INVALID_ARGUMENT, "kv descriptor is NULL");
  if (kv->head_dim != 128) return fail(TACTIC_ERR_INVALID_ARGUMENT, "head_dim must be 128 (got %d)", kv->head_dim);
  const int G = kv->group_size;
  if (!(G == 1 || G == 2 || G == 4 || G == 8))
    return fail(TACTIC_ERR_INVALID_ARGUMENT, "group_size must be 1, 2, 4 or 8 (got %d)", G);
  if (kv->batch < 1 || kv->num_kv_heads < 1) return fail(TACTIC_ERR_INVALID_ARGUMENT, "batch and heads must be >= 1");
  if (kv->seq_len < 1) return fail(TACTIC_ERR_INVALID_ARGUMENT, "seq_len must be >= 1");
  if (kv->seq_len > TACTIC_MAX_SEQ_LEN)
    return fail(TACTIC_ERR_UNSUPPORTED, "seq_len %d exceeds TACTIC_MAX_SEQ_LEN", kv->seq_len);
  r->B = kv->batch;
  r->Hkv = kv->num_kv_heads;
  r->G = G;
  r->n = kv->seq_len;
  r->sn = kv->stride_n ? kv->stride_n : 128;
  r->sh = kv->stride_h ? kv->stride_h : (long long)r->n * r->sn;
  r->sb = kv->stride_b ? kv->stride_b : (long long)r->Hkv * r->sh;
  if (r->sn % 8 || r->sh % 8 || r->sb % 8 || r->sn < 128)
    return fail(TACTIC_ERR_SHAPE, "strides must be multiples of 8 elements and stride_n >= 128");
  return TACTIC_OK;
}

uint64_t splitmix_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Reading 3: C distinct tokens, uniform without replacement -- partial Fisher-Yates
// driven by SplitMix64 seeded with seed + (unit+1) * 0x9E3779B97F4A7C15.
void sample_init(int n, int C, uint64_t seed, int unit, int* out) {
  uint64_t st = seed + (uint64_t)(unit + 1) * 0x9E3779B97F4A7C15ull;
  std::vector<int> a(n);
  for (int i = 0; i < n; ++i) a[i] = i;
  for (int j = 0; j < C; ++j) {
    const uint64_t r = (uint64_t)j + splitmix_next(st) % (uint64_t)(n - j);
    std::swap(a[j], a[(size_t)r]);
    out[j] = a[j];
  }
}

// Index memory: one device allocation carved into 256-byte aligned buffers (each with
// 16 bytes of slack).  Used twice over the same sequence of get() calls: a measuring pass
// (base == nullptr) that sizes the arena, then the carving pass -- one cudaMalloc per
// index instead of ~45 (large cudaMallocs dominate a build's host time otherwise).
struct DevAlloc {
  std::vector<void*> ptrs;
  long long bytes = 0;
  cudaError_t err = cudaSuccess;
  uint8_t* base = nullptr;
  size_t off = 0;
  template <typename T>
  T* get(size_t count) {
    if (err != cudaSuccess) return nullptr;
    const size_t b = (count * sizeof(T) + 16 + 255) & ~(size_t)255;
    const size_t o = off;
    off += b;
    bytes += (long long)b;
    return base ? (T*)(base + o) : (T*)(uintptr_t)256;  // measuring pass: a placeholder
  }
  bool reserve() {  // after the measuring pass: allocate and rewind
    void* p = nullptr;
    err = cudaMalloc(&p, off);
    if (err != cudaSuccess) return false;
    base = (uint8_t*)p;
    ptrs.push_back(p);
    off = 0;
    bytes = 0;
    return true;
  }
};

int device_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

namespace tactic {
cudaError_t func_smem_optin(const void* fn, size_t bytes, bool nonportable_cluster) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, std::pair<size_t, bool>> done;  // (bytes, non-portable)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto& have = done[{fn, dev}];
  if (have.first >= bytes && have.first > 0 && (have.second || !nonportable_cluster)) return cudaSuccess;
  if (have.first < bytes || have.first == 0) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    have.first = bytes > 0 ? bytes : 1;
  }
  if (nonportable_cluster && !have.second) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    have.second = true;
  }
  return cudaSuccess;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("TACTIC_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

// Readings 8-10 and tactic_params_t: fractions quantised to ppm, then integer rules.
static long long ppm_of(float f, float dflt) {
  const double v = (f == 0.0f ? dflt : f);
  if (!(v > 0.0) || !(v < 1.0)) return -1;
  return (long long)floor(v * 1e6 + 0.5);
}

bool sample_consts(int n, const tactic_params_t* params, SampleConsts* out) {
  const tactic_params_t d = {};
  const tactic_params_t* P = params ? params : &d;
  const long long e = ppm_of(P->exact_frac, 0.02f), q1 = ppm_of(P->p1, 0.10f), q2 = ppm_of(P->p2, 0.60f),
                  h = ppm_of(P->window_half_frac, 0.0025f);
  if (e < 1 || h < 1 || q1 < 1 || q2 <= q1 || q2 >= 1000000 || n < 1) return false;
  SampleConsts s;
  const long long nn = n;
  s.N = (int)((e * nn + 999999) / 1000000);
  s.x1 = (int)((2 * q1 * nn + 1000000) / 2000000);
  s.x2 = (int)((2 * q2 * nn + 1000000) / 2000000);
  const long long w = (2 * h * nn + 1000000) / 2000000;
  s.w = (int)(w > 1 ? w : 1);
  s.fallback = (s.x1 - s.w <= s.N) || (s.x1 + s.w >= s.x2 - s.w) || (s.x2 + s.w > n);
  s.slots = s.fallback ? n : s.N + 2 * (2 * s.w + 1);
  *out = s;
  return true;
}
}  // namespace tactic

struct tactic_index_priv {
  std::vector<void*> ptrs;
};

static void free_index(tactic_index_s* x, std::vector<void*>* ptrs) {
  for (cudaEvent_t e : x->ev_build)
    if (e) cudaEventDestroy(e);
  if (x->hg_exec) cudaGraphExecDestroy(x->hg_exec);
  if (x->hg_stream) cudaStreamDestroy(x->hg_stream);
  if (ptrs)
    for (void* p : *ptrs) cudaFree(p);
  delete x;
}

// all index allocations are recorded here (keyed by index pointer)
static bool getenv_flag(const char* name) {
  const char* e = getenv(name);
  return e && e[0] == '1';
}

static std::mutex g_mu;
static std::map<tactic_index_s*, std::vector<void*>> g_allocs;

static tactic_status_t alloc_index(const Resolved& r, int C, int iters, const tactic_params_t& prm,
                                   tactic_index_s** out) {
  const int num_ctas = prm.num_ctas;
  tactic_index_s* x = new tactic_index_s();
  x->B = r.B;
  x->Hkv = r.Hkv;
  x->G = r.G;
  x->n = r.n;
  x->C = C;
  x->units = r.B * r.Hkv;
  x->iters_req = iters;
  cudaGetDevice(&x->device);
  x->num_sms = device_sms();
  x->num_ctas = num_ctas > 0 ? num_ctas : x->num_sms;
  if (!sample_consts(r.n, &prm, &x->sc)) {
    delete x;
    return fail(TACTIC_ERR_INVALID_ARGUMENT, "sampling fractions out of range (0 < exact_frac, window_half_frac; "
                "0 < p1 < p2 < 1)");
  }
  const size_t U = x->units, n = x->n, G = x->G;
  DevAlloc A;
  auto carve = [&]() {
    x->Kp = A.get<__nv_bfloat16>(U * n * 128);
    x->Vp = A.get<__nv_bfloat16>(U * n * 128);
    x->cent = A.get<float>(U * C * 128);
    x->offsets = A.get<int>(U * (C + 1));
    x->perm = A.get<int>(U * n);
    x->assign = A.get<int>(U * n);
    x->iters_run = A.get<int>(U);
    x->all_list = A.get<int>(U * C);
    x->all_prefix = A.get<int>(U * (C + 1));
    x->all_unit_prefix = A.get<long long>(U + 1);
    x->crit = A.get<double>(U * G * C);
    x->order = A.get<int>(U * G * C);
    x->ends = A.get<int>(U * G * C);
    x->logits = A.get<float>(U * G * (size_t)x->sc.slots);
    x->fit = A.get<double>(U * G * 6);
    x->J = A.get<int>(U * G);
    x->umask = A.get<uint8_t>(U * C);
    x->union_list = A.get<int>(U * C + 4);          // +4: 16-byte bulk reads of the whole list
    x->union_prefix = A.get<int>(U * (C + 1) + 4);
    x->unit_prefix = A.get<long long>(U + 1);
    x->counter = A.get<unsigned int>(1);
    x->part_o = A.get<float>((x->num_ctas + U) * G * 128);
    x->part_lse = A.get<float>((x->num_ctas + U) * G + 4);  // +4: the merge's 16-byte bulk reads
    x->mref = A.get<float>(U * G);
    x->acc = A.get<float>(U * G * 132);
    x->acc_flag = A.get<int>(U * G);
    x->stage = A.get<double>(U * G * 2);
    x->q_stage = A.get<__nv_bfloat16>(U * G * 128);
    x->o_stage = A.get<__nv_bfloat16>(U * G * 128);
    x->unit_cnt = A.get<int>(U);
    x->head_list = A.get<int>(U * G * C + 4);
    x->head_prefix = A.get<int>(U * G * (C + 1) + 4);
    x->head_cnt2 = A.get<int>(U * G);
    x->rowmap = A.get<int>(U * G * (size_t)x->sc.slots);
    x->summ = A.get<float>(U * G * (size_t)sample_blocks(x->sc.slots) * 4);
  };
  carve();
  if (A.reserve()) carve();
  if (A.err != cudaSuccess) {
    for (void* p : A.ptrs) cudaFree(p);
    delete x;
    return cuda_fail(A.err, "index allocation");
  }
  x->device_bytes = A.bytes;
  {
    const char* tl = getenv("TACTIC_TLOG");
    if (tl && tl[0] == '1' && cudaMalloc((void**)&x->tlog, tlog_entries(U) * 8) == cudaSuccess) {
      cudaMemset(x->tlog, 0, tlog_entries(U) * 8);
      std::lock_guard<std::mutex> lk(g_mu);
      A.ptrs.push_back(x->tlog);
    }
  }
  cudaMemset(x->counter, 0, sizeof(unsigned int));
  cudaMemset(x->unit_cnt, 0, U * sizeof(int));
  cudaMemset(x->acc, 0, U * G * 132 * sizeof(float));
  cudaMemset(x->acc_flag, 0, U * G * sizeof(int));
  cudaMemset(x->head_cnt2, 0, U * G * sizeof(int));
  cudaMemset(x->order, 0, U * G * C * sizeof(int));  // valid cluster ids before the first decode

  cudaMemset(x->ends, 0, U * G * C * sizeof(int));
  cudaMemset(x->union_list, 0, (U * C + 4) * sizeof(int));   // valid (empty) work lists before
  cudaMemset(x->union_prefix, 0, (U * (C + 1) + 4) * sizeof(int));  // the first selection
  cudaMemset(x->unit_prefix, 0, (U + 1) * sizeof(long long));
  std::vector<long long> up(U + 1);
  for (size_t u = 0; u <= U; ++u) up[u] = (long long)u * (long long)n;
  cudaMemcpy(x->all_unit_prefix, up.data(), (U + 1) * sizeof(long long), cudaMemcpyHostToDevice);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_allocs[x] = A.ptrs;
  }
  *out = x;
  return TACTIC_OK;
}

static size_t smem_optin_limit() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return 227 * 1024;
  return (size_t)v;
}

// the per-unit selection keeps G x C order / end ranks and the per-block sample summaries
// in one CTA's shared memory (fit kernel); reject sizes that cannot launch
static tactic_status_t check_select_limits(const tactic_index_s* x, bool windows_exact) {
  const size_t need = fit_smem_bytes(x, windows_exact), lim = smem_optin_limit();
  if (need > lim)
    return fail(TACTIC_ERR_UNSUPPORTED,
                "selection needs %zu bytes of shared memory per unit (G = %d, C = %d, %d sampled slots%s) > %zu: "
                "reduce n_clusters or the group size", need, x->G, x->C, x->sc.slots,
                windows_exact ? ", windows-exact" : "", lim);
  return TACTIC_OK;
}

static tactic_status_t check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(TACTIC_ERR_UNSUPPORTED, "device %d is sm_%d%d; libtactic is built for sm_100a (B200)", dev, major,
                minor);
  return TACTIC_OK;
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encode() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled_t)p;
  }
  return fn;
}

static tactic_status_t make_kv_map(CUtensorMap* m, const void* base, const Resolved& r, int box_rows) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return fail(TACTIC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {128, (cuuint64_t)r.n, (cuuint64_t)r.Hkv, (cuuint64_t)r.B};
  cuuint64_t strides[3] = {(cuuint64_t)r.sn * 2, (cuuint64_t)r.sh * 2, (cuuint64_t)r.sb * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult cr = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(TACTIC_ERR_SHAPE, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
  return TACTIC_OK;
}


// Build / import share everything after the centroids are known.
static tactic_status_t build_common(const void* K, const void* V, const tactic_kv_desc_t* kv, int32_t C,
                                    int32_t iters, const tactic_params_t* params, cudaStream_t s,
                                    const float* host_cent, const int32_t* host_assign, tactic_index_t* out) {
  if (!out) return fail(TACTIC_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!K || !V) return fail(TACTIC_ERR_INVALID_ARGUMENT, "K or V is NULL");
  Resolved r;
  tactic_status_t st = resolve_kv(kv, &r);
  if (st) return st;
  if (C < 1 || C > r.n) return fail(TACTIC_ERR_INVALID_ARGUMENT, "n_clusters must be in [1, seq_len] (got %d)", C);
  if (C > TACTIC_MAX_CLUSTERS) return fail(TACTIC_ERR_UNSUPPORTED, "n_clusters %d > TACTIC_MAX_CLUSTERS", C);
  if (iters < 1) return fail(TACTIC_ERR_INVALID_ARGUMENT, "iters must be >= 1");
  if (params && params->unit_offset < 0) return fail(TACTIC_ERR_INVALID_ARGUMENT, "unit_offset < 0");
  if ((uintptr_t)K % 16 || (uintptr_t)V % 16) return fail(TACTIC_ERR_SHAPE, "K and V must be 16-byte aligned");
  if ((st = check_device())) return st;
  tactic_params_t P = {};
  if (params) P = *params;
  tactic_index_s* x = nullptr;
  if ((st = alloc_index(r, C, iters, P, &x))) return st;
  if ((st = check_select_limits(x, false))) {
    tactic_index_destroy(x);
    return st;
  }
  const int units = x->units;
  KmArgs a = {};
  a.K = (const __nv_bfloat16*)K;
  a.V = (const __nv_bfloat16*)V;
  a.sb = r.sb;
  a.sh = r.sh;
  a.sn = r.sn;
  a.B = r.B;
  a.Hkv = r.Hkv;
  a.n = r.n;
  a.C = C;
  a.Cpad = (C + 127) / 128 * 128;
  a.units = units;
  a.nblk = (r.n + 1023) / 1024;
  a.iters_req = iters;
  a.cent = x->cent;
  a.offsets = x->offsets;
  a.perm = x->perm;
  a.assign = x->assign;
  a.iters_run = x->iters_run;
  a.all_list = x->all_list;
  a.all_prefix = x->all_prefix;
  a.Kp = x->Kp;
  a.Vp = x->Vp;
  // scratch (stream-ordered)
  auto bail = [&](tactic_status_t s2) {
    tactic_index_destroy(x);
    return s2;
  };
  cudaError_t e;
  int* d_init = nullptr;
  int* d_flag = nullptr;
  const bool build = host_cent == nullptr;
  if ((e = cudaMallocAsync((void**)&a.bimg, (size_t)units * a.Cpad / 128 * 65536, s))) return bail(cuda_fail(e, "scratch"));
  if ((e = cudaMallocAsync((void**)&a.cnorm, (size_t)units * a.Cpad * 4, s))) return bail(cuda_fail(e, "scratch"));
  if ((e = cudaMallocAsync((void**)&a.blk_counts, (size_t)units * (a.nblk + 1) * C * 4, s))) return bail(cuda_fail(e, "scratch"));
  a.col_tot = a.blk_counts + (size_t)units * a.nblk * C;
  if ((e = cudaMallocAsync((void**)&a.changed, (size_t)(iters + 2) * units * 4, s))) return bail(cuda_fail(e, "scratch"));
  if ((e = cudaMallocAsync((void**)&a.converged, (size_t)units * 4, s))) return bail(cuda_fail(e, "scratch"));
  if ((e = cudaMallocAsync((void**)&d_init, (size_t)units * C * 4, s))) return bail(cuda_fail(e, "scratch"));
  if ((e = cudaMallocAsync((void**)&d_flag, 4, s))) return bail(cuda_fail(e, "scratch"));
  a.acc = nullptr;  // streamed B3 sums: 16-byte row slices, up to 64 MB of fp64 sums
  if (build && r.sn % 8 == 0 && r.sb % 8 == 0 && r.sh % 8 == 0 && ((uintptr_t)K & 15) == 0 &&
      (size_t)units * C * 128 * 8 <= (64u << 20) && !getenv_flag("TACTIC_KM_UPDATE_PER_CLUSTER")) {
    if ((e = cudaMallocAsync((void**)&a.acc, (size_t)units * C * 128 * 8, s))) return bail(cuda_fail(e, "scratch"));
    cudaMemsetAsync(a.acc, 0, (size_t)units * C * 128 * 8, s);
  }
  if (cudaEventCreate(&x->ev_build[0]) != cudaSuccess || cudaEventCreate(&x->ev_build[1]) != cudaSuccess) {
    cudaGetLastError();  // timing only: the build goes on without it
    for (cudaEvent_t& ev : x->ev_build)
      if (ev) { cudaEventDestroy(ev); ev = nullptr; }
  }
  cudaMemsetAsync(a.changed, 0, (size_t)(iters + 2) * units * 4, s);
  cudaMemsetAsync(a.converged, 0, (size_t)units * 4, s);
  cudaMemsetAsync(d_flag, 0, 4, s);
  cudaMemsetAsync(x->assign, 0xff, (size_t)units * r.n * 4, s);
  auto free_scratch = [&]() {
    cudaFreeAsync(a.bimg, s);
    cudaFreeAsync(a.cnorm, s);
    cudaFreeAsync(a.blk_counts, s);
    cudaFreeAsync(a.changed, s);
    cudaFreeAsync(a.converged, s);
    cudaFreeAsync(d_init, s);
    cudaFreeAsync(d_flag, s);
    if (a.acc) cudaFreeAsync(a.acc, s);
  };
#define CKB(expr)                                           \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) {                                \
      tactic_status_t _s = cuda_fail(_e, #expr);            \
      free_scratch();                                       \
      cudaStreamSynchronize(s);                             \
      return bail(_s);                                      \
    }                                                       \
  } while (0)
  if (P.flags & TACTIC_FLAG_VALIDATE) {
    CKB(km_check_finite(a, d_flag, s));
    int h = 0;
    CKB(cudaMemcpyAsync(&h, d_flag, 4, cudaMemcpyDeviceToHost, s));
    CKB(cudaStreamSynchronize(s));
    if (h) {
      free_scratch();
      return bail(fail(TACTIC_ERR_NOT_FINITE, "K or V contains NaN/Inf"));
    }
  }
  if (build) {
    CUtensorMap tmK;  // the assignment GEMM's A tiles (128 keys) straight from the caller's K
    if ((st = make_kv_map(&tmK, K, r, 128))) {
      free_scratch();
      cudaStreamSynchronize(s);
      return bail(st);
    }
    std::vector<int> init((size_t)units * C);
    for (int u = 0; u < units; ++u) {
      if (P.init_indices) {
        for (int j = 0; j < C; ++j) {
          const int t = P.init_indices[(size_t)u * C + j];
          if (t < 0 || t >= r.n) {
            free_scratch();
            return bail(fail(TACTIC_ERR_INVALID_ARGUMENT, "init_indices[%d][%d] = %d out of range", u, j, t));
          }
          init[(size_t)u * C + j] = t;
        }
      } else {
        sample_init(r.n, C, P.seed, P.unit_offset + u, &init[(size_t)u * C]);
      }
    }
    CKB(cudaMemcpyAsync(d_init, init.data(), init.size() * 4, cudaMemcpyHostToDevice, s));
    CKB(cudaStreamSynchronize(s));  // pageable staging buffer goes out of scope
    if (x->ev_build[0]) CKB(cudaEventRecord(x->ev_build[0], s));
    CKB(km_init_centroids(a, d_init, s));
    const bool simt = (P.flags & TACTIC_FLAG_KMEANS_SIMT) != 0;
    for (int it = 1; it <= iters; ++it) {
      CKB(km_assign(a, &tmK, it, simt, s));
      CKB(km_count_scan_scatter(a, it, s));
      CKB(km_update(a, it, s));
    }
  } else {
    for (size_t i = 0; i < (size_t)units * r.n; ++i)
      if (host_assign[i] < 0 || host_assign[i] >= C) {
        free_scratch();
        return bail(fail(TACTIC_ERR_INVALID_ARGUMENT, "assign[%zu] = %d out of [0, C)", i, host_assign[i]));
      }
    CKB(cudaMemcpyAsync(x->cent, host_cent, (size_t)units * C * 128 * 4, cudaMemcpyHostToDevice, s));
    CKB(cudaMemcpyAsync(x->assign, host_assign, (size_t)units * r.n * 4, cudaMemcpyHostToDevice, s));
    if (x->ev_build[0]) CKB(cudaEventRecord(x->ev_build[0], s));
    CKB(km_count_scan_scatter(a, 1, s));
    x->iters_req = 0;
    a.iters_req = 0;
  }
  CKB(km_finalize(a, s));
  if (x->ev_build[1]) CKB(cudaEventRecord(x->ev_build[1], s));
  free_scratch();
  if (!build) CKB(cudaStreamSynchronize(s));
#undef CKB
  *out = x;
  return TACTIC_OK;
}

extern "C" {
static bool fused_plan(tactic_index_t idx, int* M, int* R);


tactic_status_t tactic_build_index(const void* K, const void* V, const tactic_kv_desc_t* kv, int32_t n_clusters,
                                   int32_t iters, const tactic_params_t* params, void* stream,
                                   tactic_index_t* out) {
  return build_common(K, V, kv, n_clusters, iters, params, (cudaStream_t)stream, nullptr, nullptr, out);
}

tactic_status_t tactic_index_import(const void* K, const void* V, const tactic_kv_desc_t* kv, int32_t n_clusters,
                                    const float* centroids, const int32_t* assign, const tactic_params_t* params,
                                    void* stream, tactic_index_t* out) {
  if (!centroids || !assign) return fail(TACTIC_ERR_INVALID_ARGUMENT, "centroids / assign is NULL");
  return build_common(K, V, kv, n_clusters, 1, params, (cudaStream_t)stream, centroids, assign, out);
}

void tactic_index_destroy(tactic_index_t idx) {
  if (!idx) return;
  std::vector<void*> ptrs;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_allocs.find(idx);
    if (it != g_allocs.end()) {
      ptrs = it->second;
      g_allocs.erase(it);
    }
  }
  free_index(idx, &ptrs);
}

// ------------------------------------------------------------------------ recent-token tail
tactic_status_t tactic_set_tail_capacity(tactic_index_t idx, int32_t capacity) {
  if (!idx) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL index");
  if (capacity < 0) return fail(TACTIC_ERR_INVALID_ARGUMENT, "tail capacity %d < 0", capacity);
  if (idx->tail_len > 0) return fail(TACTIC_ERR_INVALID_ARGUMENT, "the tail holds %d tokens", idx->tail_len);
  if (capacity == idx->tail_cap) return TACTIC_OK;
  std::lock_guard<std::mutex> lk(g_mu);
  auto& ptrs = g_allocs[idx];
  for (void* p : {(void*)idx->Kt, (void*)idx->Vt}) {
    if (!p) continue;
    cudaFree(p);
    for (auto& q : ptrs)
      if (q == p) q = nullptr;
  }
  idx->Kt = idx->Vt = nullptr;
  idx->tail_cap = 0;
  if (capacity == 0) return TACTIC_OK;
  const size_t bytes = (size_t)idx->units * capacity * 128 * sizeof(__nv_bfloat16);
  if (cudaMalloc((void**)&idx->Kt, bytes) != cudaSuccess || cudaMalloc((void**)&idx->Vt, bytes) != cudaSuccess) {
    cudaGetLastError();
    if (idx->Kt) cudaFree(idx->Kt);
    idx->Kt = idx->Vt = nullptr;
    return fail(TACTIC_ERR_OOM, "tail buffers (%zu bytes)", 2 * bytes);
  }
  ptrs.push_back(idx->Kt);
  ptrs.push_back(idx->Vt);
  idx->tail_cap = capacity;
  return TACTIC_OK;
}

tactic_status_t tactic_append(tactic_index_t idx, const void* k_new, const void* v_new, int32_t t, void* stream) {
  if (!idx || !k_new || !v_new) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  if (t < 0) return fail(TACTIC_ERR_INVALID_ARGUMENT, "t = %d < 0", t);
  if (t == 0) return TACTIC_OK;
  if (idx->tail_cap == 0) {
    tactic_status_t st = tactic_set_tail_capacity(idx, TACTIC_TAIL_CAPACITY);
    if (st) return st;
  }
  if (idx->tail_len + t > idx->tail_cap)
    return fail(TACTIC_ERR_SHAPE, "tail full (%d + %d > capacity %d): re-cluster", idx->tail_len, t, idx->tail_cap);
  cudaStream_t s = (cudaStream_t)stream;
  CK(tactic::launch_tail_append((const __nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new, t, idx, s));
  idx->tail_len += t;
  // p >= 1 with the global split: every unit holds n + tail tokens
  CK(tactic::launch_unit_prefix_fill(idx->all_unit_prefix, idx->units, (long long)idx->n + idx->tail_len, s));
  return TACTIC_OK;
}

tactic_status_t tactic_index_tail(tactic_index_t idx, int32_t* len, int32_t* capacity) {
  if (!idx) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL index");
  if (len) *len = idx->tail_len;
  if (capacity) *capacity = idx->tail_cap;
  return TACTIC_OK;
}

tactic_status_t tactic_assign_tokens(tactic_index_t idx, const void* k, int32_t t, int32_t* assign, void* stream) {
  if (!idx || !k || !assign) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  if (t < 0) return fail(TACTIC_ERR_INVALID_ARGUMENT, "t = %d < 0", t);
  if (t == 0) return TACTIC_OK;
  CK(tactic::launch_assign((const __nv_bfloat16*)k, t, idx, assign, (cudaStream_t)stream));
  return TACTIC_OK;
}

tactic_status_t tactic_index_set_options(tactic_index_t idx, uint32_t options) {
  if (!idx) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL index");
  if (options & ~(uint32_t)(TACTIC_OPT_WINDOWS_EXACT | TACTIC_OPT_CLUSTER_DECODE | TACTIC_OPT_DETERMINISTIC))
    return fail(TACTIC_ERR_INVALID_ARGUMENT, "unknown option bits");
  tactic_status_t st = check_select_limits(idx, (options & TACTIC_OPT_WINDOWS_EXACT) != 0);
  if (st) return st;
  idx->options = options;
  return TACTIC_OK;
}

// ------------------------------------------------------------------------ Table-1 diagnostics
tactic_status_t tactic_exact_logits(const void* q, tactic_index_t idx, float* logits, void* stream) {
  if (!q || !idx || !logits) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  CK(tactic::launch_exact_logits((const __nv_bfloat16*)q, idx, logits, (cudaStream_t)stream));
  return TACTIC_OK;
}

tactic_status_t tactic_index_debug_timing(tactic_index_t idx, uint64_t* host, int32_t count) {
  if (!idx || !host) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!idx->tlog) return fail(TACTIC_ERR_UNSUPPORTED, "index created without TACTIC_TLOG=1");
  const size_t n = tlog_entries(idx->units);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(host, idx->tlog, (count < (int32_t)n ? (size_t)count : n) * 8, cudaMemcpyDeviceToHost));
  return TACTIC_OK;
}

static void sc_out(const SampleConsts& sc, tactic_sample_constants_t* out) {
  out->N = sc.N;
  out->x1 = sc.x1;
  out->x2 = sc.x2;
  out->w = sc.w;
  out->fallback = sc.fallback ? 1 : 0;
  out->slots = sc.slots;
}

tactic_status_t tactic_sample_constants(int32_t n, const tactic_params_t* params, tactic_sample_constants_t* out) {
  if (!out) return fail(TACTIC_ERR_INVALID_ARGUMENT, "out is NULL");
  SampleConsts sc;
  if (!sample_consts(n, params, &sc)) return fail(TACTIC_ERR_INVALID_ARGUMENT, "bad n or sampling fractions");
  sc_out(sc, out);
  return TACTIC_OK;
}

tactic_status_t tactic_index_sample_constants(tactic_index_t idx, tactic_sample_constants_t* out) {
  if (!idx || !out) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  sc_out(idx->sc, out);
  return TACTIC_OK;
}

tactic_status_t tactic_index_info(tactic_index_t idx, tactic_index_info_t* info) {
  if (!idx || !info) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  info->units = idx->units;
  info->batch = idx->B;
  info->num_kv_heads = idx->Hkv;
  info->group_size = idx->G;
  info->seq_len = idx->n;
  info->n_clusters = idx->C;
  info->iters_requested = idx->iters_req;
  info->device_bytes = idx->device_bytes;
  int fm = 0, fr = 0;
  info->select_cluster_size = fused_plan(idx, &fm, &fr) ? fr : 0;
  info->build_gpu_ms = -1.f;
  float ms = 0.f;
  if (idx->ev_build[0] && idx->ev_build[1] && cudaEventSynchronize(idx->ev_build[1]) == cudaSuccess &&
      cudaEventElapsedTime(&ms, idx->ev_build[0], idx->ev_build[1]) == cudaSuccess)
    info->build_gpu_ms = ms;
  cudaGetLastError();
  return TACTIC_OK;
}

tactic_status_t tactic_index_export(tactic_index_t idx, float* centroids, int32_t* assign, double* inertia,
                                    int32_t* iters_run, void* stream) {
  if (!idx) return fail(TACTIC_ERR_INVALID_ARGUMENT, "index is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t U = idx->units;
  if (centroids) CK(cudaMemcpyAsync(centroids, idx->cent, U * idx->C * 128 * 4, cudaMemcpyDeviceToHost, s));
  if (assign) CK(cudaMemcpyAsync(assign, idx->assign, U * idx->n * 4, cudaMemcpyDeviceToHost, s));
  if (iters_run) CK(cudaMemcpyAsync(iters_run, idx->iters_run, U * 4, cudaMemcpyDeviceToHost, s));
  if (inertia) {
    double* part = nullptr;
    CK(cudaMallocAsync((void**)&part, U * idx->C * sizeof(double), s));
    KmArgs a = {};
    a.n = idx->n;
    a.C = idx->C;
    a.units = idx->units;
    a.cent = idx->cent;
    a.offsets = idx->offsets;
    a.Kp = idx->Kp;
    CK(km_inertia(a, part, s));
    std::vector<double> h(U * idx->C);
    CK(cudaMemcpyAsync(h.data(), part, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(part, s));
    CK(cudaStreamSynchronize(s));
    for (size_t u = 0; u < U; ++u) {
      double t = 0.0;
      for (int j = 0; j < idx->C; ++j) t += h[u * idx->C + j];
      inertia[u] = t;
    }
  }
  CK(cudaStreamSynchronize(s));
  return TACTIC_OK;
}

// ------------------------------------------------------------------------ decode
// One-launch decode (decode_fused.cu, TACTIC_OPT_CLUSTER_DECODE): M clusters per CTA and
// R CTAs per unit cluster, or false when the index decodes through the multi-kernel chain.
// TACTIC_FUSED_M=128 prefers 128 clusters per CTA (measurement aid).
static bool fused_plan(tactic_index_t idx, int* M, int* R) {
  static const int env_m = [] { const char* e = getenv("TACTIC_FUSED_M"); return e ? atoi(e) : 0; }();
  if (!(idx->options & TACTIC_OPT_CLUSTER_DECODE) || (idx->options & TACTIC_OPT_WINDOWS_EXACT)) return false;
  const int G = idx->G, C = idx->C;
  if (!(G == 1 || G == 2 || G == 4 || G == 8) || C > 2048 || (long long)C * G > 4096 || idx->n >= (1 << 24))
    return false;
  static const bool verbose = [] { const char* e = getenv("TACTIC_VERBOSE"); return e && e[0] == '1'; }();
  if (idx->fz_checked_m == 0) {
    // first decode: the smallest M whose clusters all fit in one wave (every unit resident
    // at once), else the M that keeps the most SMs busy per wave
    idx->fz_checked_m = -1;
    long long best = 0;
    for (int m : {64, 128}) {
      if ((m == 64 && (C > 1024 || env_m == 128)) || C > 16 * m) continue;
      const int r = (C + m - 1) / m;
      // stage region (decode_fused.cu): R run blocks + R candidate blocks + >= 2 sample stages
      const size_t rblk = ((size_t)G * (m + 1) * 12 + 15) & ~(size_t)15;
      const size_t cblk = (16 + (size_t)m * (3 + G) * 4 + 15) & ~(size_t)15;
      if (r * (rblk + cblk) > 128 * 1024 || 128 * 1024 - r * cblk < 2 * 16384) continue;
      const int nc = fused_max_active_clusters(G, m, r);
      if (verbose) fprintf(stderr, "[tactic] one-launch decode G=%d M=%d R=%d: %d clusters resident\n", G, m, r, nc);
      if (nc >= idx->units) {
        idx->fz_checked_m = m;
        break;
      }
      if (nc >= 1 && (long long)nc * r > best) {
        best = (long long)nc * r;
        idx->fz_checked_m = m;
      }
    }
  }
  if (idx->fz_checked_m <= 0) return false;
  *M = idx->fz_checked_m;
  *R = (C + *M - 1) / *M;
  return true;
}

static tactic_status_t run_fused(const void* q, tactic_index_t idx, float p, int M, int R, cudaStream_t s,
                                 void* out, float* out_f32, float* lse) {
  FusedArgs a = {};
  a.q = (const __nv_bfloat16*)q;
  a.cent = idx->cent;
  a.offsets = idx->offsets;
  a.Kp = idx->Kp;
  a.Vp = idx->Vp;
  a.Kt = idx->Kt;
  a.Vt = idx->Vt;
  a.n = idx->n;
  a.C = idx->C;
  a.units = idx->units;
  a.tail_len = idx->tail_len;
  a.tail_cap = idx->tail_cap;
  a.sc = idx->sc;
  a.p = p;
  a.fixed_budget = idx->fixed_budget;
  a.crit = idx->crit;
  a.order = idx->order;
  a.ends = idx->ends;
  a.logits = idx->logits;
  a.fit = idx->fit;
  a.J = idx->J;
  a.umask = idx->umask;
  a.ulist = idx->union_list;
  a.uprefix = idx->union_prefix;
  a.unit_prefix = unit_split_ok(idx->units, idx->num_ctas) ? nullptr : idx->unit_prefix;
  a.unit_cnt = idx->counter;
  a.out = (__nv_bfloat16*)out;
  a.out_f32 = out_f32;
  a.lse = lse;
  a.tlog = idx->tlog;
  static const int dbg_stop = [] { const char* e = getenv("TACTIC_FUSED_STOP"); return e ? atoi(e) : 0; }();
  a.dbg_stop = dbg_stop;
  CK(launch_decode_fused(a, idx->G, M, R, s));
  idx->lists_valid = true;
  return TACTIC_OK;
}

// q_copy (nullable): q lives in mapped host memory; score_rank copies it there and the
// later kernels read the copy
static tactic_status_t run_selection(const void* q, tactic_index_t idx, double p, int mode, cudaStream_t s,
                                     const double* gmax, const double* gmass, double* local_max,
                                     __nv_bfloat16* q_copy = nullptr) {
  SelArgs sa = {};
  sa.q = q_copy ? q_copy : (const __nv_bfloat16*)q;
  sa.idx = idx;
  sa.p = p;
  sa.mode = mode;
  sa.gmax = gmax;
  sa.gmass = gmass;
  sa.local_max = local_max;
  // The entry kernel waits for everything before it on the stream to complete (no PDL):
  // a caller's preceding kernel produces q.  The later kernels overlap their prologues
  // with the previous kernel's tail through programmatic dependent launch.
  const bool pdl = true;
  CK(launch_score_rank((const __nv_bfloat16*)q, idx, s, false, q_copy));  // S1, S2, S3 (+ row map)
  CK(launch_sample(sa, s, pdl));                 // S4 (+ per-block fit summaries)
  // mode 0: Alg. 1 selection; mode 2: sharded stage 1 (the fit only, same kernel)
  CK(launch_fit(sa, s, pdl));                    // S5-S7
  if (mode == 0) idx->lists_valid = true;
  return TACTIC_OK;
}

static tactic_status_t run_attention(const void* q, tactic_index_t idx, bool all, cudaStream_t s, void* out,
                                     float* out_f32, float* lse, cudaEvent_t ev_mid = nullptr,
                                     bool entry = false) {
  AttnArgs aa = {};
  aa.q = (const __nv_bfloat16*)q;
  aa.Kp = idx->Kp;
  aa.Vp = idx->Vp;
  aa.seg_row = all ? idx->all_list : idx->union_list;
  aa.seg_prefix = all ? idx->all_prefix : idx->union_prefix;
  aa.unit_prefix = all ? idx->all_unit_prefix : idx->unit_prefix;
  aa.n = idx->n;
  aa.C = idx->C;
  aa.units = idx->units;
  aa.Hkv = idx->Hkv;
  aa.part_o = idx->part_o;
  aa.part_lse = idx->part_lse;
  aa.unit_cnt = idx->unit_cnt;
  aa.out = (__nv_bfloat16*)out;
  aa.out_f32 = out_f32;
  aa.lse = lse;
  aa.tlog = idx->tlog;
  aa.unit_split = unit_split_ok(idx->units, idx->num_ctas);  // else the global split (unit_prefix)
  aa.Kt = idx->Kt;
  aa.Vt = idx->Vt;
  aa.tail_len = idx->tail_len;
  aa.tail_cap = idx->tail_cap;
  if (!all && !(idx->options & TACTIC_OPT_DETERMINISTIC)) {  // the selection's fit wrote the per-head shift
    aa.mref = idx->mref;
    aa.acc = idx->acc;
    aa.acc_flag = idx->acc_flag;
    aa.dm_ok = idx->num_ctas <= idx->num_sms ? 1 : 0;
  }
  CK(launch_attention_sparse(aa, idx->G, idx->num_ctas, s, ev_mid == nullptr && !entry));  // S8 + fused S9
  if (ev_mid) CK(cudaEventRecord(ev_mid, s));
  return TACTIC_OK;
}

static tactic_status_t check_p(float p) {
  if (!(p > 0.0f) || p > 1.0f || std::isnan(p)) return fail(TACTIC_ERR_INVALID_ARGUMENT, "p must be in (0, 1] (got %g)", p);
  return TACTIC_OK;
}

tactic_status_t tactic_decode_ex(const void* q, tactic_index_t idx, float p, void* out, float* lse, void* stream) {
  if (!q || !idx || !out) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  tactic_status_t st = check_p(p);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (p >= 1.0f) return run_attention(q, idx, true, s, out, nullptr, lse, nullptr, true);  // reading 15
  int M = 0, R = 0;
  if (fused_plan(idx, &M, &R)) return run_fused(q, idx, p, M, R, s, out, nullptr, lse);
  if ((st = run_selection(q, idx, (double)p, 0, s, nullptr, nullptr, nullptr))) return st;
  return run_attention(q, idx, false, s, out, nullptr, lse);
}

tactic_status_t tactic_decode_attention_only(const void* q, tactic_index_t idx, void* out, void* stream) {
  if (!q || !idx || !out) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!idx->lists_valid)
    return fail(TACTIC_ERR_INVALID_ARGUMENT, "no selection has run on this index yet (call tactic_decode with p < 1)");
  return run_attention(q, idx, false, (cudaStream_t)stream, out, nullptr, nullptr, nullptr, true);
}

tactic_status_t tactic_decode_profiled(const void* q, tactic_index_t idx, float p, void* out,
                                       void* const* events, int32_t n_events, void* stream) {
  if (!q || !idx || !out || !events || n_events != 4) return fail(TACTIC_ERR_INVALID_ARGUMENT, "bad arguments");
  tactic_status_t st = check_p(p);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  CK(cudaEventRecord(ev[0], s));
  if (p < 1.0f && (st = run_selection(q, idx, (double)p, 0, s, nullptr, nullptr, nullptr))) return st;
  CK(cudaEventRecord(ev[1], s));
  if ((st = run_attention(q, idx, p >= 1.0f, s, out, nullptr, nullptr, ev[2]))) return st;
  CK(cudaEventRecord(ev[3], s));  // S9 is fused into the attention kernel: ev[3] == ev[2]
  return TACTIC_OK;
}

tactic_status_t tactic_decode(const void* q, tactic_index_t idx, float p, void* out, void* stream) {
  return tactic_decode_ex(q, idx, p, out, nullptr, stream);
}

// H2D q -> decode -> D2H out, enqueued on s (the body of the host-buffer call)
// device alias of a pinned, mapped host buffer (nullptr: pageable or not mapped)
static void* mapped_alias(const void* h) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

static tactic_status_t decode_host_body(const void* q_host, tactic_index_t idx, float p, void* out_host,
                                        cudaStream_t s) {
  const size_t bytes = (size_t)idx->units * idx->G * 128 * 2;
  // zero-copy: q is read over the bus by score_rank (which stages it for the later kernels)
  // and the attention's merge writes the output straight into the caller's pinned buffer;
  // the graph then holds only the decode kernels (no copy-engine round trips)
  int M = 0, R = 0;
  void* qd = mapped_alias(q_host);
  void* od = mapped_alias(out_host);
  if (qd && od && p < 1.0f && !fused_plan(idx, &M, &R) && !score_rank_prescored(idx) &&
      !getenv_flag("TACTIC_HOST_COPIES")) {
    tactic_status_t st = run_selection(qd, idx, (double)p, 0, s, nullptr, nullptr, nullptr, idx->q_stage);
    if (st) return st;
    return run_attention(idx->q_stage, idx, false, s, od, nullptr, nullptr);
  }
  CK(cudaMemcpyAsync(idx->q_stage, q_host, bytes, cudaMemcpyHostToDevice, s));
  tactic_status_t st = tactic_decode_ex(idx->q_stage, idx, p, idx->o_stage, nullptr, s);
  if (st) return st;
  CK(cudaMemcpyAsync(out_host, idx->o_stage, bytes, cudaMemcpyDeviceToHost, s));
  return TACTIC_OK;
}

tactic_status_t tactic_decode_host(const void* q_host, tactic_index_t idx, float p, void* out_host, void* stream) {
  if (!q_host || !idx || !out_host) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  tactic_status_t st = check_p(p);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const bool same = idx->hg_q == q_host && idx->hg_o == out_host && idx->hg_p == p && idx->hg_tail == idx->tail_len &&
                    idx->hg_opts == idx->options;
  if (!same) {  // (re)capture the whole call as one graph: one launch per call afterwards
    if (idx->hg_exec) cudaGraphExecDestroy(idx->hg_exec);
    idx->hg_exec = nullptr;
    idx->hg_q = q_host;
    idx->hg_o = out_host;
    idx->hg_p = p;
    idx->hg_tail = idx->tail_len;
    idx->hg_opts = idx->options;
    idx->hg_failed = false;
    if (!idx->hg_stream) CK(cudaStreamCreateWithFlags(&idx->hg_stream, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(idx->hg_stream, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      st = decode_host_body(q_host, idx, p, out_host, idx->hg_stream);
      e = cudaStreamEndCapture(idx->hg_stream, &g);
      if (st == TACTIC_OK && e == cudaSuccess && g) e = cudaGraphInstantiate(&idx->hg_exec, g, 0);
      if (g) cudaGraphDestroy(g);
    }
    if (st != TACTIC_OK || e != cudaSuccess || !idx->hg_exec) {  // e.g. pageable host buffers
      cudaGetLastError();
      idx->hg_exec = nullptr;
      idx->hg_failed = true;
    }
  }
  if (idx->hg_exec) {
    CK(cudaGraphLaunch(idx->hg_exec, s));
  } else if ((st = decode_host_body(q_host, idx, p, out_host, s))) {
    return st;
  }
  CK(cudaStreamSynchronize(s));
  return TACTIC_OK;
}

tactic_status_t tactic_decode_debug(const void* q, tactic_index_t idx, float p, void* out, float* lse,
                                    int32_t* order, int32_t* J, double* fit, uint8_t* union_mask, void* stream) {
  if (!q || !idx || !out) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  tactic_status_t st = check_p(p);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  int M = 0, R = 0;
  if (p < 1.0f && fused_plan(idx, &M, &R)) {
    if ((st = run_fused(q, idx, p, M, R, s, out, nullptr, lse))) return st;
  } else {
    if ((st = run_selection(q, idx, (double)p, 0, s, nullptr, nullptr, nullptr))) return st;
    if ((st = run_attention(q, idx, false, s, out, nullptr, lse))) return st;
  }
  const size_t U = idx->units, G = idx->G, C = idx->C;
  if (order) CK(cudaMemcpyAsync(order, idx->order, U * G * C * 4, cudaMemcpyDeviceToHost, s));
  if (J) CK(cudaMemcpyAsync(J, idx->J, U * G * 4, cudaMemcpyDeviceToHost, s));
  if (fit) CK(cudaMemcpyAsync(fit, idx->fit, U * G * 6 * 8, cudaMemcpyDeviceToHost, s));
  if (union_mask) CK(cudaMemcpyAsync(union_mask, idx->umask, U * C, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return TACTIC_OK;
}

// ------------------------------------------------------------------------ per-head loading ablation
static tactic_status_t per_head_attention(const void* q, tactic_index_t idx, void* out, cudaStream_t s) {
  const int VU = idx->units * idx->G;
  CK(tactic::launch_head_lists(idx, s));
  AttnArgs aa = {};
  aa.q = (const __nv_bfloat16*)q;
  aa.Kp = idx->Kp;
  aa.Vp = idx->Vp;
  aa.seg_row = idx->head_list;
  aa.seg_prefix = idx->head_prefix;
  aa.unit_prefix = nullptr;
  aa.n = idx->n;
  aa.C = idx->C;
  aa.units = VU;
  aa.Hkv = idx->Hkv;
  aa.part_o = idx->part_o;
  aa.part_lse = idx->part_lse;
  aa.unit_cnt = idx->head_cnt2;
  aa.out = (__nv_bfloat16*)out;
  aa.unit_split = 1;
  aa.Kt = idx->Kt;
  aa.Vt = idx->Vt;
  aa.tail_len = idx->tail_len;
  aa.tail_cap = idx->tail_cap;
  aa.kv_div = idx->G;
  CK(launch_attention_sparse(aa, 1, idx->num_ctas, s, true));
  return TACTIC_OK;
}

static tactic_status_t per_head_checks(tactic_index_t idx) {
  const int VU = idx->units * idx->G;  // (unit, head) pairs
  if (!unit_split_ok(VU, idx->num_ctas))
    return fail(TACTIC_ERR_UNSUPPORTED, "per-head attention needs units x G (%d) <= CTAs / 2", VU);
  return TACTIC_OK;
}

tactic_status_t tactic_decode_per_head(const void* q, tactic_index_t idx, float p, void* out, void* stream) {
  if (!q || !idx || !out) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  tactic_status_t st = check_p(p);
  if (st) return st;
  if (p >= 1.0f) return fail(TACTIC_ERR_UNSUPPORTED, "per-head ablation is for p < 1");
  if ((st = per_head_checks(idx))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = run_selection(q, idx, (double)p, 0, s, nullptr, nullptr, nullptr))) return st;
  return per_head_attention(q, idx, out, s);
}

tactic_status_t tactic_decode_fixed_budget(const void* q, tactic_index_t idx, int32_t budget, int32_t per_head,
                                           void* out, int32_t* J, void* stream) {
  if (!q || !idx || !out) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  if (budget < 1 || budget > idx->n) return fail(TACTIC_ERR_INVALID_ARGUMENT, "budget %d not in [1, n]", budget);
  tactic_status_t st;
  if (per_head && (st = per_head_checks(idx))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  int M = 0, R = 0;
  idx->fixed_budget = budget;  // read by the fit kernel's / cluster decode's launcher only
  const bool fused = !per_head && fused_plan(idx, &M, &R);
  st = fused ? run_fused(q, idx, 0.5f, M, R, s, out, nullptr, nullptr)
             : run_selection(q, idx, 0.5, 0, s, nullptr, nullptr, nullptr);
  idx->fixed_budget = 0;
  if (st) return st;
  if (fused) {
  } else if (per_head) {
    if ((st = per_head_attention(q, idx, out, s))) return st;
  } else if ((st = run_attention(q, idx, false, s, out, nullptr, nullptr))) {
    return st;
  }
  if (J) {
    CK(cudaMemcpyAsync(J, idx->J, (size_t)idx->units * idx->G * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return TACTIC_OK;
}

// ------------------------------------------------------------------------ dense baseline
tactic_status_t tactic_dense_workspace_size(const tactic_kv_desc_t* kv, int32_t num_ctas, size_t* bytes) {
  Resolved r;
  tactic_status_t st = resolve_kv(kv, &r);
  if (st) return st;
  if (!bytes) return fail(TACTIC_ERR_INVALID_ARGUMENT, "bytes is NULL");
  const int P = num_ctas > 0 ? num_ctas : device_sms();
  const size_t slots = (size_t)P + (size_t)r.B * r.Hkv;
  *bytes = slots * r.G * 129 * 4 + (size_t)r.B * r.Hkv * 4 + 256;  // partials + arrival counters
  return TACTIC_OK;
}

tactic_status_t tactic_dense_decode(const void* q, const void* K, const void* V, const tactic_kv_desc_t* kv,
                                    void* out, float* lse, void* workspace, size_t workspace_bytes,
                                    int32_t num_ctas, void* stream) {
  if (!q || !K || !V || !out || !workspace) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  Resolved r;
  tactic_status_t st = resolve_kv(kv, &r);
  if (st) return st;
  if ((st = check_device())) return st;
  const int P = num_ctas > 0 ? num_ctas : device_sms();
  size_t need = 0;
  tactic_dense_workspace_size(kv, P, &need);
  if (workspace_bytes < need) return fail(TACTIC_ERR_INVALID_ARGUMENT, "workspace too small (%zu < %zu)", workspace_bytes, need);
  if ((uintptr_t)K % 16 || (uintptr_t)V % 16) return fail(TACTIC_ERR_SHAPE, "K and V must be 16-byte aligned");
  CUtensorMap mk, mv;
  if ((st = make_kv_map(&mk, K, r, 64))) return st;
  if ((st = make_kv_map(&mv, V, r, 64))) return st;
  const size_t units = (size_t)r.B * r.Hkv;
  const size_t slots = (size_t)P + units;
  float* part_o = (float*)workspace;
  float* part_lse = part_o + slots * r.G * 128;
  int* unit_cnt = (int*)(part_lse + slots * r.G);
  AttnArgs aa = {};
  aa.q = (const __nv_bfloat16*)q;
  aa.n = r.n;
  aa.units = (int)units;
  aa.Hkv = r.Hkv;
  aa.part_o = part_o;
  aa.part_lse = part_lse;
  cudaStream_t s = (cudaStream_t)stream;
  aa.unit_cnt = unit_cnt;
  aa.out = (__nv_bfloat16*)out;
  aa.lse = lse;
  aa.unit_split = unit_split_ok((int)units, P);
  CK(launch_attention_dense(aa, &mk, &mv, r.G, P, s, false));  // S10 + fused merge (entry: no PDL)
  return TACTIC_OK;
}

tactic_status_t tactic_lse_merge(const float* o_parts, const float* lse_parts, int32_t n_parts, int32_t n_rows,
                                 void* out, float* lse, void* stream) {
  if (!o_parts || !lse_parts || !out) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  if (n_parts < 1 || n_rows < 1) return fail(TACTIC_ERR_INVALID_ARGUMENT, "n_parts and n_rows must be >= 1");
  CK(launch_lse_merge_plain(o_parts, lse_parts, n_parts, n_rows, (__nv_bfloat16*)out, lse, (cudaStream_t)stream));
  return TACTIC_OK;
}

// ------------------------------------------------------------------------ sharded mode
tactic_status_t tactic_decode_stage1(const void* q, tactic_index_t idx, double* local_max, void* stream) {
  if (!q || !idx || !local_max) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  return run_selection(q, idx, 0.5, 2, (cudaStream_t)stream, nullptr, nullptr, local_max);
}

tactic_status_t tactic_decode_stage1b(tactic_index_t idx, const double* global_max, double* mass, void* stream) {
  if (!idx || !global_max || !mass) return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  if (stage1b_smem_bytes(idx) > smem_optin_limit())
    return fail(TACTIC_ERR_UNSUPPORTED, "sharded stage 1b: exact head of %d ranks exceeds shared memory",
                idx->sc.fallback ? idx->n : idx->sc.N);
  SelArgs sa = {};
  sa.idx = idx;
  sa.gmax = global_max;
  sa.mass_out = mass;
  CK(launch_stage1b(sa, (cudaStream_t)stream));
  return TACTIC_OK;
}

tactic_status_t tactic_decode_stage2(const void* q, tactic_index_t idx, float p, const double* global_max,
                                     const double* global_mass, float* o_part, float* lse_part, void* stream) {
  if (!q || !idx || !global_max || !global_mass || !o_part || !lse_part)
    return fail(TACTIC_ERR_INVALID_ARGUMENT, "NULL argument");
  tactic_status_t st = check_p(p);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  SelArgs sa = {};
  sa.q = (const __nv_bfloat16*)q;
  sa.idx = idx;
  sa.p = p;
  sa.mode = 1;
  sa.gmax = global_max;
  sa.gmass = global_mass;
  // stage 2 reuses stage 1's criticalities and order (the same q on the same index)
  CK(launch_fit(sa, s, false));                  // theta* rule + union (fit kernel, mode 1)
  idx->lists_valid = true;
  return run_attention(q, idx, false, s, nullptr, o_part, lse_part);
}

// ------------------------------------------------------------------------ misc
const char* tactic_status_string(tactic_status_t s) {
  switch (s) {
    case TACTIC_OK: return "TACTIC_OK";
    case TACTIC_ERR_INVALID_ARGUMENT: return "TACTIC_ERR_INVALID_ARGUMENT";
    case TACTIC_ERR_SHAPE: return "TACTIC_ERR_SHAPE";
    case TACTIC_ERR_OOM: return "TACTIC_ERR_OOM";
    case TACTIC_ERR_CUDA: return "TACTIC_ERR_CUDA";
    case TACTIC_ERR_NOT_FINITE: return "TACTIC_ERR_NOT_FINITE";
    case TACTIC_ERR_UNSUPPORTED: return "TACTIC_ERR_UNSUPPORTED";
  }
  return "TACTIC_ERR_UNKNOWN";
}

const char* tactic_last_error(void) { return g_err.c_str(); }

const char* tactic_version(void) { return "tactic-b200 0.1.0 (sm_100a)"; }

tactic_status_t tactic_device_check(int32_t* num_sms) {
  tactic_status_t st = check_device();
  if (st) return st;
  if (num_sms) *num_sms = device_sms();
  return TACTIC_OK;
}

}  // extern "C"
