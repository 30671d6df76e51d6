// fitmath.cuh -- device arithmetic shared by the selection kernels (select.cu,
// rank_cluster.cu, decode_fused.cu): the ranking key of S2 and the float32 tail sum of
// the two-point fit y = a/x + b (App. B Alg. 1 l.4-10; DESIGN.md
// readings 11, 12, 18, 24).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace tactic {

// S2 key: order-preserving bits of -crit with the low 12 bits replaced by the cluster
// id, so one 64-bit compare orders by (-crit, id) (reading 24: criticalities
// that agree in their leading 40 mantissa bits rank by cluster id; ids < 4096).
__device__ __forceinline__ unsigned long long crit_key(double crit, int id) {
  if (crit == 0.0) crit = 0.0;  // -0 == +0
  const unsigned long long b = (unsigned long long)__double_as_longlong(-crit);
  const unsigned long long k = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending = descending crit
  return (k & ~0xFFFull) | (unsigned long long)id;
}

// H(k) - H(j) = sum_{i=j+1}^{k} 1/i for 0 <= j <= k: exact terms below 16, above that
// log1p of the ratio plus the difference of the asymptotic series 1/2x - 1/12x^2 + 1/120x^4
// (the next term is < 2.4e-10 at x = 16).
// (Reciprocals by __frcp_rn, correctly rounded like 1.f / x, without the IEEE division
// sequence: the J search evaluates this on the warp's critical path.)
__device__ __forceinline__ float harm_diff_f(int k, int j) {
  if (k <= j) return 0.f;
  float s = 0.f;
  while (j < 16 && j < k) s += __frcp_rn((float)(++j));  // tiny n only
  if (k <= j) return s;
  const float xk = (float)k, xj = (float)j;
  const float rk = __frcp_rn(xk), rj = __frcp_rn(xj);
  auto t = [](float r) {
    const float r2 = r * r;
    return r * 0.5f - r2 * (1.f / 12.f - r2 * (1.f / 120.f));
  };
  return s + log1pf((xk - xj) * rj) + (t(rk) - t(rj));
}

// sum_{i=N+1}^{k} max(0, a/i + b): the positive terms of the monotone a/i + b form one
// rank interval [lo, hi] inside (N, n] (a/i + b > 0  <=>  a + b i > 0 for i > 0), found
// once per head; each evaluation then costs one log1pf.
struct TailF {
  float a, b;
  int lo, hi;  // empty when lo > hi
  __device__ __forceinline__ float operator()(int k) const {
    const int kk = k < hi ? k : hi;
    if (kk < lo) return 0.f;
    return a * harm_diff_f(kk, lo - 1) + b * (float)(kk - lo + 1);
  }
};
__device__ __forceinline__ TailF make_tail_f(float a, float b, int N, int n) {
  TailF f = {a, b, N + 1, n};
  auto pos = [&](int i) { return fmaf(b, (float)i, a) > 0.f; };
  if (a >= 0.f && b >= 0.f) return f;
  if (a <= 0.f && b <= 0.f) { f.lo = n + 1; return f; }
  if (a > 0.f) {  // decreasing: positive for i < a / (-b)
    const float t = a / (-b);
    int top = t >= (float)n ? n : (int)floorf(t);
    while (top < n && pos(top + 1)) ++top;
    while (top > N && !pos(top)) --top;
    f.hi = top;  // top <= N: empty
    return f;
  }
  const float t = (-a) / b;  // increasing: positive for i > (-a) / b
  int lo = t >= (float)n ? n + 1 : (int)floorf(t) + 1;
  if (lo < N + 1) lo = N + 1;
  while (lo > N + 1 && pos(lo - 1)) --lo;
  while (lo <= n && !pos(lo)) ++lo;
  f.lo = lo;
  return f;
}

}  // namespace tactic
