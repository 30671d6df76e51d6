// diag.cu -- exact per-token logits for the Table-1 diagnostics.
//
// P:418-450 (§5.3, Table 1) compares token budgets -- Optimal (descending true score),
// Cluster-Optimal (clusters in criticality order, true scores) and Tactic -- and the
// achieved cumulative attention score.  All of them need the exact score of every
// token: l_{g,i} = q_g . k_i / sqrt(d) for every query head g of the unit, written here
// in the index's LAYOUT order (clusters contiguous, so a cluster's mass is a segment sum).
// Measurement tooling, not the decode path: one CTA per 128 layout rows of one unit, the
// rows bulk-copied into shared memory, the G <= 8 heads as the n = 8 columns of
// mma.sync m16n8k16 (bf16 products, fp32 accumulation).
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace tactic {

constexpr int XL_ROWS = 128;

__global__ void __launch_bounds__(XL_ROWS) exact_logits_kernel(const __nv_bfloat16* __restrict__ q,
                                                               const __nv_bfloat16* __restrict__ Kp, int n, int G,
                                                               float* __restrict__ logits) {
  __shared__ __align__(128) uint8_t rows_s[XL_ROWS * 256];
  __shared__ uint64_t bar;
  const int u = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r0 = blockIdx.x * XL_ROWS;
  const int nr = n - r0 < XL_ROWS ? n - r0 : XL_ROWS;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar, (uint32_t)nr * 256u);
    bulk_g2s(rows_s, Kp + ((size_t)u * n + r0) * 128, (uint32_t)nr * 256u, &bar);
  }
  // B fragment: n = head column (lane / 4 < G), k = dim
  uint32_t qb[8][2];
  {
    const int hcol = lane >> 2;
    const uint32_t* q32 = reinterpret_cast<const uint32_t*>(q + ((size_t)u * G + (hcol < G ? hcol : 0)) * 128);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qb[ks][0] = hcol < G ? q32[(ks * 16 + 2 * (lane & 3)) >> 1] : 0u;
      qb[ks][1] = hcol < G ? q32[(ks * 16 + 8 + 2 * (lane & 3)) >> 1] : 0u;
    }
  }
  mbar_wait(&bar, 0);
  const uint32_t sbase = smem_u32(rows_s);
#pragma unroll
  for (int gi = 0; gi < 2; ++gi) {
    const int i = (lane & 7) + ((lane >> 3) & 1) * 8;
    int li = warp * 32 + gi * 16 + i;
    const int grow = r0 + li;  // layout row: its chunk swizzle phase
    if (li >= nr) li = 0;      // past the unit's last row: any staged row, not stored
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t af[4];
      ldsm_x4(af[0], af[1], af[2], af[3], sbase + li * 256 + (swz_chunk(2 * ks + (lane >> 4), grow) << 4));
      mma_bf16_16816(s, af, qb[ks][0], qb[ks][1]);
    }
    // s[0], s[1]: row lane/4, heads 2(lane%4), +1; s[2], s[3]: row lane/4 + 8
    const int h0 = 2 * (lane & 3);
    const int ra = r0 + warp * 32 + gi * 16 + (lane >> 2), rb = ra + 8;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int h = h0 + (e & 1), r = e < 2 ? ra : rb;
      if (h < G && r < n) logits[((size_t)u * G + h) * n + r] = s[e] * 0.08838834764831845f;
    }
  }
}

cudaError_t launch_exact_logits(const __nv_bfloat16* q, const tactic_index_s* x, float* logits, cudaStream_t s) {
  dim3 grid((x->n + XL_ROWS - 1) / XL_ROWS, x->units);
  exact_logits_kernel<<<grid, XL_ROWS, 0, s>>>(q, (const __nv_bfloat16*)x->Kp, x->n, x->G, logits);
  return cudaGetLastError();
}

}  // namespace tactic
