// gemv_wring.cuh -- tuning harness: tree-order GEMV (same partials and tree
// as gemv_tree_kernel, so bit-identical) with a PER-WARP bulk-copy ring.
// A persistent CTA holds Q row quads (4 warps each: warp q of a quad folds
// partials 32q..32q+31 of the quad's current row).  Each warp streams its
// own 256-byte A segments (one per plane and fold step) through an S-stage
// shared-memory ring with cp.async.bulk + one mbarrier per stage, refilled
// by lane 0 right after the warp consumed a stage: no cross-warp barrier
// until the row's tree.  x is read through L1.  Requires n % 128 == 0,
// even lda / sA, 16-byte aligned A.
#pragma once
#include "gemv_bulk.cuh"

namespace mw {

template <int K, int Q, int J, int S>
__host__ __device__ constexpr size_t gemv_wring_smem() {
  return 2048 /* barriers: 4Q*S*8 <= 2048 */ + (size_t)4 * Q * S * K * J * 32 * sizeof(double) +
         (size_t)Q * K * 128 * sizeof(double);
}

template <int K, int VAR, int Q, int J, int S>
__global__ void __launch_bounds__(128 * Q, 1)
    gemv_wring_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                      const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                      int64_t m, int64_t n) {
  static_assert(4 * Q * S * 8 <= 2048, "barrier area");
  constexpr int P = 128;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);              // [4Q][S]
  double* ring = reinterpret_cast<double*>(smem_raw + 2048);           // [4Q][S][K][J][32]
  double* part = ring + (size_t)4 * Q * S * K * J * 32;                 // [Q][K][128]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int quad = warp >> 2, q = warp & 3;
  const int u = 32 * q + lane;
  uint64_t* full = bars + warp * S;
  double* myring = ring + (size_t)warp * S * K * J * 32;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();

  const int64_t gq = (int64_t)blockIdx.x * Q + quad;
  const int64_t stride = (int64_t)gridDim.x * Q;
  const int64_t nrows = gq < m ? (m - 1 - gq) / stride + 1 : 0;
  const int64_t ng = n / (P * J);  // fold groups per row (n % (128 J) == 0 asserted by the host)
  const int64_t total = nrows * ng;
  const uint64_t stream_once = policy_evict_first();

  auto issue = [&](int64_t idx) {
    if (idx >= total) return;
    const int s = (int)(idx % S);
    const int64_t row = gq + (idx / ng) * stride;
    const int64_t g = idx % ng;
    mbar_expect_tx(full + s, (unsigned)(K * J * 32 * sizeof(double)));
#pragma unroll
    for (int c = 0; c < K; ++c)
#pragma unroll
      for (int j = 0; j < J; ++j)
        bulk_g2s(myring + (((size_t)s * K + c) * J + j) * 32,
                 A + c * sA + row * lda + 32 * q + P * (g * J + j), 32 * sizeof(double), full + s,
                 stream_once);
  };
  if (lane == 0)
    for (int s = 0; s < S; ++s) issue(s);

  V<K> acc = zero<K>();
  double* mypart = part + (size_t)quad * K * P;
  for (int64_t idx = 0; idx < total; ++idx) {
    const int s = (int)(idx % S);
    const int64_t g = idx % ng;
    mbar_wait(full + s, (unsigned)((idx / S) & 1));
    const double* st = myring + (size_t)s * K * J * 32;
    V<K> a[J], xv[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
#pragma unroll
      for (int c = 0; c < K; ++c) a[j].c[c] = st[(c * J + j) * 32 + lane];
      xv[j] = load<K>(x, sx, u + P * (g * J + j));
    }
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(idx + S);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a[j], xv[j]));
    if (g == ng - 1) {
      const int64_t row = gq + (idx / ng) * stride;
#pragma unroll
      for (int c = 0; c < K; ++c) mypart[c * P + u] = acc.c[c];
      named_sync(1 + quad, P);
#pragma unroll 1
      for (int sd = 1; sd < P; sd <<= 1) {
        const int i0 = 2 * sd * u;
        if (i0 + sd < P) {
          V<K> l, r;
#pragma unroll
          for (int c = 0; c < K; ++c) {
            l.c[c] = mypart[c * P + i0];
            r.c[c] = mypart[c * P + i0 + sd];
          }
          const V<K> sum = Ops<K, VAR>::add(l, r);
#pragma unroll
          for (int c = 0; c < K; ++c) mypart[c * P + i0] = sum.c[c];
        }
        named_sync(1 + quad, P);
      }
      if (u == 0) {
        V<K> r0;
#pragma unroll
        for (int c = 0; c < K; ++c) r0.c[c] = mypart[c * P];
        store<K>(y, sy, row, r0);
      }
      acc = zero<K>();
    }
  }
}

}  // namespace mw
