// gemv_bulk.cuh (tuning harness only; measured slower than gemv_tree_kernel,
// see scripts/tune_gemv.py) — tree-order GEMV with the A stream on the bulk-copy (TMA)
// engine.  Same partials and pairwise tree as gemv_tree_kernel (reduce.cu:
// 128 partials per row, partial u folds t = u, u+128, ... ascending from
// exact zero), so the results are bit-identical; only the data movement and
// the work placement change:
//
//  * one persistent CTA per SM; G row groups of 4 warps (128 partials);
//  * x is staged into shared memory once per CTA (one bulk copy per plane);
//  * each group streams its rows' A planes through its own S-stage ring of
//    CH-column chunks with cp.async.bulk + an mbarrier per stage (complete_tx),
//    issued S-1 chunks ahead across row boundaries, so HBM requests stay in
//    flight while the FP64 pipe folds the current chunk and no registers hold
//    prefetched words;
//  * a group's 4 warps hand a consumed stage back with one named barrier per
//    chunk; the 128-partial tree runs level by level in shared memory under
//    the group's named barrier while the other groups keep folding.
//
// Requirements (checked by the host, else the register-prefetch kernel is
// used): n even, lda and sA even, A and x 16-byte aligned, x stride even,
// and the shared-memory footprint below <= the opt-in maximum.
#pragma once
#include "../common.cuh"

namespace mw {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Global -> shared bulk copy completing on bar (bytes multiple of 16, both
// addresses 16-byte aligned).  evict_first: A is streamed exactly once.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

// Shared-memory bytes of one CTA.
template <int K, int G, int CH, int S>
__host__ __device__ constexpr size_t gemv_bulk_smem(int64_t n) {
  return 256                                          // mbarriers (G*S + 1, <= 32)
         + (size_t)K * n * sizeof(double)             // x
         + (size_t)G * S * K * CH * sizeof(double)    // A rings
         + (size_t)G * K * 128 * sizeof(double);      // partial trees
}

template <int K, int VAR, int G, int CH, int S>
__global__ void __launch_bounds__(128 * G, 1)
    gemv_bulk_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                     const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                     int64_t m, int64_t n) {
  static_assert(CH % 128 == 0 && G * S + 1 <= 32 && G <= 15, "gemv_bulk shape");
  constexpr int P = 128;
  constexpr int J = CH / P;  // fold steps per chunk
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);  // [G][S] full, then x
  double* xs = reinterpret_cast<double*>(smem_raw + 256);  // [K][n]
  double* ring = xs + (size_t)K * n;                        // [G][S][K][CH]
  double* part = ring + (size_t)G * S * K * CH;             // [G][K][P]

  const int g = threadIdx.x / P;
  const int u = threadIdx.x % P;
  uint64_t* xbar = bars + G * S;
  if (threadIdx.x == 0) {
    for (int i = 0; i <= G * S; ++i) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t keep = policy_evict_last();
    mbar_expect_tx(xbar, (unsigned)(K * n * sizeof(double)));
#pragma unroll
    for (int c = 0; c < K; ++c)
      bulk_g2s(xs + (size_t)c * n, x + c * sx, (unsigned)(n * sizeof(double)), xbar, keep);
  }

  // This group's rows: gg, gg + stride, ...
  const int64_t gg = (int64_t)blockIdx.x * G + g;
  const int64_t stride = (int64_t)gridDim.x * G;
  const int64_t nrows = gg < m ? (m - 1 - gg) / stride + 1 : 0;
  const int64_t nc = (n + CH - 1) / CH;
  const int64_t Q = nrows * nc;
  uint64_t* full = bars + g * S;
  double* myring = ring + (size_t)g * S * K * CH;
  const uint64_t stream_once = policy_evict_first();

  auto issue = [&](int64_t q) {
    if (q >= Q) return;
    const int s = (int)(q % S);
    const int64_t row = gg + (q / nc) * stride;
    const int64_t col0 = (q % nc) * CH;
    const int64_t len = n - col0 < CH ? n - col0 : CH;
    const unsigned bytes = (unsigned)(len * sizeof(double));
    mbar_expect_tx(full + s, bytes * K);
#pragma unroll
    for (int c = 0; c < K; ++c)
      bulk_g2s(myring + ((size_t)s * K + c) * CH, A + c * sA + row * lda + col0, bytes, full + s,
               stream_once);
  };
  if (u == 0) {
#pragma unroll
    for (int q = 0; q < S - 1; ++q) issue(q);
  }
  mbar_wait(xbar, 0);

  const int64_t valid = n < P ? n : P;
  double* mypart = part + (size_t)g * K * P;
  V<K> acc = zero<K>();
  for (int64_t q = 0; q < Q; ++q) {
    // stage (q-1) % S is free once the whole group has folded chunk q-1
    if (q > 0) named_sync(1 + g, P);
    if (u == 0) issue(q + S - 1);
    const int s = (int)(q % S);
    mbar_wait(full + s, (unsigned)((q / S) & 1));
    const int64_t ci = q % nc;
    const int64_t col0 = ci * CH;
    const double* st = myring + (size_t)s * K * CH;
    if (col0 + CH <= n) {
      V<K> a[J], xv[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
          a[j].c[c] = st[c * CH + u + j * P];
          xv[j].c[c] = xs[c * n + col0 + u + j * P];
        }
      }
#pragma unroll
      for (int j = 0; j < J; ++j) acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a[j], xv[j]));
    } else {
      for (int j = 0; j < J; ++j) {
        const int64_t t = col0 + u + j * P;
        if (t < n) {
          V<K> a, xv;
#pragma unroll
          for (int c = 0; c < K; ++c) {
            a.c[c] = st[c * CH + u + j * P];
            xv.c[c] = xs[c * n + t];
          }
          acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a, xv));
        }
      }
    }
    if (ci == nc - 1) {
      // row done: the pairwise tree over the group's 128 partials
#pragma unroll
      for (int c = 0; c < K; ++c) mypart[c * P + u] = acc.c[c];
      named_sync(1 + g, P);
#pragma unroll 1
      for (int sd = 1; sd < P; sd <<= 1) {
        const int idx = 2 * sd * u;
        if (idx + sd < valid) {
          V<K> l, r;
#pragma unroll
          for (int c = 0; c < K; ++c) {
            l.c[c] = mypart[c * P + idx];
            r.c[c] = mypart[c * P + idx + sd];
          }
          const V<K> sum = Ops<K, VAR>::add(l, r);
#pragma unroll
          for (int c = 0; c < K; ++c) mypart[c * P + idx] = sum.c[c];
        }
        named_sync(1 + g, P);
      }
      if (u == 0) {
        V<K> r0;
#pragma unroll
        for (int c = 0; c < K; ++c) r0.c[c] = mypart[c * P];
        store<K>(y, sy, gg + (q / nc) * stride, r0);
      }
      acc = zero<K>();
    }
  }
}

}  // namespace mw
