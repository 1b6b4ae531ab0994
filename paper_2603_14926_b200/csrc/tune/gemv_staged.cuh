// gemv_staged.cuh -- explored GEMV variant (tuning harness only, not in
// the product): the tree kernel's partials with the A stream through a
// per-thread cp.async ring.  Measured bit-identical and no faster than
// gemv_tree_kernel at config 2 (scripts/tune_gemv.py).
#pragma once
namespace mw {

// Same partials, same order as gemv_tree_kernel (WARPS = 4, P = 128), but
// the A stream goes through a per-thread cp.async ring in shared memory:
// chunk ch + S - 1 (D elements x K planes) is in flight while chunk ch is
// folded, so each thread waits for HBM once per row instead of once per
// chunk, without holding the prefetched words in registers.  Each thread
// reads back only what it copied (cp.async.wait_group, no CTA barrier in
// the main loop).  XS: x goes through the ring too.
template <int K, int VAR, int RPC, int D, int S, bool XS>
__global__ void __launch_bounds__(128 * RPC)
    gemv_staged_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                       const double* __restrict__ x, int64_t sx, double* __restrict__ y,
                       int64_t sy, int64_t m, int64_t n) {
  constexpr int P = 128;
  constexpr int NT = P * RPC;
  constexpr int NB = XS ? 2 : 1;  // A (and x) rings
  extern __shared__ double stage[];  // [NB][S][K][D][NT]
  const int tid = threadIdx.x;
  const int slot = tid / P;
  const int u = tid % P;
  const int64_t i = blockIdx.x * (int64_t)RPC + slot;
  const bool live = i < m;
  const double* row = A + (live ? i : 0) * lda;
  const int64_t cnt = n > u ? (n - u + P - 1) / P : 0;  // elements of this partial
  const int64_t nch = cnt / D;
  auto at = [&](int b, int s, int c, int d) -> double* {
    return stage + ((((int64_t)b * S + s) * K + c) * D + d) * NT + tid;
  };
  auto issue = [&](int64_t ch) {
    const int s = (int)(ch % S);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t t = u + (ch * D + d) * P;
#pragma unroll
      for (int c = 0; c < K; ++c) {
        cp_async8(at(0, s, c, d), row + c * sA + t, 8);
        if constexpr (XS) cp_async8(at(1, s, c, d), x + c * sx + t, 8);
      }
    }
  };
#pragma unroll
  for (int p = 0; p < S - 1; ++p) {
    if (p < nch) issue(p);
    cp_async_commit();
  }
  V<K> acc = zero<K>();
  for (int64_t ch = 0; ch < nch; ++ch) {
    if (ch + S - 1 < nch) issue(ch + S - 1);
    cp_async_commit();
    cp_async_wait<S - 1>();
    const int s = (int)(ch % S);
    V<K> a[D], xv[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
#pragma unroll
      for (int c = 0; c < K; ++c) a[d].c[c] = *at(0, s, c, d);
      if constexpr (XS) {
#pragma unroll
        for (int c = 0; c < K; ++c) xv[d].c[c] = *at(1, s, c, d);
      } else {
        xv[d] = load<K>(x, sx, u + (ch * D + d) * P);
      }
    }
#pragma unroll
    for (int d = 0; d < D; ++d) acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a[d], xv[d]));
  }
  for (int64_t t = u + nch * D * P; t < n; t += P)
    acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(row, sA, t), load<K>(x, sx, t)));
  const int64_t valid = n < P ? n : P;
  __syncthreads();  // the ring is reused below as the tree buffer
  double* part = stage;  // [RPC][K][P]
#pragma unroll
  for (int c = 0; c < K; ++c) part[(slot * K + c) * P + u] = acc.c[c];
  __syncthreads();
#pragma unroll 1
  for (int s = 1; s < P; s <<= 1) {
    const int per_row = P / (2 * s);
    if (tid < RPC * per_row) {
      const int r = tid / per_row, idx = 2 * s * (tid % per_row);
      if (idx + s < valid) {
        V<K> a, b;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          a.c[c] = part[(r * K + c) * P + idx];
          b.c[c] = part[(r * K + c) * P + idx + s];
        }
        const V<K> sum = Ops<K, VAR>::add(a, b);
#pragma unroll
        for (int c = 0; c < K; ++c) part[(r * K + c) * P + idx] = sum.c[c];
      }
    }
    __syncthreads();
  }
  if (u == 0 && live) {
    V<K> r0;
#pragma unroll
    for (int c = 0; c < K; ++c) r0.c[c] = part[(slot * K + c) * P];
    store<K>(y, sy, i, r0);
  }
}

template <int K, int RPC, int D, int S, bool XS>
constexpr size_t gemv_staged_smem() {
  return (size_t)(XS ? 2 : 1) * S * K * D * 128 * RPC * sizeof(double);
}

}  // namespace mw
