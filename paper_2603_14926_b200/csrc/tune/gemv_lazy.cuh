// gemv_lazy.cuh -- tuning probe (not in libmwgpu.so): tree-order GEMV whose
// per-thread partial accumulates the TD products LAZILY: the two_prod terms
// of a_t * x_t go straight into a three-level accumulator (level 0 and 1 by
// error-free two_sums, level 2 by plain adds), which is renormalised by two
// two_sums per element, instead of a full normalised tw_mul_bf (39) followed
// by a full tw_add_bf (57): ~61 FP64 instructions per element instead of 96.
// The 128 partials combine by the same pairwise tree of tw_add_bf as
// gemv_tree_kernel.  A different rounding sequence than the tree order's
// fold: timing probe for a possible new tree-order definition.
#pragma once
#include "../common.cuh"

namespace mw {

struct LazyTD {
  double s0, s1, s2;
};

__device__ __forceinline__ void lazy_td_mac(LazyTD& s, const V<3>& a, const V<3>& x) {
  double h00, l00, h01, l01, h10, l10;
  two_prod(a.c[0], x.c[0], h00, l00);
  two_prod(a.c[0], x.c[1], h01, l01);
  two_prod(a.c[1], x.c[0], h10, l10);
  const double q = MW_ADD(MW_ADD(MW_MUL(a.c[0], x.c[2]), MW_MUL(a.c[1], x.c[1])), MW_MUL(a.c[2], x.c[0]));
  double c0, u, v, w, y, z, r, c1;
  two_sum(s.s0, h00, s.s0, c0);
  two_sum(h01, h10, u, v);
  two_sum(l00, c0, w, y);
  two_sum(u, w, z, r);
  two_sum(s.s1, z, s.s1, c1);
  s.s2 = MW_ADD(s.s2, MW_ADD(MW_ADD(MW_ADD(v, y), MW_ADD(r, c1)), MW_ADD(MW_ADD(l01, l10), q)));
  two_sum(s.s0, s.s1, s.s0, s.s1);
  two_sum(s.s1, s.s2, s.s1, s.s2);
}

template <int RPC, int D>
__global__ void __launch_bounds__(128 * RPC)
    gemv_lazy_td_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                        const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                        int64_t m, int64_t n) {
  constexpr int K = 3, VAR = BRANCH_FREE, P = 128;
  const int lane = threadIdx.x & 31;
  const int warp = (threadIdx.x >> 5) & 3;
  const int slot = threadIdx.x >> 7;
  const int64_t i = blockIdx.x * (int64_t)RPC + slot;
  const bool live = i < m;
  const double* row = A + (live ? i : 0) * lda;
  const int u = warp * 32 + lane;
  LazyTD s{0.0, 0.0, 0.0};
  int64_t t = u;
  for (; t + (D - 1) * P < n; t += D * P) {
    V<K> a[D], xv[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      a[d] = load<K>(row, sA, t + d * P);
      xv[d] = load<K>(x, sx, t + d * P);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) lazy_td_mac(s, a[d], xv[d]);
  }
  for (; t < n; t += P) lazy_td_mac(s, load<K>(row, sA, t), load<K>(x, sx, t));
  V<K> acc;
  acc.c[0] = s.s0;
  acc.c[1] = s.s1;
  acc.c[2] = s.s2;
  const int64_t valid = n < P ? n : P;
  __shared__ double part[RPC][K][P];
#pragma unroll
  for (int c = 0; c < K; ++c) part[slot][c][u] = acc.c[c];
  __syncthreads();
  const int tid = threadIdx.x;
#pragma unroll 1
  for (int st = 1; st < P; st <<= 1) {
    const int per_row = P / (2 * st);
    if (tid < RPC * per_row) {
      const int r = tid / per_row, idx = 2 * st * (tid % per_row);
      if (idx + st < valid) {
        V<K> p, q;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          p.c[c] = part[r][c][idx];
          q.c[c] = part[r][c][idx + st];
        }
        const V<K> sum = Ops<K, VAR>::add(p, q);
#pragma unroll
        for (int c = 0; c < K; ++c) part[r][c][idx] = sum.c[c];
      }
    }
    __syncthreads();
  }
  if (warp == 0 && lane == 0 && live) {
    V<K> r0;
#pragma unroll
    for (int c = 0; c < K; ++c) r0.c[c] = part[slot][c][0];
    store<K>(y, sy, i, r0);
  }
}


// The same lazy accumulation with the next group's A loads issued (and
// pinned by a warp barrier) before the current group is folded.
template <int RPC, int D, int MINB>
__global__ void __launch_bounds__(128 * RPC, MINB)
    gemv_lazy_pin_td_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                            const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                            int64_t m, int64_t n) {
  constexpr int K = 3, VAR = BRANCH_FREE, P = 128;
  const int lane = threadIdx.x & 31;
  const int warp = (threadIdx.x >> 5) & 3;
  const int slot = threadIdx.x >> 7;
  const int64_t i = blockIdx.x * (int64_t)RPC + slot;
  const bool live = i < m;
  const double* row = A + (live ? i : 0) * lda;
  const int u = warp * 32 + lane;
  const int ulast = warp * 32 + 31;
  const int64_t ng = n > ulast ? ((n - ulast + P - 1) / P) / D : 0;
  LazyTD s{0.0, 0.0, 0.0};
  int64_t t = u;
  V<K> cur[D], nxt[D];
  if (ng > 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) cur[d] = load<K>(row, sA, t + d * P);
  }
  for (int64_t g = 0; g < ng; ++g) {
    const bool more = g + 1 < ng;
    if (more) {
#pragma unroll
      for (int d = 0; d < D; ++d) nxt[d] = load<K>(row, sA, t + (D + d) * P);
    }
    __syncwarp();
#pragma unroll
    for (int d = 0; d < D; ++d) lazy_td_mac(s, cur[d], load<K>(x, sx, t + d * P));
    t += D * P;
    if (more) {
#pragma unroll
      for (int d = 0; d < D; ++d) cur[d] = nxt[d];
    }
  }
  for (; t < n; t += P) lazy_td_mac(s, load<K>(row, sA, t), load<K>(x, sx, t));
  V<K> acc;
  acc.c[0] = s.s0;
  acc.c[1] = s.s1;
  acc.c[2] = s.s2;
  const int64_t valid = n < P ? n : P;
  __shared__ double part[RPC][K][P];
#pragma unroll
  for (int c = 0; c < K; ++c) part[slot][c][u] = acc.c[c];
  __syncthreads();
  const int tid = threadIdx.x;
#pragma unroll 1
  for (int st = 1; st < P; st <<= 1) {
    const int per_row = P / (2 * st);
    if (tid < RPC * per_row) {
      const int r = tid / per_row, idx = 2 * st * (tid % per_row);
      if (idx + st < valid) {
        V<K> p, q;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          p.c[c] = part[r][c][idx];
          q.c[c] = part[r][c][idx + st];
        }
        const V<K> sum = Ops<K, VAR>::add(p, q);
#pragma unroll
        for (int c = 0; c < K; ++c) part[r][c][idx] = sum.c[c];
      }
    }
    __syncthreads();
  }
  if (warp == 0 && lane == 0 && live) {
    V<K> r0;
#pragma unroll
    for (int c = 0; c < K; ++c) r0.c[c] = part[slot][c][0];
    store<K>(y, sy, i, r0);
  }
}

}  // namespace mw
