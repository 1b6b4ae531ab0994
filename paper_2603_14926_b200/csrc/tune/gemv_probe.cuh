// gemv_probe.cuh -- diagnostic variants of gemv_tree_kernel (tuning harness
// only): MODE 1 = same FP64 fold with operands synthesised in registers (no
// loads); MODE 2 = same loads with an integer XOR instead of the fold.
#pragma once
namespace mw {
template <int K, int VAR, int MODE, int WARPS = 4, int RPC = 2, int D = 4>
__global__ void __launch_bounds__(32 * WARPS * RPC)
    gemv_probe_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                      const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                      int64_t m, int64_t n) {
  constexpr int P = 32 * WARPS;
  const int lane = threadIdx.x & 31;
  const int warp = (threadIdx.x >> 5) % WARPS;
  const int slot = (threadIdx.x >> 5) / WARPS;
  const int64_t i = blockIdx.x * (int64_t)RPC + slot;
  const bool live = i < m;
  const double* row = A + (live ? i : 0) * lda;
  const int u = warp * 32 + lane;
  V<K> acc = zero<K>();
  unsigned long long h = 0;
  V<K> a0 = load<K>(row, sA, u), x0 = load<K>(x, sx, u);
  int64_t t = u;
  for (; t + (D - 1) * P < n; t += D * P) {
    V<K> a[D], xv[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (MODE == 1) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
          a[d].c[c] = __longlong_as_double(__double_as_longlong(a0.c[c]) ^ ((t + d) & 7));
          xv[d].c[c] = __longlong_as_double(__double_as_longlong(x0.c[c]) ^ ((t + 2 * d) & 7));
        }
      } else {
        a[d] = load<K>(row, sA, t + d * P);
        xv[d] = load<K>(x, sx, t + d * P);
      }
    }
    if (MODE == 2) {
#pragma unroll
      for (int d = 0; d < D; ++d)
#pragma unroll
        for (int c = 0; c < K; ++c) h ^= __double_as_longlong(a[d].c[c]) ^ __double_as_longlong(xv[d].c[c]);
    } else {
#pragma unroll
      for (int d = 0; d < D; ++d) acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a[d], xv[d]));
    }
  }
  if (live && (acc.c[0] == 1.2345 || h == 12345)) y[i] = acc.c[K - 1] + (double)h;
}
}  // namespace mw

namespace mw {
// Tree-order GEMV variants (same partials / tree as gemv_tree_kernel, so
// bit-identical): a 128-thread CTA owns RT consecutive rows; thread u folds
// partial u of all RT rows (RT independent chains sharing each x load);
// D elements per group; PIPE: group g+1 is loaded before group g is folded
// (register double buffer) so HBM/L2 latency overlaps the fold.
template <int K, int VAR, int RT, int D, bool PIPE, int MINB = 1>
__global__ void __launch_bounds__(128, MINB)
    gemv_rt_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                   const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                   int64_t m, int64_t n) {
  constexpr int P = 128;
  const int u = threadIdx.x;
  const int64_t i0 = blockIdx.x * (int64_t)RT;
  const double* rows[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) rows[r] = A + (i0 + r < m ? i0 + r : 0) * lda;
  V<K> acc[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) acc[r] = zero<K>();
  const int64_t cnt = n > u ? (n - u + P - 1) / P : 0;  // elements of partial u
  const int64_t ng = cnt / D;
  auto ld = [&](V<K> (&a)[RT][D], V<K> (&xv)[D], int64_t gi) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t t = u + (gi * D + d) * P;
      xv[d] = load<K>(x, sx, t);
#pragma unroll
      for (int r = 0; r < RT; ++r) a[r][d] = load<K>(rows[r], sA, t);
    }
  };
  auto fold = [&](V<K> (&a)[RT][D], V<K> (&xv)[D]) {
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int r = 0; r < RT; ++r) acc[r] = Ops<K, VAR>::add(acc[r], Ops<K, VAR>::mul(a[r][d], xv[d]));
  };
  if (PIPE) {
    V<K> a0[RT][D], x0[D];
    if (ng > 0) ld(a0, x0, 0);
    for (int64_t gi = 0; gi < ng; ++gi) {
      V<K> a1[RT][D], x1[D];
      if (gi + 1 < ng) ld(a1, x1, gi + 1);
      fold(a0, x0);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        x0[d] = x1[d];
#pragma unroll
        for (int r = 0; r < RT; ++r) a0[r][d] = a1[r][d];
      }
    }
  } else {
    for (int64_t gi = 0; gi < ng; ++gi) {
      V<K> a0[RT][D], x0[D];
      ld(a0, x0, gi);
      fold(a0, x0);
    }
  }
  for (int64_t t = u + ng * D * P; t < n; t += P) {
    const V<K> xv = load<K>(x, sx, t);
#pragma unroll
    for (int r = 0; r < RT; ++r)
      acc[r] = Ops<K, VAR>::add(acc[r], Ops<K, VAR>::mul(load<K>(rows[r], sA, t), xv));
  }
  const int64_t valid = n < P ? n : P;
  __shared__ double part[RT][K][P];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c) part[r][c][u] = acc[r].c[c];
  __syncthreads();
#pragma unroll 1
  for (int s = 1; s < P; s <<= 1) {
    const int per_row = P / (2 * s);
    for (int w = u; w < RT * per_row; w += P) {
      const int r = w / per_row, idx = 2 * s * (w % per_row);
      if (idx + s < valid) {
        V<K> l, rr;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          l.c[c] = part[r][c][idx];
          rr.c[c] = part[r][c][idx + s];
        }
        const V<K> sum = Ops<K, VAR>::add(l, rr);
#pragma unroll
        for (int c = 0; c < K; ++c) part[r][c][idx] = sum.c[c];
      }
    }
    __syncthreads();
  }
  if (u < RT && i0 + u < m) {
    V<K> r0;
#pragma unroll
    for (int c = 0; c < K; ++c) r0.c[c] = part[u][c][0];
    store<K>(y, sy, i0 + u, r0);
  }
}
}  // namespace mw

namespace mw {
// Experimental fold order (timing only): P = 128 * C partials per row, 128
// threads per row, thread u folds the C partials u, u+128, ... (partial v
// folds t = v, v + P, ...) as C independent chains stepped together, D
// elements per chain loaded ahead; the partials combine by the pairwise
// tree over P in shared memory.
template <int K, int VAR, int C, int D, int RPC = 1>
__global__ void __launch_bounds__(128 * RPC)
    gemv_mc_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                   const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                   int64_t m, int64_t n) {
  constexpr int P = 128 * C;
  const int u = threadIdx.x % 128, slot = threadIdx.x / 128;
  const int64_t i = blockIdx.x * (int64_t)RPC + slot;
  const bool live = i < m;
  const double* row = A + (live ? i : 0) * lda;
  V<K> acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = zero<K>();
  int64_t t = u;
  for (; t + (int64_t)(D - 1) * P + (C - 1) * 128 < n; t += (int64_t)D * P) {
    V<K> a[D][C], xv[D][C];
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        a[d][c] = load<K>(row, sA, t + d * P + c * 128);
        xv[d][c] = load<K>(x, sx, t + d * P + c * 128);
      }
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = Ops<K, VAR>::add(acc[c], Ops<K, VAR>::mul(a[d][c], xv[d][c]));
  }
  for (; t < n; t += P)
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (t + c * 128 < n)
        acc[c] = Ops<K, VAR>::add(acc[c], Ops<K, VAR>::mul(load<K>(row, sA, t + c * 128), load<K>(x, sx, t + c * 128)));
  __shared__ double part[RPC][K][P];
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int k = 0; k < K; ++k) part[slot][k][u + c * 128] = acc[c].c[k];
  __syncthreads();
  const int64_t valid = n < P ? n : P;
#pragma unroll 1
  for (int s = 1; s < P; s <<= 1) {
    const int pairs = P / (2 * s);
    for (int w = u; w < pairs; w += 128) {
      const int idx = 2 * s * w;
      if (idx + s < valid) {
        V<K> l, r;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          l.c[k] = part[slot][k][idx];
          r.c[k] = part[slot][k][idx + s];
        }
        const V<K> sum = Ops<K, VAR>::add(l, r);
#pragma unroll
        for (int k = 0; k < K; ++k) part[slot][k][idx] = sum.c[k];
      }
    }
    __syncthreads();
  }
  if (u == 0 && live) {
    V<K> r0;
#pragma unroll
    for (int k = 0; k < K; ++k) r0.c[k] = part[slot][k][0];
    store<K>(y, sy, i, r0);
  }
}
}  // namespace mw

namespace mw {
// Experimental fold order (timing only): 128 partials per row, partial u
// folds the column PAIRS (2u + 256j, 2u + 1 + 256j), j ascending, so every
// A and x access is one 16-byte load per lane (LDG.128); D pairs ahead.
template <int K, int VAR, int D, int RPC = 2>
__global__ void __launch_bounds__(128 * RPC)
    gemv_v2_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                   const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                   int64_t m, int64_t n) {
  constexpr int P = 128;
  const int u = threadIdx.x % P, slot = threadIdx.x / P;
  const int64_t i = blockIdx.x * (int64_t)RPC + slot;
  const bool live = i < m;
  const double* row = A + (live ? i : 0) * lda;
  V<K> acc = zero<K>();
  auto ld2 = [&](const double* base, int64_t stride, int64_t t, V<K>& lo, V<K>& hi) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const double2 v = *reinterpret_cast<const double2*>(base + c * stride + t);
      lo.c[c] = v.x;
      hi.c[c] = v.y;
    }
  };
  for (int64_t t = 2 * u; t < n; t += (int64_t)2 * P * D) {
    V<K> a0[D], a1[D], x0[D], x1[D];
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (t + (int64_t)2 * P * d < n) {
        ld2(row, sA, t + (int64_t)2 * P * d, a0[d], a1[d]);
        ld2(x, sx, t + (int64_t)2 * P * d, x0[d], x1[d]);
      }
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (t + (int64_t)2 * P * d < n) {
        acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a0[d], x0[d]));
        acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a1[d], x1[d]));
      }
  }
  __shared__ double part[RPC][K][P];
#pragma unroll
  for (int k = 0; k < K; ++k) part[slot][k][u] = acc.c[k];
  __syncthreads();
#pragma unroll 1
  for (int s = 1; s < P; s <<= 1) {
    const int per_row = P / (2 * s);
    const int tid = threadIdx.x;
    if (tid < RPC * per_row) {
      const int r = tid / per_row, idx = 2 * s * (tid % per_row);
      V<K> l, rr;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        l.c[k] = part[r][k][idx];
        rr.c[k] = part[r][k][idx + s];
      }
      const V<K> sum = Ops<K, VAR>::add(l, rr);
#pragma unroll
      for (int k = 0; k < K; ++k) part[r][k][idx] = sum.c[k];
    }
    __syncthreads();
  }
  if (u == 0 && live) {
    V<K> r0;
#pragma unroll
    for (int k = 0; k < K; ++k) r0.c[k] = part[slot][k][0];
    store<K>(y, sy, i, r0);
  }
}
}  // namespace mw

namespace mw {
// gemv_tree_kernel's partials and tree (bit-identical) with x staged in
// shared memory once per CTA (RPC rows share it): the fold loads only A
// from global memory; x comes from shared memory.
template <int K, int VAR, int RPC, int D>
__global__ void __launch_bounds__(128 * RPC, 1)
    gemv_xs_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                   const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                   int64_t m, int64_t n) {
  constexpr int P = 128;
  extern __shared__ double xs[];  // [K][n], then part [RPC][K][P]
  double* part = xs + (size_t)K * n;
  const int u = threadIdx.x % P, slot = threadIdx.x / P;
  for (int64_t e = threadIdx.x; e < (int64_t)K * n; e += blockDim.x) {
    const int64_t c = e / n, t = e % n;
    xs[e] = x[c * sx + t];
  }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)RPC + slot; i - slot < m; i += (int64_t)gridDim.x * RPC) {
    const bool live = i < m;
    const double* row = A + (live ? i : 0) * lda;
    V<K> acc = zero<K>();
    int64_t t = u;
    for (; t + (D - 1) * P < n; t += D * P) {
      V<K> a[D];
#pragma unroll
      for (int d = 0; d < D; ++d) a[d] = load<K>(row, sA, t + d * P);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        V<K> xv;
#pragma unroll
        for (int c = 0; c < K; ++c) xv.c[c] = xs[c * n + t + d * P];
        acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a[d], xv));
      }
    }
    for (; t < n; t += P) {
      V<K> xv;
#pragma unroll
      for (int c = 0; c < K; ++c) xv.c[c] = xs[c * n + t];
      acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(row, sA, t), xv));
    }
    const int64_t valid = n < P ? n : P;
#pragma unroll
    for (int c = 0; c < K; ++c) part[(slot * K + c) * P + u] = acc.c[c];
    __syncthreads();
#pragma unroll 1
    for (int s = 1; s < P; s <<= 1) {
      const int per_row = P / (2 * s);
      const int tid = threadIdx.x;
      if (tid < RPC * per_row) {
        const int r = tid / per_row, idx = 2 * s * (tid % per_row);
        if (idx + s < valid) {
          V<K> l, rr;
#pragma unroll
          for (int c = 0; c < K; ++c) {
            l.c[c] = part[(r * K + c) * P + idx];
            rr.c[c] = part[(r * K + c) * P + idx + s];
          }
          const V<K> sum = Ops<K, VAR>::add(l, rr);
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
    __syncthreads();
  }
}
}  // namespace mw

namespace mw {
// gemv_tree_kernel with A read through streaming loads (ld.global.cs:
// evict-first, A is read exactly once); same partials and tree.
template <int K, int VAR, int RPC, int D>
__global__ void __launch_bounds__(128 * RPC)
    gemv_cs_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                   const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                   int64_t m, int64_t n) {
  constexpr int P = 128;
  const int u = threadIdx.x % P, slot = threadIdx.x / P;
  const int64_t i = blockIdx.x * (int64_t)RPC + slot;
  const bool live = i < m;
  const double* row = A + (live ? i : 0) * lda;
  V<K> acc = zero<K>();
  int64_t t = u;
  for (; t + (D - 1) * P < n; t += D * P) {
    V<K> a[D], xv[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
#pragma unroll
      for (int c = 0; c < K; ++c) a[d].c[c] = __ldcs(row + c * sA + t + d * P);
      xv[d] = load<K>(x, sx, t + d * P);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a[d], xv[d]));
  }
  for (; t < n; t += P)
    acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(row, sA, t), load<K>(x, sx, t)));
  __shared__ double part[RPC][K][P];
#pragma unroll
  for (int c = 0; c < K; ++c) part[slot][c][u] = acc.c[c];
  __syncthreads();
  const int64_t valid = n < P ? n : P;
#pragma unroll 1
  for (int s = 1; s < P; s <<= 1) {
    const int per_row = P / (2 * s);
    const int tid = threadIdx.x;
    if (tid < RPC * per_row) {
      const int r = tid / per_row, idx = 2 * s * (tid % per_row);
      if (idx + s < valid) {
        V<K> l, rr;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          l.c[c] = part[r][c][idx];
          rr.c[c] = part[r][c][idx + s];
        }
        const V<K> sum = Ops<K, VAR>::add(l, rr);
#pragma unroll
        for (int c = 0; c < K; ++c) part[r][c][idx] = sum.c[c];
      }
    }
    __syncthreads();
  }
  if (u == 0 && live) {
    V<K> r0;
#pragma unroll
    for (int c = 0; c < K; ++c) r0.c[c] = part[slot][c][0];
    store<K>(y, sy, i, r0);
  }
}
}  // namespace mw
