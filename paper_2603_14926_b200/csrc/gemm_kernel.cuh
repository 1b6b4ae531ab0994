// gemm_kernel.cuh — the tiled DD/TD/QD GEMM kernel template (see gemm.cu
// for the semantics and the design notes).  Parameterised by a tile
// configuration Cf {BM, BN, BK, TM, TN, MINB}; gemm.cu instantiates the
// product configurations, the tuning harness (tune/) explores others.
#pragma once

#include "common.cuh"

namespace mw {

constexpr int GEMM_GROUP_M = 16;

// Cf::VEC = true: A staged transposed (t-major, rows contiguous) and each
// thread owns contiguous rows / columns, so register fragments load as
// 128-bit double2 pairs (half the LDS instructions).  Same arithmetic and
// order: results are bit-identical.
template <int K, class C>
struct GemmSmem {
  static constexpr int APAD = C::VEC ? C::BM + 2 : C::BK + 2;  // A tile row stride (doubles)
  static constexpr int A_ELEMS = C::VEC ? K * C::BK * APAD : K * C::BM * APAD;
  static constexpr int B_ELEMS = K * C::BK * C::BN;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr int STAGES = 2;
  static constexpr size_t BYTES = sizeof(double) * STAGE * STAGES;
};

// EXT = false: one product from an exact zero (the hot path); EXT = true:
// a batch of products (blockIdx.y strides the batch) with an optional
// initial accumulator Cin, used by the Strassen scheme.
template <int K, int VAR, bool EXT, class Cf>
__global__ void __launch_bounds__((Cf::BM / Cf::TM) * (Cf::BN / Cf::TN), Cf::MINB)
    gemm_kernel(const double* __restrict__ A0, int64_t lda, int64_t sA,
                const double* __restrict__ B0, int64_t ldb, int64_t sB, double* __restrict__ C0,
                int64_t ldc, int64_t sC, int64_t m, int64_t n, int64_t kd,
                const double* __restrict__ Cin0, int64_t ldci, int64_t sCi, int64_t batch,
                int64_t bsA, int64_t bsB, int64_t bsC, int64_t bsCi) {
  using S = GemmSmem<K, Cf>;
  constexpr int BM = Cf::BM, BN = Cf::BN, BK = Cf::BK, TM = Cf::TM, TN = Cf::TN;
  constexpr int TX = BN / TN, TY = BM / TM, NT = TX * TY;
  extern __shared__ __align__(16) double smem[];

  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  // Grouped raster: consecutive CTAs walk GROUP_M tile-rows of one
  // tile-column band, so the ~300 co-resident CTAs share A and B panels in
  // L2 and B is streamed from HBM ~grid_m/GROUP_M times instead of grid_m.
  const int64_t grid_m = (m + BM - 1) / BM, grid_n = (n + BN - 1) / BN;
  const int64_t pid = blockIdx.x;
  const int64_t per_group = (int64_t)GEMM_GROUP_M * grid_n;
  const int64_t first_m = (pid / per_group) * GEMM_GROUP_M;
  const int64_t gsize = (grid_m - first_m) < GEMM_GROUP_M ? (grid_m - first_m) : GEMM_GROUP_M;
  const int64_t in_group = pid % per_group;
  const int64_t m0 = (first_m + in_group % gsize) * BM, n0 = (in_group / gsize) * BN;

  auto As = [&](int st, int c, int row, int t) -> double& {
    if (Cf::VEC) return smem[st * S::STAGE + (c * BK + t) * S::APAD + row];
    return smem[st * S::STAGE + (c * BM + row) * S::APAD + t];
  };
  // column of the thread's q-th output
  auto col_of = [&](int q) { return Cf::VEC ? tx * TN + q : tx + q * TX; };
  auto Bs = [&](int st, int c, int t, int col) -> double& {
    return smem[st * S::STAGE + S::A_ELEMS + (c * BK + t) * BN + col];
  };

  auto load_stage = [&](const double* __restrict__ A, const double* __restrict__ B, int st,
                        int64_t k0) {
    // A tile: K x BM x BK, consecutive threads walk a row's BK doubles.
#pragma unroll
    for (int e = tid; e < K * BM * BK; e += NT) {
      const int c = e / (BM * BK), rem = e % (BM * BK);
      const int row = Cf::VEC ? rem % BM : rem / BK, t = Cf::VEC ? rem / BM : rem % BK;
      const int64_t gi = m0 + row, gt = k0 + t;
      const bool ok = gi < m && gt < kd;
      const double* src = ok ? A + c * sA + gi * lda + gt : A;
      cp_async8(&As(st, c, row, t), src, ok ? 8 : 0);
    }
    // B tile: K x BK x BN, consecutive threads walk a row's BN doubles.
#pragma unroll
    for (int e = tid; e < K * BK * BN; e += NT) {
      const int c = e / (BK * BN), rem = e % (BK * BN), t = rem / BN, col = rem % BN;
      const int64_t gt = k0 + t, gj = n0 + col;
      const bool ok = gt < kd && gj < n;
      const double* src = ok ? B + c * sB + gt * ldb + gj : B;
      cp_async8(&Bs(st, c, t, col), src, ok ? 8 : 0);
    }
  };

  // Interior tiles of 16-byte aligned operands (every tile of the benchmark
  // shapes): the same stage as 16-byte copies with no edge predicates -- half
  // the copy instructions and a fraction of the address arithmetic, which all
  // issue between the FP64 instructions of the other warps.
  auto load_stage_fast = [&](const double* __restrict__ A, const double* __restrict__ B, int st,
                             int64_t k0) {
    constexpr int HA = BK / 2, HB = BN / 2;
#pragma unroll
    for (int p = tid; p < K * BM * HA; p += NT) {
      const int c = p / (BM * HA), rem = p % (BM * HA), row = rem / HA, t = 2 * (rem % HA);
      cp_async16(&As(st, c, row, t), A + c * sA + (m0 + row) * lda + (k0 + t), 16);
    }
#pragma unroll
    for (int p = tid; p < K * BK * HB; p += NT) {
      const int c = p / (BK * HB), rem = p % (BK * HB), t = rem / HB, col = 2 * (rem % HB);
      cp_async16(&Bs(st, c, t, col), B + c * sB + (k0 + t) * ldb + (n0 + col), 16);
    }
  };
  const bool fast_ok = !Cf::VEC && (BK % 2 == 0) && (BN % 2 == 0) && m0 + BM <= m && n0 + BN <= n &&
                       (((reinterpret_cast<uintptr_t>(A0) | reinterpret_cast<uintptr_t>(B0)) & 15) == 0) &&
                       (((lda | ldb | sA | sB | (EXT ? (bsA | bsB) : 0)) & 1) == 0);

  const int64_t nbatch = EXT ? batch : 1;
  for (int64_t bi = EXT ? blockIdx.y : 0; bi < nbatch; bi += EXT ? gridDim.y : 1) {
  if (EXT && bi != blockIdx.y) __syncthreads();  // smem reuse across batch items
  const double* __restrict__ A = EXT ? A0 + bi * bsA : A0;
  const double* __restrict__ B = EXT ? B0 + bi * bsB : B0;
  double* __restrict__ C = EXT ? C0 + bi * bsC : C0;
  const double* __restrict__ Cin = (EXT && Cin0) ? Cin0 + bi * bsCi : nullptr;
  V<K> acc[TM][TN];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int q = 0; q < TN; ++q) {
      acc[r][q] = zero<K>();
      // optional initial accumulator (the Strassen peel folds start from a
      // product, linalg.py:470-500)
      const int64_t gi = m0 + ty * TM + r, gj = n0 + col_of(q);
      if (EXT && Cin && gi < m && gj < n) acc[r][q] = load<K>(Cin + gi * ldci + gj, sCi, 0);
    }

  const int64_t ntiles = (kd + BK - 1) / BK;
  if (ntiles > 0) {
    if (fast_ok && BK <= kd)
      load_stage_fast(A, B, 0, 0);
    else
      load_stage(A, B, 0, 0);
    cp_async_commit();
  }
  for (int64_t kt = 0; kt < ntiles; ++kt) {
    const int st = (int)(kt & 1);
    if (kt + 1 < ntiles) {
      if (fast_ok && (kt + 2) * BK <= kd)
        load_stage_fast(A, B, st ^ 1, (kt + 1) * BK);
      else
        load_stage(A, B, st ^ 1, (kt + 1) * BK);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int64_t rem = kd - kt * BK;
    const int tvalid = rem < BK ? (int)rem : BK;
#pragma unroll 1
    for (int t = 0; t < tvalid; ++t) {
      V<K> a[TM], b[TN];
      if (Cf::VEC) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
#pragma unroll
          for (int r = 0; r < TM; r += 2) {
            const double2 v = *reinterpret_cast<const double2*>(&As(st, c, ty * TM + r, t));
            a[r].c[c] = v.x;
            a[r + 1].c[c] = v.y;
          }
#pragma unroll
          for (int q = 0; q < TN; q += 2) {
            const double2 v = *reinterpret_cast<const double2*>(&Bs(st, c, t, tx * TN + q));
            b[q].c[c] = v.x;
            b[q + 1].c[c] = v.y;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < TM; ++r)
#pragma unroll
          for (int c = 0; c < K; ++c) a[r].c[c] = As(st, c, ty * TM + r, t);
#pragma unroll
        for (int q = 0; q < TN; ++q)
#pragma unroll
          for (int c = 0; c < K; ++c) b[q].c[c] = Bs(st, c, t, tx + q * TX);
      }
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int q = 0; q < TN; ++q)
          acc[r][q] = Ops<K, VAR>::add(acc[r][q], Ops<K, VAR>::mul(a[r], b[q]));
    }
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < TM; ++r) {
    const int64_t gi = m0 + ty * TM + r;
    if (gi >= m) continue;
#pragma unroll
    for (int q = 0; q < TN; ++q) {
      const int64_t gj = n0 + col_of(q);
      if (gj >= n) continue;
#pragma unroll
      for (int c = 0; c < K; ++c) C[c * sC + gi * ldc + gj] = acc[r][q].c[c];
    }
  }
  }  // batch
}

}  // namespace mw
