// dk.cu — one Durand-Kerner sweep in complex K-word arithmetic.
//
// Reference: roots.dk_iterate (roots.py:240-315).  For every root i
// (Jacobi: all read the frozen previous state):
//   numerator   acc = (1, 0); for c = n-1..0: acc = c_mul(acc, z_i);
//               acc = c_add(acc, (coef_c, 0))                (271-276)
//   denominator den = (1, 0); for j = 0..n-1: f = c_sub(z_i, z_j), the
//               j == i factor pinned to (1, 0); den = c_mul(den, f) (278-293)
//   step        mag = dr^2 + di^2; num = acc * conj(den);
//               step = num / mag (Newton reciprocal)          (297-303)
//   update      z_i - step; |step| = hypot(step_re0, step_im0) (305-308)
// with the local 3M complex product (roots.py:258-267).
//
// exact_order = 1: the numerator and the denominator of root i run on two
// lanes of different warps (independent chains), each replaying the
// reference order op for op; the tail follows on the numerator lane.  Bit
// exact.  The reciprocal of mag is computed once and applied to both
// parts, which is the identical op sequence the reference runs twice.
//
// exact_order = 0 (tree): a warp per root.  Lane l owns factors
// j = l, l+32, ... (ascending, from (1,0)) and the coefficient block
// [l*B, (l+1)*B) of the monic polynomial, evaluated by Horner and scaled by
// (z^B)^l; lane results combine in a pairwise shuffle tree.  Same
// arithmetic per term, reassociated: within the n*2^-p relative bound.
#include <climits>

#include "common.cuh"

namespace mw {

template <int K, int VAR>
struct Cx {
  V<K> re, im;
};

template <int K, int VAR>
__device__ __forceinline__ Cx<K, VAR> c_mul(const Cx<K, VAR>& a, const Cx<K, VAR>& b) {
  using O = Ops<K, VAR>;
  V<K> p1 = O::mul(a.re, b.re);
  V<K> p2 = O::mul(a.im, b.im);
  V<K> p3 = O::mul(O::add(a.re, a.im), O::add(b.re, b.im));
  Cx<K, VAR> r;
  r.re = O::add(p1, neg(p2));
  r.im = O::add(O::add(p3, neg(p1)), neg(p2));
  return r;
}

template <int K, int VAR>
__device__ __forceinline__ Cx<K, VAR> c_one() {
  Cx<K, VAR> r;
  r.re = constant<K>(1.0);
  r.im = zero<K>();
  return r;
}

// Shared tail: step = acc * conj(den) / |den|^2, z - step (roots.py:297-308).
template <int K, int VAR>
__device__ __forceinline__ void dk_tail(const Cx<K, VAR>& acc, const Cx<K, VAR>& den,
                                        const Cx<K, VAR>& z, double* zre_out, double* zim_out,
                                        int64_t so, double* step_mag, int64_t i) {
  using O = Ops<K, VAR>;
  V<K> mag = O::add(O::mul(den.re, den.re), O::mul(den.im, den.im));
  V<K> num_re = O::add(O::mul(acc.re, den.re), O::mul(acc.im, den.im));
  V<K> num_im = O::add(O::mul(acc.im, den.re), neg(O::mul(acc.re, den.im)));
  V<K> rcp = recip_newton<K, VAR>(mag);
  V<K> step_re = O::mul(num_re, rcp);
  V<K> step_im = O::mul(num_im, rcp);
  store<K>(zre_out, so, i, O::add(z.re, neg(step_re)));
  store<K>(zim_out, so, i, O::add(z.im, neg(step_im)));
  step_mag[i] = hypot(step_re.c[0], step_im.c[0]);
}

constexpr int DK_EXACT_ROOTS = 32;  // roots per CTA (two warps: num + den)
constexpr int DK_CH = 128;          // roots staged in smem per chunk

template <int K, int VAR>
__global__ void __launch_bounds__(2 * DK_EXACT_ROOTS)
    dk_exact_kernel(const double* __restrict__ coeffs, int64_t sc, int64_t n,
                    const double* __restrict__ zre, const double* __restrict__ zim, int64_t sz,
                    int64_t i0, int64_t i1, double* __restrict__ zre_out,
                    double* __restrict__ zim_out, int64_t so, double* __restrict__ step_mag,
                    int* __restrict__ flag) {
  using O = Ops<K, VAR>;
  __shared__ double zs[2][K][DK_CH];
  __shared__ double dx[2][K][DK_EXACT_ROOTS];
  const int lane = threadIdx.x & 31;
  const bool is_den = threadIdx.x >= 32;
  const int64_t i = i0 + (int64_t)blockIdx.x * DK_EXACT_ROOTS + lane;
  const bool live = i < i1;

  Cx<K, VAR> z;
  z.re = live ? load<K>(zre, sz, i) : zero<K>();
  z.im = live ? load<K>(zim, sz, i) : zero<K>();
  Cx<K, VAR> acc = c_one<K, VAR>();

  if (!is_den) {
    for (int64_t c = n - 1; c >= 0; --c) {
      acc = c_mul(acc, z);
      Cx<K, VAR> ci;
      ci.re = load<K>(coeffs, sc, c);
      ci.im = zero<K>();
      acc.re = O::add(acc.re, ci.re);
      acc.im = O::add(acc.im, ci.im);
    }
  }
  // denominator: all threads stage z_j chunks (both warps join the syncs)
  for (int64_t j0 = 0; j0 < n; j0 += DK_CH) {
    const int cnt = (int)((n - j0) < DK_CH ? (n - j0) : DK_CH);
    __syncthreads();
    for (int e = threadIdx.x; e < K * cnt; e += 2 * DK_EXACT_ROOTS) {
      const int c = e / cnt, jj = e % cnt;
      zs[0][c][jj] = zre[c * sz + j0 + jj];
      zs[1][c][jj] = zim[c * sz + j0 + jj];
    }
    __syncthreads();
    if (is_den) {
      for (int jj = 0; jj < cnt; ++jj) {
        const int64_t j = j0 + jj;
        Cx<K, VAR> zj, f;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          zj.re.c[c] = zs[0][c][jj];
          zj.im.c[c] = zs[1][c][jj];
        }
        f.re = O::add(z.re, neg(zj.re));
        f.im = O::add(z.im, neg(zj.im));
        if (j == i) f = c_one<K, VAR>();
        if (live && fabs(f.re.c[0]) + fabs(f.im.c[0]) == 0.0) {
          const long long key = (long long)j * n + i;
          atomicMin(flag, key > INT_MAX ? INT_MAX : (int)key);
        }
        acc = c_mul(acc, f);
      }
    }
  }
  __syncthreads();
  if (is_den) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      dx[0][c][lane] = acc.re.c[c];
      dx[1][c][lane] = acc.im.c[c];
    }
  }
  __syncthreads();
  if (!is_den && live) {
    Cx<K, VAR> den;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      den.re.c[c] = dx[0][c][lane];
      den.im.c[c] = dx[1][c][lane];
    }
    dk_tail<K, VAR>(acc, den, z, zre_out, zim_out, so, step_mag, i);
  }
}

// ----------------------------------------------------------- tree order
constexpr int DK_TREE_WARPS = 4;  // roots per CTA

template <int K, int VAR>
__device__ __forceinline__ Cx<K, VAR> shfl_down_cx(const Cx<K, VAR>& v, int s) {
  Cx<K, VAR> r;
  r.re = shfl_down<K>(v.re, s);
  r.im = shfl_down<K>(v.im, s);
  return r;
}

template <int K, int VAR>
__global__ void __launch_bounds__(32 * DK_TREE_WARPS)
    dk_tree_kernel(const double* __restrict__ coeffs, int64_t sc, int64_t n,
                   const double* __restrict__ zre, const double* __restrict__ zim, int64_t sz,
                   int64_t i0, int64_t i1, double* __restrict__ zre_out,
                   double* __restrict__ zim_out, int64_t so, double* __restrict__ step_mag,
                   int* __restrict__ flag) {
  using O = Ops<K, VAR>;
  const int lane = threadIdx.x & 31;
  const int64_t i = i0 + (int64_t)blockIdx.x * DK_TREE_WARPS + (threadIdx.x >> 5);
  if (i >= i1) return;
  Cx<K, VAR> z;
  z.re = load<K>(zre, sz, i);
  z.im = load<K>(zim, sz, i);

  // ---- denominator: lane l folds j = l, l+32, ... ascending
  Cx<K, VAR> den = c_one<K, VAR>();
  for (int64_t j = lane; j < n; j += 32) {
    Cx<K, VAR> f;
    f.re = O::add(z.re, neg(load<K>(zre, sz, j)));
    f.im = O::add(z.im, neg(load<K>(zim, sz, j)));
    if (j == i) f = c_one<K, VAR>();
    if (fabs(f.re.c[0]) + fabs(f.im.c[0]) == 0.0) {
      const long long key = (long long)j * n + i;
      atomicMin(flag, key > INT_MAX ? INT_MAX : (int)key);
    }
    den = c_mul(den, f);
  }

  // ---- numerator: monic coefficients a_0..a_n (a_n = 1), block size B
  const int64_t B = (n + 1 + 31) / 32;
  const int64_t lo = lane * B;
  const int64_t hi = (lo + B < n + 1) ? lo + B : n + 1;  // [lo, hi)
  Cx<K, VAR> p;
  p.re = zero<K>();
  p.im = zero<K>();
  if (lo < hi) {
    // Horner over the block: p = a_{hi-1}; p = p*z + a_c for c = hi-2..lo
    Cx<K, VAR> a;
    a.re = (hi - 1 == n) ? constant<K>(1.0) : load<K>(coeffs, sc, hi - 1);
    a.im = zero<K>();
    p = a;
    for (int64_t c = hi - 2; c >= lo; --c) {
      p = c_mul(p, z);
      p.re = O::add(p.re, load<K>(coeffs, sc, c));
      p.im = O::add(p.im, zero<K>());
    }
  }
  // w = z^B by square-and-multiply, then the lane's scale (z^B)^lane
  Cx<K, VAR> w = c_one<K, VAR>(), sq = z;
  for (int64_t e = B; e > 0; e >>= 1) {
    if (e & 1) w = c_mul(w, sq);
    if (e > 1) sq = c_mul(sq, sq);
  }
  Cx<K, VAR> scale = c_one<K, VAR>(), wp = w;
  for (int e = lane; e > 0; e >>= 1) {
    if (e & 1) scale = c_mul(scale, wp);
    if (e > 1) wp = c_mul(wp, wp);
  }
  Cx<K, VAR> term = c_mul(p, scale);
  const bool has_block = lo < hi;
  const int nblocks = (int)((n + 1 + B - 1) / B);

  // ---- pairwise shuffle trees (product for den, sum for the numerator)
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    Cx<K, VAR> od = shfl_down_cx(den, s);
    Cx<K, VAR> ot = shfl_down_cx(term, s);
    if ((lane & (2 * s - 1)) == 0) {
      if (lane + s < 32 && lane + s < n) den = c_mul(den, od);
      if (has_block && lane + s < nblocks) {
        term.re = O::add(term.re, ot.re);
        term.im = O::add(term.im, ot.im);
      }
    }
  }
  if (lane == 0) dk_tail<K, VAR>(term, den, z, zre_out, zim_out, so, step_mag, i);
}

template <int K, int VAR>
struct DkLaunch {
  static int run(const double* coeffs, int64_t sc, int64_t n, const double* zre,
                 const double* zim, int64_t sz, int64_t i0, int64_t i1, double* zre_out,
                 double* zim_out, int64_t so, double* step_mag, int* flag, int exact,
                 cudaStream_t st) {
    const int64_t cnt = i1 - i0;
    if (exact) {
      const int64_t blocks = (cnt + DK_EXACT_ROOTS - 1) / DK_EXACT_ROOTS;
      dk_exact_kernel<K, VAR><<<(unsigned)blocks, 2 * DK_EXACT_ROOTS, 0, st>>>(
          coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so, step_mag, flag);
    } else {
      const int64_t blocks = (cnt + DK_TREE_WARPS - 1) / DK_TREE_WARPS;
      dk_tree_kernel<K, VAR><<<(unsigned)blocks, 32 * DK_TREE_WARPS, 0, st>>>(
          coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so, step_mag, flag);
    }
    return launch_status();
  }
};

}  // namespace mw

using namespace mw;

extern "C" int mw_dk_sweep(int k, int variant, const double* coeffs, int64_t sc, int64_t n,
                           const double* zre, const double* zim, int64_t sz, int64_t i0,
                           int64_t i1, double* zre_out, double* zim_out, int64_t so,
                           double* step_mag, int* flag_dev, int exact_order, void* stream) {
  if (k < 2 || k > 4) return MW_ERR_INVALID;
  if (variant == 0 && k != 2) return MW_ERR_UNSUPPORTED;
  if (variant != 0 && variant != 1) return MW_ERR_INVALID;
  if (n < 1 || i0 < 0 || i1 < i0 || i1 > n) return MW_ERR_INVALID;
  if (i1 == i0) return MW_OK;
  if (!coeffs || !zre || !zim || !zre_out || !zim_out || !step_mag || !flag_dev)
    return MW_ERR_INVALID;
  if (sc < n || sz < n || so < n) return MW_ERR_INVALID;
  return dispatch<DkLaunch>(k, variant, coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out,
                            so, step_mag, flag_dev, exact_order ? 1 : 0, as_stream(stream));
}
