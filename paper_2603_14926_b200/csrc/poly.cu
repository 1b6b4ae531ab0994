// poly.cu — Estrin and complex-argument polynomial evaluation, batched
// over points.
//
// Reference (pkg/src/mwfloat/poly.py):
//   estrin_eval / estrin_eval_batched (106-153): coefficients zero-padded
//     to a power of two; repeat { level[i] = add(level[2i], mul(level[2i+1],
//     x)); x = mul(x, x) unless this was the last level }.
//   eval_complex (156-178): the same two schemes over (re, im) pairs with
//     the 3M complex product (multiword.cmul, 683-692) and cadd (675-676),
//     coefficients (a_i, 0).
// The kernels run one point per thread.  Estrin is evaluated in post-order
// with a per-thread stack of pending left siblings (one per tree level),
// which computes every node from the same children with the same power as
// the level-by-level reference: bit-exact per point.  Horner for complex
// points mirrors the real Horner kernel.
#include "common.cuh"

namespace mw {

constexpr int POLY_LMAX = 26;  // up to 2^26 padded coefficients

// ---------------------------------------------------------------- rings
template <int K, int VAR>
struct RealRing {
  using T = V<K>;
  static __device__ __forceinline__ T mul(const T& a, const T& b) { return Ops<K, VAR>::mul(a, b); }
  static __device__ __forceinline__ T add(const T& a, const T& b) { return Ops<K, VAR>::add(a, b); }
  static __device__ __forceinline__ T coef(const double* c, int64_t sc, int64_t i) { return load<K>(c, sc, i); }
  static __device__ __forceinline__ T zero_() { return zero<K>(); }
  static __device__ __forceinline__ T ld(const double* re, const double*, int64_t s, int64_t i) {
    return load<K>(re, s, i);
  }
  static __device__ __forceinline__ void st(double* re, double*, int64_t s, int64_t i, const T& v) {
    store<K>(re, s, i, v);
  }
};

template <int K, int VAR>
struct CplxRing {
  struct T {
    V<K> re, im;
  };
  // multiword.cmul (683-692): p1 = ar*br, p2 = ai*bi, p3 = (ar+ai)(br+bi);
  // re = p1 - p2, im = (p3 - p1) - p2, subtraction = add of the negation.
  static __device__ __forceinline__ T mul(const T& a, const T& b) {
    using O = Ops<K, VAR>;
    V<K> p1 = O::mul(a.re, b.re);
    V<K> p2 = O::mul(a.im, b.im);
    V<K> p3 = O::mul(O::add(a.re, a.im), O::add(b.re, b.im));
    T r;
    r.re = O::add(p1, neg(p2));
    r.im = O::add(O::add(p3, neg(p1)), neg(p2));
    return r;
  }
  static __device__ __forceinline__ T add(const T& a, const T& b) {
    T r;
    r.re = Ops<K, VAR>::add(a.re, b.re);
    r.im = Ops<K, VAR>::add(a.im, b.im);
    return r;
  }
  static __device__ __forceinline__ T coef(const double* c, int64_t sc, int64_t i) {
    T r;
    r.re = load<K>(c, sc, i);
    r.im = zero<K>();
    return r;
  }
  static __device__ __forceinline__ T zero_() {
    T r;
    r.re = zero<K>();
    r.im = zero<K>();
    return r;
  }
  static __device__ __forceinline__ T ld(const double* re, const double* im, int64_t s, int64_t i) {
    T r;
    r.re = load<K>(re, s, i);
    r.im = load<K>(im, s, i);
    return r;
  }
  static __device__ __forceinline__ void st(double* re, double* im, int64_t s, int64_t i, const T& v) {
    store<K>(re, s, i, v.re);
    store<K>(im, s, i, v.im);
  }
};

// ------------------------------------------------------------- kernels
template <class R>
__global__ void __launch_bounds__(128) estrin_kernel(const double* __restrict__ coeffs, int64_t sc,
                                                     int64_t degree, int levels,
                                                     const double* __restrict__ xre,
                                                     const double* __restrict__ xim, int64_t sx,
                                                     double* __restrict__ yre,
                                                     double* __restrict__ yim, int64_t sy,
                                                     int64_t npts) {
  using T = typename R::T;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (levels == 0) {  // a single coefficient: returned as is
      R::st(yre, yim, sy, p, R::coef(coeffs, sc, 0));
      continue;
    }
    T pw[POLY_LMAX];
    T stack[POLY_LMAX + 1];
    pw[0] = R::ld(xre, xim, sx, p);
    for (int l = 1; l < levels; ++l) pw[l] = R::mul(pw[l - 1], pw[l - 1]);
    const int64_t pairs = (int64_t)1 << (levels - 1);
    for (int64_t i = 0; i < pairs; ++i) {
      const T left = (2 * i <= degree) ? R::coef(coeffs, sc, 2 * i) : R::zero_();
      const T right = (2 * i + 1 <= degree) ? R::coef(coeffs, sc, 2 * i + 1) : R::zero_();
      T v = R::add(left, R::mul(right, pw[0]));
      int j = 1;
      for (int64_t idx = i; idx & 1; idx >>= 1, ++j) v = R::add(stack[j], R::mul(v, pw[j]));
      stack[j] = v;
    }
    R::st(yre, yim, sy, p, stack[levels]);
  }
}

template <class R>
__global__ void __launch_bounds__(128) horner_ring_kernel(const double* __restrict__ coeffs,
                                                          int64_t sc, int64_t degree,
                                                          const double* __restrict__ xre,
                                                          const double* __restrict__ xim,
                                                          int64_t sx, double* __restrict__ yre,
                                                          double* __restrict__ yim, int64_t sy,
                                                          int64_t npts) {
  using T = typename R::T;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
       p += (int64_t)gridDim.x * blockDim.x) {
    const T z = R::ld(xre, xim, sx, p);
    T acc = R::coef(coeffs, sc, degree);
    for (int64_t i = degree - 1; i >= 0; --i) acc = R::add(R::mul(acc, z), R::coef(coeffs, sc, i));
    R::st(yre, yim, sy, p, acc);
  }
}

template <int K, int VAR>
struct PolyLaunch {
  static int run(const double* coeffs, int64_t sc, int64_t degree, const double* xre,
                 const double* xim, int64_t sx, double* yre, double* yim, int64_t sy, int64_t npts,
                 int method, int cplx, cudaStream_t st) {
    int levels = 0;
    while (((int64_t)1 << levels) < degree + 1) ++levels;
    if (levels > POLY_LMAX) return MW_ERR_INVALID;
    int64_t blocks = (npts + 127) / 128;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (method == 1) {
      if (cplx)
        estrin_kernel<CplxRing<K, VAR>><<<(unsigned)blocks, 128, 0, st>>>(
            coeffs, sc, degree, levels, xre, xim, sx, yre, yim, sy, npts);
      else
        estrin_kernel<RealRing<K, VAR>><<<(unsigned)blocks, 128, 0, st>>>(
            coeffs, sc, degree, levels, xre, xim, sx, yre, yim, sy, npts);
    } else {
      if (cplx)
        horner_ring_kernel<CplxRing<K, VAR>><<<(unsigned)blocks, 128, 0, st>>>(
            coeffs, sc, degree, xre, xim, sx, yre, yim, sy, npts);
      else
        horner_ring_kernel<RealRing<K, VAR>><<<(unsigned)blocks, 128, 0, st>>>(
            coeffs, sc, degree, xre, xim, sx, yre, yim, sy, npts);
    }
    return launch_status();
  }
};

}  // namespace mw

using namespace mw;

extern "C" int mw_poly_eval(int k, int variant, const double* coeffs, int64_t sc, int64_t degree,
                            const double* xre, const double* xim, int64_t sx, double* yre,
                            double* yim, int64_t sy, int64_t npts, int method, void* stream) {
  if (k < 2 || k > 4) return MW_ERR_INVALID;
  if (variant != 0 && variant != 1) return MW_ERR_INVALID;
  if (method != 0 && method != 1) return MW_ERR_INVALID;
  if (degree < 0 || npts < 0) return MW_ERR_INVALID;
  if (npts == 0) return MW_OK;
  const int cplx = xim != nullptr;
  if (!coeffs || !xre || !yre || (cplx && !yim) || sc < degree + 1 || sx < npts || sy < npts)
    return MW_ERR_INVALID;
  return dispatch<PolyLaunch>(k, variant, coeffs, sc, degree, xre, xim, sx, yre, yim, sy, npts,
                              method, cplx, as_stream(stream));
}
