// horner.cu — batched Horner evaluation of one K-word polynomial.
//
// Semantics (poly.horner_eval, poly.py:89-96), per point x:
//   acc = a[deg];  for i = deg-1 .. 0:  acc = add(mul(acc, x), a[i])
// Bit-exact per point.  The reference evaluates one point per call; the
// lane-batched fold over _BATCH_* (batch.py:178-194) is the same sequence
// across lanes.
//
// Design: one point per thread-slot, PPT independent points per thread for
// ILP (the Horner step is one long dependent chain: QD mul+add depth ~60).
// The coefficients are staged through shared memory in chunks of CH words
// (uniform across the CTA: every read is a broadcast), highest chunk first.
// Points are loaded/stored once, coalesced per plane.
//
// TD / QD points that are plain doubles (x = (x0, +0, ...): the usual case,
// and the benchmark's config 4) take td_/qd_mul_bf_d, the branch-free
// product with the operations removed that +0 low words determine (QD 63
// instead of 106 FP64 instructions, TD 30 instead of 39; mw_eft.cuh; the DD
// product has none to remove) -- bit-identical for finite values; a
// CTA in which some such thread ends with a non-finite component (overflow,
// or a NaN / inf in the inputs) re-runs through the full product, so the
// result is the reference's in every case.  The choice is per thread from the
// point's own words: no flag, no pre-pass, nothing stored between calls.
#include "common.cuh"

namespace mw {

constexpr int HORNER_THREADS = 128;
constexpr int HORNER_CH = 256;

template <int K>
struct HornerCfg;
template <> struct HornerCfg<2> { static constexpr int PPT = 2; };
template <> struct HornerCfg<3> { static constexpr int PPT = 2; };
template <> struct HornerCfg<4> { static constexpr int PPT = 2; };

template <int K, int VAR>
__global__ void __launch_bounds__(HORNER_THREADS)
    horner_kernel(const double* __restrict__ coeffs, int64_t sc, int64_t degree,
                  const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                  int64_t npts) {
  constexpr int PPT = HornerCfg<K>::PPT;
  __shared__ double cs[K][HORNER_CH];
  const int64_t base = (int64_t)blockIdx.x * HORNER_THREADS * PPT + threadIdx.x;

  V<K> xv[PPT], acc[PPT];
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int64_t p = base + (int64_t)j * HORNER_THREADS;
    xv[j] = p < npts ? load<K>(x, sx, p) : zero<K>();
    acc[j] = load<K>(coeffs, sc, degree);
  }

  // double-valued points: every low word is +0.0 (bit pattern 0)
  constexpr bool FAST = VAR == BRANCH_FREE && MulByDouble<K>::available;
  bool dbl = false;
  if constexpr (FAST) {
    dbl = true;
#pragma unroll
    for (int j = 0; j < PPT; ++j)
#pragma unroll
      for (int c = 1; c < K; ++c) dbl = dbl && __double_as_longlong(xv[j].c[c]) == 0;
  }

  // coefficients deg-1 .. 0, in chunks [lo, hi) walked downward; pass 1 is
  // the full-product re-run of a CTA in which some double-valued thread saw
  // a non-finite result (never taken on finite data)
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t hi = degree; hi > 0; hi -= HORNER_CH) {
      const int64_t lo = hi > HORNER_CH ? hi - HORNER_CH : 0;
      const int cnt = (int)(hi - lo);
      __syncthreads();
      for (int e = threadIdx.x; e < K * cnt; e += HORNER_THREADS) {
        const int c = e / cnt, i = e % cnt;
        cs[c][i] = coeffs[c * sc + lo + i];
      }
      __syncthreads();
      if constexpr (FAST) {
        if (dbl) {
#pragma unroll 1
          for (int i = cnt - 1; i >= 0; --i) {
            V<K> a;
#pragma unroll
            for (int c = 0; c < K; ++c) a.c[c] = cs[c][i];
#pragma unroll
            for (int j = 0; j < PPT; ++j)
              acc[j] = MulByDouble<K>::add(MulByDouble<K>::mul(acc[j], xv[j].c[0]), a);
          }
          continue;
        }
      }
#pragma unroll 1
      for (int i = cnt - 1; i >= 0; --i) {
        V<K> a;
#pragma unroll
        for (int c = 0; c < K; ++c) a.c[c] = cs[c][i];
#pragma unroll
        for (int j = 0; j < PPT; ++j) acc[j] = Ops<K, VAR>::add(Ops<K, VAR>::mul(acc[j], xv[j]), a);
      }
    }
    bool redo = false;
    if constexpr (FAST) {
      if (pass == 0 && dbl) {
#pragma unroll
        for (int j = 0; j < PPT; ++j)
#pragma unroll
          for (int c = 0; c < K; ++c) redo = redo || !isfinite(acc[j].c[c]);
      }
      redo = __syncthreads_or(redo) != 0;  // uniform: the chunk loop has CTA barriers
    }
    if (!redo) break;
    // every thread of the CTA runs again on the full product (those already
    // on it recompute the same bits)
    dbl = false;
#pragma unroll
    for (int j = 0; j < PPT; ++j) acc[j] = load<K>(coeffs, sc, degree);
  }

#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int64_t p = base + (int64_t)j * HORNER_THREADS;
    if (p < npts) store<K>(y, sy, p, acc[j]);
  }
}

template <int K, int VAR>
struct HornerLaunch {
  static int run(const double* coeffs, int64_t sc, int64_t degree, const double* x, int64_t sx,
                 double* y, int64_t sy, int64_t npts, cudaStream_t st) {
    constexpr int PPT = HornerCfg<K>::PPT;
    const int64_t per_block = (int64_t)HORNER_THREADS * PPT;
    const int64_t blocks = (npts + per_block - 1) / per_block;
    if (blocks > 0x7fffffffLL) return MW_ERR_INVALID;
    horner_kernel<K, VAR><<<(unsigned)blocks, HORNER_THREADS, 0, st>>>(coeffs, sc, degree, x, sx,
                                                                       y, sy, npts);
    return launch_status();
  }
};

}  // namespace mw

using namespace mw;

extern "C" int mw_horner(int k, int variant, const double* coeffs, int64_t sc, int64_t degree,
                         const double* x, int64_t sx, double* y, int64_t sy, int64_t npts,
                         void* stream) {
  if (k < 2 || k > 4) return MW_ERR_INVALID;
  if (variant != 0 && variant != 1) return MW_ERR_INVALID;
  if (degree < 0 || npts < 0) return MW_ERR_INVALID;
  if (npts == 0) return MW_OK;
  if (!coeffs || !x || !y || sc < degree + 1 || sx < npts || sy < npts) return MW_ERR_INVALID;
  return dispatch<HornerLaunch>(k, variant, coeffs, sc, degree, x, sx, y, sy, npts,
                                as_stream(stream));
}
