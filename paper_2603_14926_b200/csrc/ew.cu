// ew.cu — lane-wise K-word kernels: add, sub, mul, div, axpy.
//
// These replace the numpy lane loop behind batch.batch_add / batch_mul /
// batch_div (batch.py:204-231) and the axpy built from them.  Each lane
// runs the reference op sequence, so results are bit-exact.  HBM-bound:
// a lane moves (2 or 1 inputs + 1 output) x K x 8 bytes.  When every plane
// base is 16-byte aligned and every plane stride even, a thread handles two
// adjacent lanes with 128-bit loads/stores per plane; otherwise one lane
// with 64-bit accesses.
#include "common.cuh"

namespace mw {

enum EwOp : int { EW_ADD = 0, EW_SUB = 1, EW_MUL = 2, EW_DIV = 3, EW_AXPY = 4 };

template <int K, int VAR, int OP>
__device__ __forceinline__ V<K> ew_apply(const V<K>& a, const V<K>& b) {
  if (OP == EW_ADD) return Ops<K, VAR>::add(a, b);
  if (OP == EW_SUB) return Ops<K, VAR>::add(a, neg(b));
  if (OP == EW_MUL) return Ops<K, VAR>::mul(a, b);
  if (OP == EW_DIV) return div_newton<K, VAR>(a, b);
  // EW_AXPY: a = x lane, b = y lane; batch_mul(alpha, x) then batch_add(., y)
  return a;
}

template <int K, int VAR, int OP>
__global__ void __launch_bounds__(256) ew_kernel_v2(const double* a, int64_t sa,
                                                    const double* b, int64_t sb,
                                                    double* out, int64_t so,
                                                    int64_t npairs, V<K> alpha) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs;
       p += (int64_t)gridDim.x * blockDim.x) {
    V<K> a0, a1, b0, b1;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      double2 va = reinterpret_cast<const double2*>(a + c * sa)[p];
      double2 vb = reinterpret_cast<const double2*>(b + c * sb)[p];
      a0.c[c] = va.x;
      a1.c[c] = va.y;
      b0.c[c] = vb.x;
      b1.c[c] = vb.y;
    }
    V<K> r0, r1;
    if (OP == EW_AXPY) {
      r0 = Ops<K, VAR>::add(Ops<K, VAR>::mul(alpha, a0), b0);
      r1 = Ops<K, VAR>::add(Ops<K, VAR>::mul(alpha, a1), b1);
    } else {
      r0 = ew_apply<K, VAR, OP>(a0, b0);
      r1 = ew_apply<K, VAR, OP>(a1, b1);
    }
#pragma unroll
    for (int c = 0; c < K; ++c)
      reinterpret_cast<double2*>(out + c * so)[p] = make_double2(r0.c[c], r1.c[c]);
  }
}

template <int K, int VAR, int OP>
__global__ void __launch_bounds__(256) ew_kernel_v1(const double* a, int64_t sa,
                                                    const double* b, int64_t sb,
                                                    double* out, int64_t so,
                                                    int64_t n, V<K> alpha) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    V<K> x = load<K>(a, sa, i);
    V<K> y = load<K>(b, sb, i);
    V<K> r = (OP == EW_AXPY) ? Ops<K, VAR>::add(Ops<K, VAR>::mul(alpha, x), y)
                             : ew_apply<K, VAR, OP>(x, y);
    store<K>(out, so, i, r);
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <int K, int VAR, int OP>
struct EwLaunch {
  static int run(const double* a, int64_t sa, const double* b, int64_t sb, double* out,
                 int64_t so, int64_t n, const double* alpha_host, cudaStream_t st) {
    V<K> alpha = zero<K>();
    if (OP == EW_AXPY)
      for (int c = 0; c < K; ++c) alpha.c[c] = alpha_host[c];
    const int threads = 256;
    const int64_t max_blocks = (int64_t)sm_count() * 16;
    bool vec = (n % 2 == 0) && aligned16(a) && aligned16(b) && aligned16(out) &&
               (sa % 2 == 0) && (sb % 2 == 0) && (so % 2 == 0);
    // the second lane of a pair must not alias across planes for in-place
    // ops; in-place (out == a or b) is fine because each thread reads its
    // lanes before writing them.
    if (vec) {
      int64_t np = n / 2;
      int64_t blocks = (np + threads - 1) / threads;
      if (blocks > max_blocks) blocks = max_blocks;
      ew_kernel_v2<K, VAR, OP><<<(unsigned)blocks, threads, 0, st>>>(a, sa, b, sb, out, so, np,
                                                                     alpha);
    } else {
      int64_t blocks = (n + threads - 1) / threads;
      if (blocks > max_blocks) blocks = max_blocks;
      ew_kernel_v1<K, VAR, OP><<<(unsigned)blocks, threads, 0, st>>>(a, sa, b, sb, out, so, n,
                                                                     alpha);
    }
    return launch_status();
  }
};

template <int K, int VAR> struct EwAdd : EwLaunch<K, VAR, EW_ADD> {};
template <int K, int VAR> struct EwSub : EwLaunch<K, VAR, EW_SUB> {};
template <int K, int VAR> struct EwMul : EwLaunch<K, VAR, EW_MUL> {};
template <int K, int VAR> struct EwDiv : EwLaunch<K, VAR, EW_DIV> {};
template <int K, int VAR> struct EwAxpy : EwLaunch<K, VAR, EW_AXPY> {};

static int ew_check(int k, const void* a, int64_t sa, const void* b, int64_t sb,
                    const void* out, int64_t so, int64_t n) {
  if (k < 2 || k > 4 || n < 0) return MW_ERR_INVALID;
  if (n == 0) return MW_OK;
  if (!a || !b || !out) return MW_ERR_INVALID;
  if (sa < n || sb < n || so < n) return MW_ERR_INVALID;
  return 1;  // proceed
}

}  // namespace mw

using namespace mw;

#define MW_EW_ENTRY(NAME, FUNCTOR)                                                         \
  extern "C" int NAME(int k, int variant, const double* a, int64_t sa, const double* b,   \
                      int64_t sb, double* out, int64_t so, int64_t n, void* stream) {     \
    int chk = ew_check(k, a, sa, b, sb, out, so, n);                                       \
    if (chk <= 0) {                                                                        \
      if (chk == MW_OK) return (variant == 0 || variant == 1) ? MW_OK : MW_ERR_INVALID;    \
      return chk;                                                                          \
    }                                                                                      \
    return dispatch<FUNCTOR>(k, variant, a, sa, b, sb, out, so, n, (const double*)nullptr, \
                             as_stream(stream));                                           \
  }

MW_EW_ENTRY(mw_ew_add, EwAdd)
MW_EW_ENTRY(mw_ew_sub, EwSub)
MW_EW_ENTRY(mw_ew_mul, EwMul)
MW_EW_ENTRY(mw_ew_div, EwDiv)

extern "C" int mw_axpy(int k, int variant, const double* alpha_host, const double* x,
                       int64_t sx, double* y, int64_t sy, int64_t n, void* stream) {
  int chk = ew_check(k, x, sx, y, sy, y, sy, n);
  if (chk <= 0) {
    if (chk == MW_OK) return (variant == 0 || variant == 1) ? MW_OK : MW_ERR_INVALID;
    return chk;
  }
  if (!alpha_host) return MW_ERR_INVALID;
  return dispatch<EwAxpy>(k, variant, x, sx, (const double*)y, sy, y, sy, n, alpha_host,
                          as_stream(stream));
}

// ------------------------------------------------------------- raw EFTs
// The error-free transformations themselves over arrays (eft.py:51-83):
// op 0 quick_two_sum, 1 two_sum, 2 two_prod; (s, e) per element.
namespace mw {
template <int OP>
__global__ void __launch_bounds__(256) eft_kernel(const double* __restrict__ a,
                                                  const double* __restrict__ b,
                                                  double* __restrict__ s, double* __restrict__ e,
                                                  int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double ss, ee;
    if (OP == 0) quick_two_sum(a[i], b[i], ss, ee);
    if (OP == 1) two_sum(a[i], b[i], ss, ee);
    if (OP == 2) two_prod(a[i], b[i], ss, ee);
    s[i] = ss;
    e[i] = ee;
  }
}
}  // namespace mw

extern "C" int mw_eft(int op, const double* a, const double* b, double* s, double* e, int64_t n,
                      void* stream) {
  if (op < 0 || op > 2 || n < 0) return MW_ERR_INVALID;
  if (n == 0) return MW_OK;
  if (!a || !b || !s || !e) return MW_ERR_INVALID;
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 16;
  if (blocks > cap) blocks = cap;
  cudaStream_t st = as_stream(stream);
  if (op == 0) eft_kernel<0><<<(unsigned)blocks, 256, 0, st>>>(a, b, s, e, n);
  if (op == 1) eft_kernel<1><<<(unsigned)blocks, 256, 0, st>>>(a, b, s, e, n);
  if (op == 2) eft_kernel<2><<<(unsigned)blocks, 256, 0, st>>>(a, b, s, e, n);
  return launch_status();
}

// ------------------------------------------- kernels outside the dispatch
// The reference's named kernels that no (K, Variant) entry selects
// (multiword.py:104-115 dw_add_sloppy, 325-358 tw_mul_cleaned), the
// renormalisers (191-241 tw_/qw_renormalize, 710-719 normalize) and the
// correctly rounded fma (eft.py:33-48), over component planes.
namespace mw {
template <int OP>
__global__ void __launch_bounds__(256) named_kernel(const double* __restrict__ a, int64_t sa,
                                                    const double* __restrict__ b, int64_t sb,
                                                    double* __restrict__ out, int64_t so,
                                                    int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (OP == MW_NAMED_DW_ADD_SLOPPY) {
      store<2>(out, so, i, dd_add_sloppy(load<2>(a, sa, i), load<2>(b, sb, i)));
    } else {
      store<3>(out, so, i, tw_mul_cleaned(load<3>(a, sa, i), load<3>(b, sb, i)));
    }
  }
}

// in: M = 2 / 4 / 5 planes (K = 2: quick_two_sum(c0, c1); K = 3:
// tw_renormalize(s0, s1, s2, t0); K = 4: qw_renormalize(x0..x4)) -> K planes
template <int K>
__global__ void __launch_bounds__(256) renorm_kernel(const double* __restrict__ in, int64_t si,
                                                     double* __restrict__ out, int64_t so,
                                                     int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    V<K> r;
    if constexpr (K == 2) {
      quick_two_sum(in[i], in[si + i], r.c[0], r.c[1]);
    } else if constexpr (K == 3) {
      r = tw_renormalize(in[i], in[si + i], in[2 * si + i], in[3 * si + i]);
    } else {
      r = qw_renormalize(in[i], in[si + i], in[2 * si + i], in[3 * si + i], in[4 * si + i]);
    }
    store<K>(out, so, i, r);
  }
}

__global__ void __launch_bounds__(256) fma_kernel(const double* __restrict__ a,
                                                  const double* __restrict__ b,
                                                  const double* __restrict__ c,
                                                  double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = MW_FMA(a[i], b[i], c[i]);
}

static unsigned lane_blocks(int64_t n) {
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 16;
  return (unsigned)(blocks > cap ? cap : blocks);
}
}  // namespace mw

extern "C" int mw_named_op(int op, const double* a, int64_t sa, const double* b, int64_t sb,
                           double* out, int64_t so, int64_t n, void* stream) {
  if (op != MW_NAMED_DW_ADD_SLOPPY && op != MW_NAMED_TW_MUL_CLEANED) return MW_ERR_INVALID;
  if (n < 0) return MW_ERR_INVALID;
  if (n == 0) return MW_OK;
  if (!a || !b || !out || sa < n || sb < n || so < n) return MW_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  if (op == MW_NAMED_DW_ADD_SLOPPY)
    named_kernel<MW_NAMED_DW_ADD_SLOPPY><<<lane_blocks(n), 256, 0, st>>>(a, sa, b, sb, out, so, n);
  else
    named_kernel<MW_NAMED_TW_MUL_CLEANED><<<lane_blocks(n), 256, 0, st>>>(a, sa, b, sb, out, so, n);
  return launch_status();
}

extern "C" int mw_renormalize(int k, const double* in, int64_t si, double* out, int64_t so,
                              int64_t n, void* stream) {
  if (k < 2 || k > 4 || n < 0) return MW_ERR_INVALID;
  if (n == 0) return MW_OK;
  if (!in || !out || si < n || so < n) return MW_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  if (k == 2) renorm_kernel<2><<<lane_blocks(n), 256, 0, st>>>(in, si, out, so, n);
  if (k == 3) renorm_kernel<3><<<lane_blocks(n), 256, 0, st>>>(in, si, out, so, n);
  if (k == 4) renorm_kernel<4><<<lane_blocks(n), 256, 0, st>>>(in, si, out, so, n);
  return launch_status();
}

extern "C" int mw_fma(const double* a, const double* b, const double* c, double* out, int64_t n,
                      void* stream) {
  if (n < 0) return MW_ERR_INVALID;
  if (n == 0) return MW_OK;
  if (!a || !b || !c || !out) return MW_ERR_INVALID;
  fma_kernel<<<lane_blocks(n), 256, 0, as_stream(stream)>>>(a, b, c, out, n);
  return launch_status();
}
