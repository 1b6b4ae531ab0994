// gemm.cu — C = A B in DD/TD/QD on the FP64 pipe.
//
// Semantics: every C_ij folds t ascending from an exact zero,
//   acc = add(acc, mul(A_it, B_tj)),
// exactly as linalg._rows_kernel_simd / _rows_kernel_scalar
// (linalg.py:284-314, driven by matmul naive, linalg.py:549-569).  The BF
// kernels are bitwise commutative, so this is bit-exact with the reference.
//
// Design (B200, FP64-pipe bound): a CTA computes a BM x BN tile of C with
// (BM/TM) x (BN/TN) threads, each owning a TM x TN register tile
// (rows ty*TM + r, columns tx + q*TX so a warp's B reads are contiguous).
// A and B K-plane tiles of depth BK are staged in shared memory with
// cp.async (8-byte, zero-filled at the matrix edges) in a 2-stage ring so
// the next tile streams in while the current one is consumed.  Arithmetic
// intensity is ~29/96/209 FP64 ops per (2K x 8 B) of smem traffic, so the
// kernel is bound by FP64 issue, not memory; the only overhead on the
// pipe is the exact-zero start (one add per output).
#include "gemm_kernel.cuh"

namespace mw {

template <int K>
struct GemmCfg;
// DD: 64x64 tile, 4x4 per thread, 256 threads.
template <>
struct GemmCfg<2> {
  static constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4, MINB = 2;
  static constexpr bool VEC = false;
};
// TD and QD: 64x32 tile, 4x2 per thread, 256 threads.  (Tile sweep on
// B200 with tune/gemm_tune.cu + scripts/tune_gemm.py: every non-spilling
// configuration lands within 1-3 % of these; all are bit-identical.)
template <>
struct GemmCfg<3> {
  static constexpr int BM = 64, BN = 32, BK = 16, TM = 4, TN = 2, MINB = 2;
  static constexpr bool VEC = false;
};
template <>
struct GemmCfg<4> {
  static constexpr int BM = 64, BN = 32, BK = 16, TM = 4, TN = 2, MINB = 2;
  static constexpr bool VEC = false;
};

template <int K, int VAR>
struct GemmLaunch {
  static int run(const double* A, int64_t lda, int64_t sA, const double* B, int64_t ldb,
                 int64_t sB, double* C, int64_t ldc, int64_t sC, int64_t m, int64_t n, int64_t kd,
                 const double* Cin, int64_t ldci, int64_t sCi, int64_t batch, int64_t bsA,
                 int64_t bsB, int64_t bsC, int64_t bsCi, cudaStream_t st) {
    using Cf = GemmCfg<K>;
    constexpr int NT = (Cf::BM / Cf::TM) * (Cf::BN / Cf::TN);
    const size_t smem = GemmSmem<K, Cf>::BYTES;
    // the dynamic-smem opt-in is per device; setting it twice is harmless
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
      cudaFuncSetAttribute(gemm_kernel<K, VAR, false, Cf>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      cudaFuncSetAttribute(gemm_kernel<K, VAR, true, Cf>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
    const int64_t tiles = ((n + Cf::BN - 1) / Cf::BN) * ((m + Cf::BM - 1) / Cf::BM);
    if (tiles > 0x7fffffffLL) return MW_ERR_INVALID;
    if (batch == 1 && Cin == nullptr) {
      gemm_kernel<K, VAR, false, Cf><<<(unsigned)tiles, NT, smem, st>>>(
          A, lda, sA, B, ldb, sB, C, ldc, sC, m, n, kd, nullptr, 0, 0, 1, 0, 0, 0, 0);
    } else {
      const unsigned gy = (unsigned)(batch < 65535 ? batch : 65535);
      gemm_kernel<K, VAR, true, Cf><<<dim3((unsigned)tiles, gy), NT, smem, st>>>(
          A, lda, sA, B, ldb, sB, C, ldc, sC, m, n, kd, Cin, ldci, sCi, batch, bsA, bsB, bsC, bsCi);
    }
    return launch_status();
  }
};

}  // namespace mw

using namespace mw;

extern "C" int mw_gemm_batched(int k, int variant, const double* A, int64_t lda, int64_t sA,
                               int64_t bsA, const double* B, int64_t ldb, int64_t sB, int64_t bsB,
                               double* C, int64_t ldc, int64_t sC, int64_t bsC, const double* Cin,
                               int64_t ldci, int64_t sCi, int64_t bsCi, int64_t m, int64_t n,
                               int64_t kd, int64_t batch, void* stream) {
  if (k < 2 || k > 4) return MW_ERR_INVALID;
  if (variant != 0 && variant != 1) return MW_ERR_INVALID;
  if (m < 0 || n < 0 || kd < 0 || batch < 0) return MW_ERR_INVALID;
  if (m == 0 || n == 0 || batch == 0) return MW_OK;
  if (!C || ldc < n) return MW_ERR_INVALID;
  if (kd > 0 && (!A || !B || lda < kd || ldb < n)) return MW_ERR_INVALID;
  if (Cin && ldci < n) return MW_ERR_INVALID;
  if (batch > 1 && (bsA < 0 || bsB < 0 || bsC < 0 || (Cin && bsCi < 0))) return MW_ERR_INVALID;
  return dispatch<GemmLaunch>(k, variant, A, lda, sA, B, ldb, sB, C, ldc, sC, m, n, kd, Cin, ldci,
                              sCi, batch, bsA, bsB, bsC, bsCi, as_stream(stream));
}

extern "C" int mw_gemm(int k, int variant, const double* A, int64_t lda, int64_t sA,
                       const double* B, int64_t ldb, int64_t sB, double* C, int64_t ldc,
                       int64_t sC, int64_t m, int64_t n, int64_t kd, void* stream) {
  if (k < 2 || k > 4) return MW_ERR_INVALID;
  if (variant != 0 && variant != 1) return MW_ERR_INVALID;
  if (m < 0 || n < 0 || kd < 0) return MW_ERR_INVALID;
  if (m == 0 || n == 0) return MW_OK;
  if (!C || ldc < n || sC < (m - 1) * ldc + n) return MW_ERR_INVALID;
  if (kd > 0) {
    if (!A || !B || lda < kd || ldb < n) return MW_ERR_INVALID;
    if (sA < (m - 1) * lda + kd || sB < (kd - 1) * ldb + n) return MW_ERR_INVALID;
  }
  return dispatch<GemmLaunch>(k, variant, A, lda, sA, B, ldb, sB, C, ldc, sC, m, n, kd,
                              (const double*)nullptr, (int64_t)0, (int64_t)0, (int64_t)1,
                              (int64_t)0, (int64_t)0, (int64_t)0, (int64_t)0, as_stream(stream));
}
