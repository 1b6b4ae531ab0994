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
#include <atomic>
#include "gemm_kernel.cuh"

namespace mw {

// Tile configurations per K.  Slot 0 is the full-size optimum (tile sweep
// on B200 with tune/gemm_tune.cu + scripts/tune_gemm.py: every
// non-spilling configuration lands within 1-4 % of it; all are
// bit-identical).  Slots 1 and 2 are smaller tiles for row-block shards:
// a GEMM is FP64-pipe bound, so its time follows the busiest SM's share,
// ceil(tiles / SMs) tiles, and at n/8 rows the big tiles leave SMs with one
// tile fewer than others (DD 512 x 4096: 3.46 tiles per SM -> 4).
// gemm_pick() chooses the slot minimising ceil(tiles / SMs) * tile area /
// relative efficiency per variant (measured, scripts/tune_gemm_shards.py
// and scripts/time_gemm_std_tiles.py: DD at 512
// rows 16.55 -> 14.83 ms, TD at 256 rows 6.74 -> 6.15, QD at 512 rows
// 28.96 -> 25.46 ms; full sizes keep slot 0).
template <int bm, int bn, int tm, int tn, int minb>
struct GemmTile {
  static constexpr int BM = bm, BN = bn, BK = 16, TM = tm, TN = tn, MINB = minb;
  static constexpr bool VEC = false;
};
template <int K>
struct GemmCfgs;
template <>
struct GemmCfgs<2> {
  using C0 = GemmTile<64, 64, 4, 4, 2>;
  using C1 = GemmTile<32, 64, 2, 4, 2>;
  using C2 = GemmTile<32, 32, 2, 2, 2>;
  static constexpr double REL[3] = {1.0, 0.979, 0.959};
  static constexpr double REL_STD[3] = {1.0, 0.979, 0.959};  // DD Standard add is branch-free
};
template <>
struct GemmCfgs<3> {
  using C0 = GemmTile<64, 32, 4, 2, 2>;
  using C1 = GemmTile<32, 32, 2, 2, 2>;
  using C2 = GemmTile<32, 16, 2, 1, 4>;
  static constexpr double REL[3] = {1.0, 0.989, 0.963};
  static constexpr double REL_STD[3] = {0.990, 0.987, 1.0};
};
template <>
struct GemmCfgs<4> {
  using C0 = GemmTile<64, 32, 4, 2, 2>;
  using C1 = GemmTile<32, 32, 2, 2, 2>;
  using C2 = GemmTile<32, 16, 2, 1, 4>;
  static constexpr double REL[3] = {1.0, 0.993, 0.980};
  // Standard QD: the renormalisation's divergent branches serialise a
  // thread's MACs, so small register tiles win (n = 2048: 373 / 254 / 234 ms)
  static constexpr double REL_STD[3] = {0.628, 0.924, 1.0};
};
template <int K>
using GemmCfg = typename GemmCfgs<K>::C0;

template <class Cf>
static double gemm_cost(int64_t m, int64_t n, int sms, double rel) {
  const int64_t tiles = ((n + Cf::BN - 1) / Cf::BN) * ((m + Cf::BM - 1) / Cf::BM);
  const int64_t per_sm = (tiles + sms - 1) / sms;
  return (double)per_sm * Cf::BM * Cf::BN / rel;
}

template <int K, int VAR>
static int gemm_pick(int64_t m, int64_t n, int policy) {
  // policy (mw_tuning.gemm_tile): 0 = choose per call, 1..3 = slot 0..2
  if (policy > 0) return policy - 1;
  using Cs = GemmCfgs<K>;
  const int sms = sm_count();
  const double* rel = VAR == BRANCH_FREE ? Cs::REL : Cs::REL_STD;
  const double c0 = gemm_cost<typename Cs::C0>(m, n, sms, rel[0]);
  const double c1 = gemm_cost<typename Cs::C1>(m, n, sms, rel[1]);
  const double c2 = gemm_cost<typename Cs::C2>(m, n, sms, rel[2]);
  return (c1 < c0 && c1 <= c2) ? 1 : (c2 < c0 && c2 < c1) ? 2 : 0;
}

template <int K, int VAR, class Cf>
static int gemm_launch(const double* A, int64_t lda, int64_t sA, const double* B, int64_t ldb,
                       int64_t sB, double* C, int64_t ldc, int64_t sC, int64_t m, int64_t n,
                       int64_t kd, const double* Cin, int64_t ldci, int64_t sCi, int64_t batch,
                       int64_t bsA, int64_t bsB, int64_t bsC, int64_t bsCi, cudaStream_t st) {
  constexpr int NT = (Cf::BM / Cf::TM) * (Cf::BN / Cf::TN);
  const size_t smem = GemmSmem<K, Cf>::BYTES;
  // the dynamic-smem opt-in is per device; setting it twice is harmless
  static std::atomic<bool> attr_set[64];  // lazy per-device init; idempotent, race-free
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

template <int K, int VAR>
struct GemmLaunch {
  static int run(const double* A, int64_t lda, int64_t sA, const double* B, int64_t ldb,
                 int64_t sB, double* C, int64_t ldc, int64_t sC, int64_t m, int64_t n, int64_t kd,
                 const double* Cin, int64_t ldci, int64_t sCi, int64_t batch, int64_t bsA,
                 int64_t bsB, int64_t bsC, int64_t bsCi, int policy, cudaStream_t st) {
    using Cs = GemmCfgs<K>;
    // batched products (the Strassen leaves) keep slot 0
    const int slot = (batch == 1 && Cin == nullptr) ? gemm_pick<K, VAR>(m, n, policy) : 0;
    if (slot == 1)
      return gemm_launch<K, VAR, typename Cs::C1>(A, lda, sA, B, ldb, sB, C, ldc, sC, m, n, kd, Cin,
                                                  ldci, sCi, batch, bsA, bsB, bsC, bsCi, st);
    if (slot == 2)
      return gemm_launch<K, VAR, typename Cs::C2>(A, lda, sA, B, ldb, sB, C, ldc, sC, m, n, kd, Cin,
                                                  ldci, sCi, batch, bsA, bsB, bsC, bsCi, st);
    return gemm_launch<K, VAR, typename Cs::C0>(A, lda, sA, B, ldb, sB, C, ldc, sC, m, n, kd, Cin,
                                                ldci, sCi, batch, bsA, bsB, bsC, bsCi, st);
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
                              sCi, batch, bsA, bsB, bsC, bsCi, 0, as_stream(stream));
}

extern "C" int mw_gemm(int k, int variant, const double* A, int64_t lda, int64_t sA,
                       const double* B, int64_t ldb, int64_t sB, double* C, int64_t ldc,
                       int64_t sC, int64_t m, int64_t n, int64_t kd, void* stream) {
  return mw_gemm_ex(k, variant, A, lda, sA, B, ldb, sB, C, ldc, sC, m, n, kd, nullptr, stream);
}

extern "C" int mw_gemm_ex(int k, int variant, const double* A, int64_t lda, int64_t sA,
                          const double* B, int64_t ldb, int64_t sB, double* C, int64_t ldc,
                          int64_t sC, int64_t m, int64_t n, int64_t kd, const mw_tuning* tune,
                          void* stream) {
  mw_tuning t;
  if (!tuning_resolve(tune, &t)) return MW_ERR_INVALID;
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
                              (int64_t)0, (int64_t)0, (int64_t)0, (int64_t)0, t.gemm_tile,
                              as_stream(stream));
}
