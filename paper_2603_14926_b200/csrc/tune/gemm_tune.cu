// gemm_tune.cu — tuning harness (NOT part of the product library): the
// product GEMM kernel template instantiated with alternative tile
// configurations, so scripts/tune_gemm.py can time them on a B200 and
// check their output is bit-identical to the product kernel.
#include "../gemm_kernel.cuh"
#include "../reduce.cu"  // GEMV kernel template (its C-ABI symbols stay private to this .so)
#include "gemv_forms.cuh"
#include "gemv_staged.cuh"
#include "gemv_bulk.cuh"
#include "gemv_probe.cuh"
#include "gemv_wring.cuh"
#include "gemv_pin.cuh"

namespace mw {
#define CFGV(NAME, bm, bn, bk, tm, tn, minb, vec)                             \
  struct NAME {                                                               \
    static constexpr int BM = bm, BN = bn, BK = bk, TM = tm, TN = tn, MINB = minb; \
    static constexpr bool VEC = vec;                                          \
  };
#define CFG(NAME, bm, bn, bk, tm, tn, minb) CFGV(NAME, bm, bn, bk, tm, tn, minb, false)
CFG(C64x64_44_2, 64, 64, 16, 4, 4, 2)
CFG(C64x32_42_3, 64, 32, 16, 4, 2, 3)
CFG(C32x64_24_3, 32, 64, 16, 2, 4, 3)
CFG(C64x64_44_2_bk8, 64, 64, 8, 4, 4, 2)
CFG(C32x64_24_2, 32, 64, 16, 2, 4, 2)
CFG(C32x32_22_3, 32, 32, 16, 2, 2, 3)
CFG(C64x32_42_2, 64, 32, 16, 4, 2, 2)
CFG(C32x32_22_2, 32, 32, 16, 2, 2, 2)
CFG(C16x32_12_4, 16, 32, 16, 1, 2, 4)
CFG(C32x16_21_4, 32, 16, 16, 2, 1, 4)
CFG(C32x32_22_2_bk32, 32, 32, 32, 2, 2, 2)
CFG(C32x64_24_1, 32, 64, 16, 2, 4, 1)
CFGV(V64x64_44_2, 64, 64, 16, 4, 4, 2, true)
CFGV(V64x32_42_2, 64, 32, 16, 4, 2, 2, true)
CFGV(V32x32_22_2, 32, 32, 16, 2, 2, 2, true)
CFGV(V64x64_44_2_bk8, 64, 64, 8, 4, 4, 2, true)

static int64_t g_rows = 0;  // 0: square; else rows of A / C (row-block shard)
template <int K, class Cf>
static int launch(const double* A, const double* B, double* C, int64_t n, cudaStream_t st) {
  constexpr int NT = (Cf::BM / Cf::TM) * (Cf::BN / Cf::TN);
  const size_t smem = GemmSmem<K, Cf>::BYTES;
  cudaFuncSetAttribute(gemm_kernel<K, BRANCH_FREE, false, Cf>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t m = g_rows ? g_rows : n;
  const int64_t tiles = ((n + Cf::BN - 1) / Cf::BN) * ((m + Cf::BM - 1) / Cf::BM);
  gemm_kernel<K, BRANCH_FREE, false, Cf><<<(unsigned)tiles, NT, smem, st>>>(
      A, n, m * n, B, n, n * n, C, n, m * n, m, n, n, nullptr, 0, 0, 1, 0, 0, 0, 0);
  return launch_status();
}

template <int K>
static int run(int cfg, const double* A, const double* B, double* C, int64_t n, cudaStream_t st) {
  switch (cfg) {
    case 0: return launch<K, C64x64_44_2>(A, B, C, n, st);
    case 1: return launch<K, C64x32_42_3>(A, B, C, n, st);
    case 2: return launch<K, C32x64_24_3>(A, B, C, n, st);
    case 3: return launch<K, C64x64_44_2_bk8>(A, B, C, n, st);
    case 4: return launch<K, C32x64_24_2>(A, B, C, n, st);
    case 5: return launch<K, C32x32_22_3>(A, B, C, n, st);
    case 6: return launch<K, C64x32_42_2>(A, B, C, n, st);
    case 7: return launch<K, C32x32_22_2>(A, B, C, n, st);
    case 8: return launch<K, C16x32_12_4>(A, B, C, n, st);
    case 9: return launch<K, C32x16_21_4>(A, B, C, n, st);
    case 10: return launch<K, C32x32_22_2_bk32>(A, B, C, n, st);
    case 11: return launch<K, C32x64_24_1>(A, B, C, n, st);
    case 12: return launch<K, V64x64_44_2>(A, B, C, n, st);
    case 13: return launch<K, V64x32_42_2>(A, B, C, n, st);
    case 14: return launch<K, V32x32_22_2>(A, B, C, n, st);
    case 15: return launch<K, V64x64_44_2_bk8>(A, B, C, n, st);
    default: return MW_ERR_INVALID;
  }
}

int sm_count() { return 148; }
}  // namespace mw

using namespace mw;

extern "C" int mwt_num_configs(void) { return 16; }
extern "C" const char* mwt_config_name(int cfg) {
  static const char* names[] = {"64x64_44_2", "64x32_42_3", "32x64_24_3", "64x64_44_2_bk8",
                                "32x64_24_2", "32x32_22_3", "64x32_42_2", "32x32_22_2",
                                "16x32_12_4", "32x16_21_4", "32x32_22_2_bk32", "32x64_24_1",
                                "V64x64_44_2", "V64x32_42_2", "V32x32_22_2", "V64x64_44_2_bk8"};
  return (cfg >= 0 && cfg < 16) ? names[cfg] : "?";
}
extern "C" void mwt_gemm_set_rows(int64_t rows) { g_rows = rows; }
extern "C" int mwt_gemm(int cfg, int k, const double* A, const double* B, double* C, int64_t n,
                        void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (k == 2) return run<2>(cfg, A, B, C, n, st);
  if (k == 3) return run<3>(cfg, A, B, C, n, st);
  if (k == 4) return run<4>(cfg, A, B, C, n, st);
  return MW_ERR_INVALID;
}

// ---- GEMV variants: (warps per row, rows per CTA, loads ahead)
// plane stride of A (elements): m * n unless set (padding experiments)
static int64_t g_gemv_sa = 0;
static inline int64_t gemv_sa(int64_t m, int64_t n) { return g_gemv_sa > 0 ? g_gemv_sa : m * n; }
// row stride override (0 = n; -1 = every row reads row 0: A stays L2-resident)
static int64_t g_gemv_lda = 0;
static inline int64_t gemv_lda(int64_t n) { return g_gemv_lda == 0 ? n : (g_gemv_lda < 0 ? 0 : g_gemv_lda); }
extern "C" void mwt_gemv_set_lda(int64_t v) { g_gemv_lda = v; }
extern "C" void mwt_gemv_set_sa(int64_t sa) { g_gemv_sa = sa; }
template <int K, int W, int R, int D>
static int gemv_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                       cudaStream_t st) {
  gemv_tree_kernel<K, BRANCH_FREE, W, R, D><<<(unsigned)((m + R - 1) / R), 32 * W * R, 0, st>>>(
      A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int SLOTS, int D, bool PERSIST, bool XPF = true, int MINB = 1>
static int gemv_ptree_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                             cudaStream_t st) {
  auto kern = gemv_ptree_kernel<K, BRANCH_FREE, SLOTS, D, XPF, MINB>;
  int64_t grid = (m + SLOTS - 1) / SLOTS;
  if (PERSIST) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128 * SLOTS, 0);
    const int64_t slots = (int64_t)148 * per_sm * SLOTS;
    const int64_t rows_per_slot = (m + slots - 1) / slots;
    grid = (m + rows_per_slot * SLOTS - 1) / (rows_per_slot * SLOTS);
  }
  kern<<<(unsigned)grid, 128 * SLOTS, 0, st>>>(A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int D, int S>
static int gemv_cg_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                          cudaStream_t st) {
  if (n % (128 * D)) return MW_ERR_INVALID;
  auto kern = gemv_cg_kernel<K, BRANCH_FREE, D, S>;
  const int smem = 4 * S * K * D * 32 * (int)sizeof(double);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<(unsigned)m, 128, smem, st>>>(A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int D, int RPC>
static int gemv_u2_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                          cudaStream_t st) {
  gemv_u2_kernel<K, BRANCH_FREE, D, RPC><<<(unsigned)((m + RPC - 1) / RPC), 64 * RPC, 0, st>>>(
      A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int D, int WPC>
static int gemv_w1_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                          cudaStream_t st) {
  gemv_w1_kernel<K, BRANCH_FREE, D, WPC><<<(unsigned)((m + WPC - 1) / WPC), 32 * WPC, 0, st>>>(
      A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int D, int MINB, int CPS>
static int gemv_dyn_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                           cudaStream_t st) {
  static unsigned int* ctr = nullptr;
  if (!ctr) {
    cudaMalloc(&ctr, 2 * sizeof(unsigned int));
    cudaMemset(ctr, 0, 2 * sizeof(unsigned int));
    cudaDeviceSynchronize();
  }
  auto kern = gemv_dyn_kernel<K, BRANCH_FREE, D, MINB>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, 0);
  if (CPS > 0 && CPS < per_sm) per_sm = CPS;
  int64_t grid = (int64_t)148 * per_sm;
  if (grid > m) grid = m;
  kern<<<(unsigned)grid, 128, 0, st>>>(A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n, ctr);
  return launch_status();
}
template <int K, int R, int D, int S, bool XS>
static int gemv_staged_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                              cudaStream_t st) {
  constexpr size_t smem = gemv_staged_smem<K, R, D, S, XS>();
  auto kern = gemv_staged_kernel<K, BRANCH_FREE, R, D, S, XS>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<(unsigned)((m + R - 1) / R), 128 * R, smem, st>>>(A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int G, int CH, int S>
static int gemv_bulk_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                            cudaStream_t st) {
  const size_t smem = gemv_bulk_smem<K, G, CH, S>(n);
  if (smem > 227 * 1024) return MW_ERR_INVALID;
  auto kern = gemv_bulk_kernel<K, BRANCH_FREE, G, CH, S>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = sm_count();
  if ((int64_t)grid * G > m) grid = (int)((m + G - 1) / G);
  kern<<<grid, 128 * G, smem, st>>>(A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int MODE>
static int gemv_probe_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                             cudaStream_t st) {
  gemv_probe_kernel<K, BRANCH_FREE, MODE><<<(unsigned)((m + 1) / 2), 256, 0, st>>>(A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int RT, int D, bool PIPE, int MINB = 1>
static int gemv_rt_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                          cudaStream_t st) {
  gemv_rt_kernel<K, BRANCH_FREE, RT, D, PIPE, MINB><<<(unsigned)((m + RT - 1) / RT), 128, 0, st>>>(
      A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int Q, int J, int S>
static int gemv_wring_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                             cudaStream_t st) {
  if (n % (128 * J)) return MW_ERR_INVALID;
  const size_t smem = gemv_wring_smem<K, Q, J, S>();
  if (smem > 227 * 1024) return MW_ERR_INVALID;
  auto kern = gemv_wring_kernel<K, BRANCH_FREE, Q, J, S>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = sm_count();
  if ((int64_t)grid * Q > m) grid = (int)((m + Q - 1) / Q);
  kern<<<grid, 128 * Q, smem, st>>>(A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int C, int D, int RPC>
static int gemv_mc_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                          cudaStream_t st) {
  gemv_mc_kernel<K, BRANCH_FREE, C, D, RPC><<<(unsigned)((m + RPC - 1) / RPC), 128 * RPC, 0, st>>>(
      A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int D, int RPC>
static int gemv_v2_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                          cudaStream_t st) {
  if (n % 256) return MW_ERR_INVALID;
  gemv_v2_kernel<K, BRANCH_FREE, D, RPC><<<(unsigned)((m + RPC - 1) / RPC), 128 * RPC, 0, st>>>(
      A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int RPC, int D, int CPS>
static int gemv_xs_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                          cudaStream_t st) {
  const size_t smem = ((size_t)K * n + (size_t)RPC * K * 128) * sizeof(double);
  if (smem > 227 * 1024 / CPS) return MW_ERR_INVALID;
  auto kern = gemv_xs_kernel<K, BRANCH_FREE, RPC, D>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t grid = (int64_t)148 * CPS;
  const int64_t need = (m + RPC - 1) / RPC;
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, 128 * RPC, smem, st>>>(A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int RPC, int D>
static int gemv_cs_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                          cudaStream_t st) {
  gemv_cs_kernel<K, BRANCH_FREE, RPC, D><<<(unsigned)((m + RPC - 1) / RPC), 128 * RPC, 0, st>>>(
      A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K, int RPC, int D, int PIN, int MINB = 1>
static int gemv_pin_launch(const double* A, const double* x, double* y, int64_t m, int64_t n,
                           cudaStream_t st) {
  gemv_pin_kernel<K, BRANCH_FREE, RPC, D, PIN, MINB>
      <<<(unsigned)((m + RPC - 1) / RPC), 128 * RPC, 0, st>>>(A, gemv_lda(n), gemv_sa(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K>
static int gemv_run(int cfg, const double* A, const double* x, double* y, int64_t m, int64_t n,
                    cudaStream_t st) {
  switch (cfg) {
    case 0: return gemv_launch<K, 4, 2, 4>(A, x, y, m, n, st);
    case 1: return gemv_launch<K, 1, 8, 8>(A, x, y, m, n, st);
    case 2: return gemv_launch<K, 1, 8, 4>(A, x, y, m, n, st);
    case 3: return gemv_launch<K, 2, 4, 4>(A, x, y, m, n, st);
    case 4: return gemv_launch<K, 2, 4, 8>(A, x, y, m, n, st);
    case 5: return gemv_launch<K, 4, 2, 2>(A, x, y, m, n, st);
    case 6: return gemv_launch<K, 4, 1, 4>(A, x, y, m, n, st);
    case 7: return gemv_launch<K, 8, 1, 2>(A, x, y, m, n, st);
    case 8: return gemv_staged_launch<K, 2, 4, 2, false>(A, x, y, m, n, st);
    case 9: return gemv_staged_launch<K, 2, 4, 3, false>(A, x, y, m, n, st);
    case 10: return gemv_staged_launch<K, 1, 4, 2, false>(A, x, y, m, n, st);
    case 11: return gemv_staged_launch<K, 1, 4, 3, false>(A, x, y, m, n, st);
    case 12: return gemv_staged_launch<K, 2, 2, 2, false>(A, x, y, m, n, st);
    case 13: return gemv_staged_launch<K, 2, 2, 4, false>(A, x, y, m, n, st);
    case 14: return gemv_staged_launch<K, 1, 4, 2, true>(A, x, y, m, n, st);
    case 15: return gemv_staged_launch<K, 2, 4, 2, true>(A, x, y, m, n, st);
    case 16: return gemv_staged_launch<K, 1, 8, 2, false>(A, x, y, m, n, st);
    case 17: return gemv_staged_launch<K, 1, 2, 4, false>(A, x, y, m, n, st);
    case 18: return gemv_bulk_launch<K, 8, 256, 2>(A, x, y, m, n, st);
    case 19: return gemv_bulk_launch<K, 6, 256, 3>(A, x, y, m, n, st);
    case 20: return gemv_bulk_launch<K, 4, 512, 2>(A, x, y, m, n, st);
    case 21: return gemv_bulk_launch<K, 8, 128, 3>(A, x, y, m, n, st);
    case 22: return gemv_bulk_launch<K, 6, 256, 2>(A, x, y, m, n, st);
    case 23: return gemv_bulk_launch<K, 4, 256, 3>(A, x, y, m, n, st);
    case 24: return gemv_bulk_launch<K, 5, 256, 2>(A, x, y, m, n, st);
    case 25: return gemv_bulk_launch<K, 7, 128, 4>(A, x, y, m, n, st);
    case 26: return gemv_probe_launch<K, 1>(A, x, y, m, n, st);
    case 27: return gemv_probe_launch<K, 2>(A, x, y, m, n, st);
    case 28: return gemv_rt_launch<K, 1, 4, false>(A, x, y, m, n, st);
    case 29: return gemv_rt_launch<K, 1, 2, true>(A, x, y, m, n, st);
    case 30: return gemv_rt_launch<K, 1, 4, true>(A, x, y, m, n, st);
    case 31: return gemv_rt_launch<K, 2, 2, false>(A, x, y, m, n, st);
    case 32: return gemv_rt_launch<K, 2, 4, false>(A, x, y, m, n, st);
    case 33: return gemv_rt_launch<K, 2, 2, true>(A, x, y, m, n, st);
    case 34: return gemv_rt_launch<K, 2, 1, true>(A, x, y, m, n, st);
    case 35: return gemv_rt_launch<K, 1, 2, true, 8>(A, x, y, m, n, st);
    case 36: return gemv_rt_launch<K, 2, 2, true, 4>(A, x, y, m, n, st);
    case 37: return gemv_rt_launch<K, 1, 1, true, 12>(A, x, y, m, n, st);
    case 38: return gemv_wring_launch<K, 8, 2, 4>(A, x, y, m, n, st);
    case 39: return gemv_wring_launch<K, 8, 2, 3>(A, x, y, m, n, st);
    case 40: return gemv_wring_launch<K, 6, 2, 4>(A, x, y, m, n, st);
    case 41: return gemv_wring_launch<K, 6, 4, 2>(A, x, y, m, n, st);
    case 42: return gemv_wring_launch<K, 4, 4, 3>(A, x, y, m, n, st);
    case 43: return gemv_wring_launch<K, 8, 1, 6>(A, x, y, m, n, st);
    case 44: return gemv_wring_launch<K, 6, 2, 3>(A, x, y, m, n, st);
    case 45: return gemv_mc_launch<K, 2, 2, 1>(A, x, y, m, n, st);
    case 46: return gemv_mc_launch<K, 2, 1, 1>(A, x, y, m, n, st);
    case 47: return gemv_mc_launch<K, 2, 2, 2>(A, x, y, m, n, st);
    case 48: return gemv_mc_launch<K, 2, 1, 2>(A, x, y, m, n, st);
    case 49: return gemv_mc_launch<K, 1, 4, 1>(A, x, y, m, n, st);
    case 50: return gemv_mc_launch<K, 4, 1, 1>(A, x, y, m, n, st);
    case 51: return gemv_v2_launch<K, 2, 2>(A, x, y, m, n, st);
    case 52: return gemv_v2_launch<K, 2, 1>(A, x, y, m, n, st);
    case 53: return gemv_v2_launch<K, 1, 2>(A, x, y, m, n, st);
    case 54: return gemv_v2_launch<K, 4, 1>(A, x, y, m, n, st);
    case 55: return gemv_xs_launch<K, 8, 4, 1>(A, x, y, m, n, st);
    case 56: return gemv_xs_launch<K, 6, 4, 1>(A, x, y, m, n, st);
    case 57: return gemv_xs_launch<K, 4, 4, 2>(A, x, y, m, n, st);
    case 58: return gemv_xs_launch<K, 8, 2, 1>(A, x, y, m, n, st);
    case 59: return gemv_cs_launch<K, 2, 4>(A, x, y, m, n, st);
    case 60: return gemv_cs_launch<K, 1, 4>(A, x, y, m, n, st);
    case 61: return gemv_ptree_launch<K, 1, 4, true>(A, x, y, m, n, st);
    case 62: return gemv_ptree_launch<K, 2, 4, true>(A, x, y, m, n, st);
    case 63: return gemv_ptree_launch<K, 1, 2, true>(A, x, y, m, n, st);
    case 64: return gemv_ptree_launch<K, 2, 2, true>(A, x, y, m, n, st);
    case 65: return gemv_ptree_launch<K, 4, 4, true>(A, x, y, m, n, st);
    case 66: return gemv_ptree_launch<K, 1, 8, true>(A, x, y, m, n, st);
    case 67: return gemv_ptree_launch<K, 1, 4, false>(A, x, y, m, n, st);
    case 68: return gemv_ptree_launch<K, 2, 4, false>(A, x, y, m, n, st);
    case 69: return gemv_ptree_launch<K, 2, 8, true>(A, x, y, m, n, st);
    case 70: return gemv_ptree_launch<K, 1, 4, true, false, 1>(A, x, y, m, n, st);
    case 71: return gemv_ptree_launch<K, 2, 4, true, false, 1>(A, x, y, m, n, st);
    case 72: return gemv_ptree_launch<K, 1, 4, true, false, 8>(A, x, y, m, n, st);
    case 73: return gemv_ptree_launch<K, 2, 4, true, false, 4>(A, x, y, m, n, st);
    case 74: return gemv_ptree_launch<K, 1, 4, false, false, 1>(A, x, y, m, n, st);
    case 75: return gemv_ptree_launch<K, 2, 4, false, false, 1>(A, x, y, m, n, st);
    case 76: return gemv_ptree_launch<K, 1, 4, false, false, 8>(A, x, y, m, n, st);
    case 77: return gemv_ptree_launch<K, 2, 4, false, false, 4>(A, x, y, m, n, st);
    case 78: return gemv_ptree_launch<K, 1, 2, false, false, 8>(A, x, y, m, n, st);
    case 79: return gemv_ptree_launch<K, 1, 2, true, false, 8>(A, x, y, m, n, st);
    case 80: return gemv_cg_launch<K, 4, 3>(A, x, y, m, n, st);
    case 81: return gemv_cg_launch<K, 4, 4>(A, x, y, m, n, st);
    case 82: return gemv_cg_launch<K, 2, 4>(A, x, y, m, n, st);
    case 83: return gemv_cg_launch<K, 2, 6>(A, x, y, m, n, st);
    case 84: return gemv_cg_launch<K, 2, 3>(A, x, y, m, n, st);
    case 85: return gemv_cg_launch<K, 1, 8>(A, x, y, m, n, st);
    case 86: return gemv_cg_launch<K, 4, 2>(A, x, y, m, n, st);
    case 87: return gemv_cg_launch<K, 8, 2>(A, x, y, m, n, st);
    case 88: return gemv_u2_launch<K, 2, 1>(A, x, y, m, n, st);
    case 89: return gemv_u2_launch<K, 2, 2>(A, x, y, m, n, st);
    case 90: return gemv_u2_launch<K, 4, 1>(A, x, y, m, n, st);
    case 91: return gemv_u2_launch<K, 4, 2>(A, x, y, m, n, st);
    case 92: return gemv_u2_launch<K, 1, 2>(A, x, y, m, n, st);
    case 93: return gemv_u2_launch<K, 2, 4>(A, x, y, m, n, st);
    case 94: return gemv_w1_launch<K, 1, 1>(A, x, y, m, n, st);
    case 95: return gemv_w1_launch<K, 2, 1>(A, x, y, m, n, st);
    case 96: return gemv_w1_launch<K, 1, 2>(A, x, y, m, n, st);
    case 97: return gemv_w1_launch<K, 2, 2>(A, x, y, m, n, st);
    case 98: return gemv_w1_launch<K, 1, 4>(A, x, y, m, n, st);
    case 99: return gemv_w1_launch<K, 4, 1>(A, x, y, m, n, st);
    case 100: return gemv_dyn_launch<K, 4, 1, 0>(A, x, y, m, n, st);
    case 101: return gemv_dyn_launch<K, 4, 8, 0>(A, x, y, m, n, st);
    case 102: return gemv_dyn_launch<K, 2, 8, 0>(A, x, y, m, n, st);
    case 103: return gemv_dyn_launch<K, 4, 6, 0>(A, x, y, m, n, st);
    case 104: return gemv_dyn_launch<K, 4, 8, 4>(A, x, y, m, n, st);
    case 105: return gemv_dyn_launch<K, 4, 8, 6>(A, x, y, m, n, st);
    case 106: return gemv_pin_launch<K, 2, 4, 1>(A, x, y, m, n, st);
    case 107: return gemv_pin_launch<K, 2, 2, 1>(A, x, y, m, n, st);
    case 108: return gemv_pin_launch<K, 1, 4, 1>(A, x, y, m, n, st);
    case 109: return gemv_pin_launch<K, 1, 2, 1>(A, x, y, m, n, st);
    case 110: return gemv_pin_launch<K, 2, 4, 0>(A, x, y, m, n, st);
    case 111: return gemv_pin_launch<K, 4, 2, 1>(A, x, y, m, n, st);
    case 112: return gemv_pin_launch<K, 2, 8, 1>(A, x, y, m, n, st);
    case 113: return gemv_pin_launch<K, 1, 8, 1>(A, x, y, m, n, st);
    case 114: return gemv_pin_launch<K, 2, 4, 3>(A, x, y, m, n, st);
    case 115: return gemv_pin_launch<K, 4, 4, 1>(A, x, y, m, n, st);
    default: return MW_ERR_INVALID;
  }
}
extern "C" int mwt_gemv_num_configs(void) { return 116; }
extern "C" const char* mwt_gemv_config_name(int cfg) {
  static const char* names[] = {"W4_R2_D4", "W1_R8_D8", "W1_R8_D4", "W2_R4_D4", "W2_R4_D8",
                                "W4_R2_D2", "W4_R1_D4", "W8_R1_D2", "st_R2_D4_S2", "st_R2_D4_S3",
                                "st_R1_D4_S2", "st_R1_D4_S3", "st_R2_D2_S2", "st_R2_D2_S4",
                                "stx_R1_D4_S2", "stx_R2_D4_S2", "st_R1_D8_S2", "st_R1_D2_S4",
                                "bk_G8_C256_S2", "bk_G6_C256_S3", "bk_G4_C512_S2", "bk_G8_C128_S3",
                                "bk_G6_C256_S2", "bk_G4_C256_S3", "bk_G5_C256_S2", "bk_G7_C128_S4", "probe_fp64", "probe_mem",
                                "rt1_D4", "rt1_D2_P", "rt1_D4_P", "rt2_D2", "rt2_D4", "rt2_D2_P",
                                "rt2_D1_P", "rt1_D2_P_b8", "rt2_D2_P_b4", "rt1_D1_P_b12",
                                "wr_Q8_J2_S4", "wr_Q8_J2_S3", "wr_Q6_J2_S4", "wr_Q6_J4_S2", "wr_Q4_J4_S3",
                                "wr_Q8_J1_S6", "wr_Q6_J2_S3", "mc_C2_D2", "mc_C2_D1", "mc_C2_D2_R2",
                                "mc_C2_D1_R2", "mc_C1_D4", "mc_C4_D1", "v2_D2_R2", "v2_D2_R1", "v2_D1_R2", "v2_D4_R1",
                                "xs_R8_D4", "xs_R6_D4", "xs_R4_D4_c2", "xs_R8_D2", "cs_R2_D4", "cs_R1_D4",
                                "pt_S1_D4", "pt_S2_D4", "pt_S1_D2", "pt_S2_D2", "pt_S4_D4", "pt_S1_D8",
                                "np_S1_D4", "np_S2_D4", "pt_S2_D8", "pn_S1_D4", "pn_S2_D4", "pn_S1_D4_m8",
                                "pn_S2_D4_m4", "nn_S1_D4", "nn_S2_D4", "nn_S1_D4_m8", "nn_S2_D4_m4", "nn_S1_D2_m8", "pn_S1_D2_m8",
                                "cg_D4_S3", "cg_D4_S4", "cg_D2_S4", "cg_D2_S6", "cg_D2_S3", "cg_D1_S8", "cg_D4_S2", "cg_D8_S2",
                                "u2_D2_R1", "u2_D2_R2", "u2_D4_R1", "u2_D4_R2", "u2_D1_R2", "u2_D2_R4",
                                "w1_D1_W1", "w1_D2_W1", "w1_D1_W2", "w1_D2_W2", "w1_D1_W4", "w1_D4_W1",
                                "dy_D4", "dy_D4_m8", "dy_D2_m8", "dy_D4_m6", "dy_D4_m8_c4", "dy_D4_m8_c6",
                                "pin_R2_D4", "pin_R2_D2", "pin_R1_D4", "pin_R1_D2", "pin0_R2_D4", "pin_R4_D2",
                                "pin_R2_D8", "pin_R1_D8", "pin3_R2_D4", "pin_R4_D4"};
  return (cfg >= 0 && cfg < 116) ? names[cfg] : "?";
}
extern "C" int mwt_gemv(int cfg, int k, const double* A, const double* x, double* y, int64_t m,
                        int64_t n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (k == 3) return gemv_run<3>(cfg, A, x, y, m, n, st);
  if (k == 4) return gemv_run<4>(cfg, A, x, y, m, n, st);
  return MW_ERR_INVALID;
}
