// Small tuning harness for the pinned-prefetch GEMV probe (fast to build):
// config 0 = the product kernel, others = gemv_pin_kernel shapes.  Same
// entry points as libmwtune.so so scripts/tune_gemv.py can drive it
// (TUNELIB=libmwpin.so).
#include "../reduce.cu"
#include "gemv_pin.cuh"
#include "gemv_lazy.cuh"
using namespace mw;
static int64_t g_sa = 0, g_lda = 0;
extern "C" void mwt_gemv_set_lda(int64_t v) { g_lda = v; }
extern "C" void mwt_gemv_set_sa(int64_t v) { g_sa = v; }
static inline int64_t SA(int64_t m, int64_t n) { return g_sa > 0 ? g_sa : m * n; }
static inline int64_t LDA(int64_t n) { return g_lda == 0 ? n : (g_lda < 0 ? 0 : g_lda); }
template <int K, int RPC, int D, int PIN, int MINB>
static int pin(const double* A, const double* x, double* y, int64_t m, int64_t n, cudaStream_t st) {
  gemv_pin_kernel<K, BRANCH_FREE, RPC, D, PIN, MINB>
      <<<(unsigned)((m + RPC - 1) / RPC), 128 * RPC, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
  return launch_status();
}
template <int K>
static int run(int cfg, const double* A, const double* x, double* y, int64_t m, int64_t n, cudaStream_t st) {
  switch (cfg) {
    case 0:
      if (K == 3)
        gemv_tree_kernel<K, BRANCH_FREE, 4, 2, 4><<<(unsigned)((m + 1) / 2), 256, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
      else
        gemv_tree_kernel<K, BRANCH_FREE, 4, 1, 4><<<(unsigned)m, 128, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
      return launch_status();
    case 1: return pin<K, 1, 2, 1, 8>(A, x, y, m, n, st);
    case 2: return pin<K, 1, 2, 1, 6>(A, x, y, m, n, st);
    case 3: return pin<K, 1, 1, 1, 8>(A, x, y, m, n, st);
    case 4: return pin<K, 1, 1, 1, 6>(A, x, y, m, n, st);
    case 5: return pin<K, 1, 4, 1, 6>(A, x, y, m, n, st);
    case 6: return pin<K, 2, 2, 1, 4>(A, x, y, m, n, st);
    case 7: return pin<K, 2, 1, 1, 4>(A, x, y, m, n, st);
    case 8: return pin<K, 2, 2, 1, 3>(A, x, y, m, n, st);
    case 9: return pin<K, 1, 1, 1, 10>(A, x, y, m, n, st);
    case 10:
      if (K != 3) return MW_ERR_INVALID;
      gemv_lazy_td_kernel<2, 4><<<(unsigned)((m + 1) / 2), 256, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
      return launch_status();
    case 11:
      if (K != 3) return MW_ERR_INVALID;
      gemv_lazy_td_kernel<1, 4><<<(unsigned)m, 128, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
      return launch_status();
    case 12:
      if (K != 3) return MW_ERR_INVALID;
      gemv_lazy_td_kernel<2, 2><<<(unsigned)((m + 1) / 2), 256, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
      return launch_status();
    case 13:
      if (K != 3) return MW_ERR_INVALID;
      gemv_lazy_pin_td_kernel<1, 4, 1><<<(unsigned)m, 128, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
      return launch_status();
    case 14:
      if (K != 3) return MW_ERR_INVALID;
      gemv_lazy_pin_td_kernel<1, 2, 1><<<(unsigned)m, 128, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
      return launch_status();
    case 15:
      if (K != 3) return MW_ERR_INVALID;
      gemv_lazy_pin_td_kernel<1, 4, 6><<<(unsigned)m, 128, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
      return launch_status();
    case 16:
      if (K != 3) return MW_ERR_INVALID;
      gemv_lazy_pin_td_kernel<1, 8, 1><<<(unsigned)m, 128, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
      return launch_status();
    case 17:
      if (K != 3) return MW_ERR_INVALID;
      gemv_lazy_pin_td_kernel<2, 4, 1><<<(unsigned)((m + 1) / 2), 256, 0, st>>>(A, LDA(n), SA(m, n), x, n, y, m, m, n);
      return launch_status();
    default: return MW_ERR_INVALID;
  }
}
extern "C" int mwt_gemv_num_configs(void) { return 18; }
extern "C" const char* mwt_gemv_config_name(int cfg) {
  static const char* names[] = {"product", "pin_R1_D2_m8", "pin_R1_D2_m6", "pin_R1_D1_m8", "pin_R1_D1_m6",
                                "pin_R1_D4_m6", "pin_R2_D2_m4", "pin_R2_D1_m4", "pin_R2_D2_m3", "pin_R1_D1_m10",
                                "lazy_R2_D4", "lazy_R1_D4", "lazy_R2_D2",
                                "lzpin_R1_D4", "lzpin_R1_D2", "lzpin_R1_D4_m6", "lzpin_R1_D8", "lzpin_R2_D4"};
  return (cfg >= 0 && cfg < 18) ? names[cfg] : "?";
}
extern "C" int mwt_gemv(int cfg, int k, const double* A, const double* x, double* y, int64_t m, int64_t n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (k == 3) return run<3>(cfg, A, x, y, m, n, st);
  if (k == 4) return run<4>(cfg, A, x, y, m, n, st);
  return MW_ERR_INVALID;
}
