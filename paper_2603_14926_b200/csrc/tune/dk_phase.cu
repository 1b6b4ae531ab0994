// dk_phase.cu -- tuning harness: the tree DK sweep built with phase
// timestamps (MW_DK_PROFILE: %globaltimer per CTA at each phase boundary of
// dk_treem_kernel), read back by scripts/dk_phases.py.
#define MW_DK_PROFILE 1
#include "../dk_kernels.cuh"

namespace mw {
int sm_count() { return 148; }
}  // namespace mw
using namespace mw;

extern "C" int dkp_sweep(int k, const double* coeffs, int64_t n, const double* zre,
                         const double* zim, int64_t i0, int64_t i1, double* zre_out,
                         double* zim_out, double* step_mag, int* flag, double* ws, int roots,
                         void* stream) {
  mw_tuning tune = tuning_defaults();
  tune.dk_tree_roots = roots;
  cudaStream_t st = (cudaStream_t)stream;
  if (k == 3)
    return dk_tree_launch<3, BRANCH_FREE, false>(coeffs, n, n, zre, zim, n, i0, i1, zre_out, zim_out,
                                                 n, step_mag, flag, DkPeers{}, ws, tune, st);
  if (k == 4)
    return dk_tree_launch<4, BRANCH_FREE, false>(coeffs, n, n, zre, zim, n, i0, i1, zre_out, zim_out,
                                                 n, step_mag, flag, DkPeers{}, ws, tune, st);
  return MW_ERR_INVALID;
}

extern "C" int dkp_read(unsigned long long* host, int ctas) {
  return (int)cudaMemcpyFromSymbol(host, g_dk_prof, sizeof(unsigned long long) * 12 * ctas);
}
