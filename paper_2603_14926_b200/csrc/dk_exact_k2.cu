// dk_exact_k2.cu — instantiates the exact-order DK sweep launchers for K = 2
// (split out of dk.cu so the kernels compile in parallel).
#include "dk_kernels.cuh"

namespace mw {
MW_DK_FOR_K(template, dk_exact_launch, 2)
}  // namespace mw
