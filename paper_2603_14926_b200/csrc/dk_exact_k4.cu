// dk_exact_k4.cu — instantiates the exact-order DK sweep launchers for K = 4
// (split out of dk.cu so the kernels compile in parallel).
#include "dk_kernels.cuh"

namespace mw {
MW_DK_FOR_K(template, dk_exact_launch, 4)
}  // namespace mw
