// dk_tree_k4_bf.cu — instantiates the tree-order DK sweep launchers for
// K = 4, variant bf (split out of dk.cu so the kernels compile in parallel).
#include "dk_kernels.cuh"

namespace mw {
template MW_DK_LAUNCH_SIG(dk_tree_launch, 4, 1, false);
template MW_DK_LAUNCH_SIG(dk_tree_launch, 4, 1, true);
}  // namespace mw
