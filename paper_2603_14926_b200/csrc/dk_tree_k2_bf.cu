// dk_tree_k2_bf.cu — instantiates the tree-order DK sweep launchers for
// K = 2, variant bf (split out of dk.cu so the kernels compile in parallel).
#include "dk_kernels.cuh"

namespace mw {
template MW_DK_LAUNCH_SIG(dk_tree_launch, 2, 1, false);
template MW_DK_LAUNCH_SIG(dk_tree_launch, 2, 1, true);
}  // namespace mw
