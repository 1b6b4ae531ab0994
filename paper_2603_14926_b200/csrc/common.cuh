// common.cuh — launch helpers shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mwgpu.h"
#include "mw_eft.cuh"

namespace mw {

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Cached SM count of the current device (148 on B200).
int sm_count();

// Per-call tuning (include/mwgpu.h): NULL -> the defaults; out-of-range
// values -> false (the entry point returns MW_ERR_INVALID).
inline mw_tuning tuning_defaults() { return mw_tuning{0, 1, -1, 32, 1}; }
inline bool tuning_resolve(const mw_tuning* in, mw_tuning* out) {
  *out = in ? *in : tuning_defaults();
  const mw_tuning& t = *out;
  if (t.gemm_tile < 0 || t.gemm_tile > 3) return false;
  if (t.dot_cluster != 0 && t.dot_cluster != 1) return false;
  if (t.dk_tree_roots != -1 && t.dk_tree_roots != 0 && t.dk_tree_roots != 1 && t.dk_tree_roots != 2 &&
      t.dk_tree_roots != 4)
    return false;
  if (t.dk_exact_roots < 1 || t.dk_exact_roots > 32) return false;
  if (t.dk_exact_split != 0 && t.dk_exact_split != 1) return false;
  return true;
}

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MW_OK : static_cast<int>(e);
}

// (k, variant) -> F<K, VAR>::run(args...) for k = 2, 3, 4 and both variants.
template <template <int, int> class F, typename... Args>
int dispatch(int k, int variant, Args... args) {
  if (variant == BRANCH_FREE) {
    switch (k) {
      case 2: return F<2, BRANCH_FREE>::run(args...);
      case 3: return F<3, BRANCH_FREE>::run(args...);
      case 4: return F<4, BRANCH_FREE>::run(args...);
      default: return MW_ERR_INVALID;
    }
  }
  if (variant == STANDARD) {
    switch (k) {
      case 2: return F<2, STANDARD>::run(args...);
      case 3: return F<3, STANDARD>::run(args...);
      case 4: return F<4, STANDARD>::run(args...);
      default: return MW_ERR_INVALID;
    }
  }
  return MW_ERR_INVALID;
}

// 8-byte asynchronous global->shared copy; src_bytes = 0 zero-fills.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int K>
__device__ __forceinline__ V<K> shfl_down(const V<K>& v, int s) {
  V<K> r;
#pragma unroll
  for (int c = 0; c < K; ++c) r.c[c] = __shfl_down_sync(0xffffffffu, v.c[c], s);
  return r;
}

}  // namespace mw
