// gemv_pin.cuh -- tuning probe (not in libmwgpu.so): the tree-order GEMV of
// gemv_tree_kernel (same 128 partials per row, same pairwise tree, so
// bit-identical) with a register double buffer whose next-group loads are
// PINNED above the current group's fold.  The round-1/2 "P" variants
// (gemv_rt_kernel<..., PIPE>) had their prefetch loads sunk below the fold
// by ptxas; here a warp barrier (a memory-ordering point that ptxas does not
// move global loads across) sits between the prefetch and the fold, so the
// LDGs of group g+1 are issued before the first FP64 instruction of group g.
// Only A (the HBM stream) is prefetched; x comes from L1/L2 at its use.
#pragma once
#include "../common.cuh"

namespace mw {

template <int PIN>
__device__ __forceinline__ void gemv_pin_fence() {
  if (PIN == 1) __syncwarp();
  if (PIN == 2) asm volatile("bar.warp.sync 0xffffffff;" ::: "memory");
  if (PIN == 3) asm volatile("" ::: "memory");
}

template <int K, int VAR, int RPC, int D, int PIN, int MINB = 1>
__global__ void __launch_bounds__(128 * RPC, MINB)
    gemv_pin_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                    const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                    int64_t m, int64_t n) {
  constexpr int P = 128;
  const int lane = threadIdx.x & 31;
  const int warp = (threadIdx.x >> 5) & 3;
  const int slot = threadIdx.x >> 7;
  const int64_t i = blockIdx.x * (int64_t)RPC + slot;
  const bool live = i < m;
  const double* row = A + (live ? i : 0) * lda;
  const int u = warp * 32 + lane;
  // full groups every lane of the warp has (warp-uniform, so the barrier is
  // reached by all 32 lanes): elements of the warp's last partial / D
  const int ulast = warp * 32 + 31;
  const int64_t ng = n > ulast ? ((n - ulast + P - 1) / P) / D : 0;
  V<K> acc = zero<K>();
  int64_t t = u;
  V<K> cur[D], nxt[D];
  if (ng > 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) cur[d] = load<K>(row, sA, t + d * P);
  }
  for (int64_t g = 0; g < ng; ++g) {
    const bool more = g + 1 < ng;
    if (more) {
#pragma unroll
      for (int d = 0; d < D; ++d) nxt[d] = load<K>(row, sA, t + (D + d) * P);
    }
    gemv_pin_fence<PIN>();
#pragma unroll
    for (int d = 0; d < D; ++d)
      acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(cur[d], load<K>(x, sx, t + d * P)));
    t += D * P;
    if (more) {
#pragma unroll
      for (int d = 0; d < D; ++d) cur[d] = nxt[d];
    }
  }
  for (; t < n; t += P)
    acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(row, sA, t), load<K>(x, sx, t)));
  const int64_t valid = n < P ? n : P;
  __shared__ double part[RPC][K][P];
#pragma unroll
  for (int c = 0; c < K; ++c) part[slot][c][u] = acc.c[c];
  __syncthreads();
  const int tid = threadIdx.x;
#pragma unroll 1
  for (int s = 1; s < P; s <<= 1) {
    const int per_row = P / (2 * s);
    if (tid < RPC * per_row) {
      const int r = tid / per_row, idx = 2 * s * (tid % per_row);
      if (idx + s < valid) {
        V<K> a, b;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          a.c[c] = part[r][c][idx];
          b.c[c] = part[r][c][idx + s];
        }
        const V<K> sum = Ops<K, VAR>::add(a, b);
#pragma unroll
        for (int c = 0; c < K; ++c) part[r][c][idx] = sum.c[c];
      }
    }
    __syncthreads();
  }
  if (warp == 0 && lane == 0 && live) {
    V<K> r0;
#pragma unroll
    for (int c = 0; c < K; ++c) r0.c[c] = part[slot][c][0];
    store<K>(y, sy, i, r0);
  }
}

}  // namespace mw
