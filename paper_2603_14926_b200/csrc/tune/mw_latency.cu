// mw_latency.cu — microbenchmark (not product): dependent-chain latency of
// the branch-free K-word add and mul on one warp (all lanes active), in SM
// cycles per op, and the same with 2 and 4 independent chains per thread.
// It bounds the exact-order DK sweep (one dependent chain per root).
#include <cstdio>
#include <cuda_runtime.h>

#include "../common.cuh"

using namespace mw;

template <int K, int OP, int CH>
__global__ void chain(double* io, long long* cycles, int n) {
  V<K> x[CH], b;
#pragma unroll
  for (int c = 0; c < K; ++c) b.c[c] = io[c] * (c ? 1e-17 : 1.0);
#pragma unroll
  for (int h = 0; h < CH; ++h)
#pragma unroll
    for (int c = 0; c < K; ++c) x[h].c[c] = io[K + c] * (c ? 1e-17 : 1.0) + h + threadIdx.x;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int h = 0; h < CH; ++h) {
      if (OP == 0) x[h] = Ops<K, BRANCH_FREE>::add(x[h], b);
      else x[h] = Ops<K, BRANCH_FREE>::mul(x[h], b);
    }
  }
  __syncwarp();
  long long t1 = clock64();
#pragma unroll
  for (int h = 0; h < CH; ++h)
#pragma unroll
    for (int c = 0; c < K; ++c) io[2 * K + threadIdx.x * K * CH + h * K + c] = x[h].c[c];
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

template <int K, int OP, int CH>
static double run(double* d, long long* c) {
  const int n = 2048;
  for (int rep = 0; rep < 2; ++rep) chain<K, OP, CH><<<1, 32>>>(d, c, n);
  long long cyc = 0;
  cudaMemcpy(&cyc, c, sizeof(cyc), cudaMemcpyDeviceToHost);
  return (double)cyc / n;  // cycles per step (CH ops)
}

int main() {
  double h[8] = {1.0000001, 0.3, 0.7, 0.1, 0.99999, 0.5, 0.25, 0.125};
  double* d;
  long long* c;
  cudaMalloc(&d, 4096 * sizeof(double));
  cudaMalloc(&c, sizeof(long long));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  printf("cycles per step, one warp (32 lanes); CH independent chains per thread\n");
  printf("K=2 add: CH1 %.0f CH2 %.0f CH4 %.0f | mul: CH1 %.0f CH2 %.0f CH4 %.0f\n", run<2, 0, 1>(d, c),
         run<2, 0, 2>(d, c), run<2, 0, 4>(d, c), run<2, 1, 1>(d, c), run<2, 1, 2>(d, c), run<2, 1, 4>(d, c));
  printf("K=3 add: CH1 %.0f CH2 %.0f CH4 %.0f | mul: CH1 %.0f CH2 %.0f CH4 %.0f\n", run<3, 0, 1>(d, c),
         run<3, 0, 2>(d, c), run<3, 0, 4>(d, c), run<3, 1, 1>(d, c), run<3, 1, 2>(d, c), run<3, 1, 4>(d, c));
  printf("K=4 add: CH1 %.0f CH2 %.0f CH4 %.0f | mul: CH1 %.0f CH2 %.0f CH4 %.0f\n", run<4, 0, 1>(d, c),
         run<4, 0, 2>(d, c), run<4, 0, 4>(d, c), run<4, 1, 1>(d, c), run<4, 1, 2>(d, c), run<4, 1, 4>(d, c));
  return 0;
}
