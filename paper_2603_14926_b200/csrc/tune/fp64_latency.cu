// fp64_latency.cu — microbenchmark (not product): dependent-chain latency
// of DADD / DMUL / DFMA on one thread, in SM clock cycles.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cycles, int n) {
  double x = out[0], a = out[1], b = out[2];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) x = __dadd_rn(x, b);
      if (OP == 1) x = __dmul_rn(x, a);
      if (OP == 2) x = __fma_rn(x, a, b);
    }
  }
  long long t1 = clock64();
  out[3] = x;
  cycles[0] = t1 - t0;
}

// Throughput of ONE warp with 8 independent chains (ILP 8) per thread.
__global__ void warp_tput(double* out, long long* cycles, int n) {
  double x[8], b = out[2];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = out[0] + c;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = __dadd_rn(x[c], b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  out[3 + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  double h[4] = {1.0, 1.0000001, 1e-9, 0.0};
  double* d;
  long long* c;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&c, sizeof(long long));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  const char* names[] = {"DADD", "DMUL", "DFMA"};
  for (int op = 0; op < 3; ++op) {
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) chain<0><<<1, 1>>>(d, c, n);
      if (op == 1) chain<1><<<1, 1>>>(d, c, n);
      if (op == 2) chain<2><<<1, 1>>>(d, c, n);
    }
    long long cyc = 0;
    cudaMemcpy(&cyc, c, sizeof(cyc), cudaMemcpyDeviceToHost);
    printf("%s dependent latency: %.2f cycles/op\n", names[op], (double)cyc / (n * 16.0));
  }
  double* d2;
  cudaMalloc(&d2, 4096 * sizeof(double));
  cudaMemcpy(d2, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int warps = 1; warps <= 8; warps *= 2) {
    const int n = 2048;
    warp_tput<<<1, 32 * warps>>>(d2, c, n);
    warp_tput<<<1, 32 * warps>>>(d2, c, n);
    long long cyc = 0;
    cudaMemcpy(&cyc, c, sizeof(cyc), cudaMemcpyDeviceToHost);
    const double instr = n * 32.0;  // warp instructions per warp
    printf("%d warp(s)/CTA, ILP 8: %.2f cycles per warp-DADD per warp (%.1f lanes/clk/SM)\n", warps,
           cyc / instr, 32.0 * warps * instr / cyc);
  }
  return 0;
}
