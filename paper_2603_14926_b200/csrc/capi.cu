// capi.cu — library metadata, device helpers and the FP64 pipe
// microbenchmark used as the roofline denominator.
#include <atomic>
#include "common.cuh"

namespace mw {

// Per-device cache (one process may drive several GPUs); a benign race
// only repeats the query.
int sm_count() {
  static std::atomic<int> cached[64];  // zero-initialised; racing first calls store the same value
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cached[dev].load(std::memory_order_relaxed) == 0) {
    int v = 0;
    cached[dev] = (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
                   v > 0)
                      ? v
                      : 148;
  }
  return cached[dev];
}

// CHAINS independent dependent chains per thread keep the FP64 pipe busy
// without any memory traffic.  op 0: DFMA x = x*a + b; op 1: DADD x = x + b.
template <int OP>
__global__ void __launch_bounds__(256) fp64_peak_kernel(int iters, double* sink) {
  constexpr int CHAINS = 8;
  double x[CHAINS];
  const double a = 0.999999999 + threadIdx.x * 1e-12, b = 1e-9;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = 1.0 + c * 1e-3 + blockIdx.x * 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) x[c] = OP == 0 ? __fma_rn(x[c], a, b) : __dadd_rn(x[c], b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  sink[blockIdx.x * (int64_t)blockDim.x + threadIdx.x] = s;
}

}  // namespace mw

using namespace mw;

extern "C" const char* mw_version(void) { return "mwgpu 0.1 sm_100a"; }

extern "C" const char* mw_status_string(int status) {
  if (status == MW_OK) return "ok";
  if (status == MW_ERR_INVALID) return "invalid argument";
  if (status == MW_ERR_UNSUPPORTED) return "no device kernel for this (k, variant)";
  if (status > 0) return cudaGetErrorString(static_cast<cudaError_t>(status));
  return "unknown status";
}

extern "C" int mw_device_sm_count(void) { return sm_count(); }

// Each thread runs 8 chains x 8 unrolled steps per iteration: the op count
// is blocks * threads * iters * 64.
extern "C" int mw_fp64_peak_kernel(int op, int blocks, int threads, int iters, double* sink,
                                   void* stream) {
  if (blocks < 1 || threads < 1 || threads > 256 || iters < 1 || !sink) return MW_ERR_INVALID;
  if (op == 0)
    fp64_peak_kernel<0><<<blocks, threads, 0, as_stream(stream)>>>(iters, sink);
  else if (op == 1)
    fp64_peak_kernel<1><<<blocks, threads, 0, as_stream(stream)>>>(iters, sink);
  else
    return MW_ERR_INVALID;
  return launch_status();
}
