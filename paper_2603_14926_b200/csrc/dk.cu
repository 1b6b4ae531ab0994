// dk.cu — the Durand-Kerner sweep C-ABI (kernels: dk_kernels.cuh).
#include "dk_kernels.cuh"

namespace mw {

#define MW_DK_EXTERN(FN) \
  MW_DK_FOR_K(extern template, FN, 2) MW_DK_FOR_K(extern template, FN, 3) MW_DK_FOR_K(extern template, FN, 4)
MW_DK_EXTERN(dk_exact_launch)
MW_DK_EXTERN(dk_tree_launch)

template <int K, int VAR>
struct DkLaunch {
  static int run(const double* coeffs, int64_t sc, int64_t n, const double* zre,
                 const double* zim, int64_t sz, int64_t i0, int64_t i1, double* zre_out,
                 double* zim_out, int64_t so, double* step_mag, int* flag, int exact, double* ws,
                 mw_tuning tune, unsigned long long* max_bits, cudaStream_t st) {
    DkPeers none{};
    none.max_bits = max_bits;
    if (exact)
      return dk_exact_launch<K, VAR, false>(coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out,
                                            so, step_mag, flag, none, ws, tune, st);
    return dk_tree_launch<K, VAR, false>(coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out,
                                         so, step_mag, flag, none, ws, tune, st);
  }
};

template <int K, int VAR>
struct DkPeerLaunch {
  static int run(const double* coeffs, int64_t sc, int64_t n, const double* state_in,
                 int64_t i0, int64_t i1, double* state_out, double* step_mag, int* flag,
                 int exact, DkPeers peers, double* ws, cudaStream_t st) {
    const double* zre = state_in;
    const double* zim = state_in + (int64_t)K * n;
    double* ore = state_out;
    double* oim = state_out + (int64_t)K * n;
    if (exact)
      return dk_exact_launch<K, VAR, true>(coeffs, sc, n, zre, zim, n, i0, i1, ore, oim, n,
                                           step_mag, flag, peers, ws, tuning_defaults(), st);
    return dk_tree_launch<K, VAR, true>(coeffs, sc, n, zre, zim, n, i0, i1, ore, oim, n,
                                        step_mag, flag, peers, ws, tuning_defaults(), st);
  }
};

}  // namespace mw

using namespace mw;

extern "C" int mw_tuning_defaults(mw_tuning* t) {
  if (!t) return MW_ERR_INVALID;
  *t = tuning_defaults();
  return MW_OK;
}

extern "C" int mw_dk_sweep(int k, int variant, const double* coeffs, int64_t sc, int64_t n,
                           const double* zre, const double* zim, int64_t sz, int64_t i0,
                           int64_t i1, double* zre_out, double* zim_out, int64_t so,
                           double* step_mag, int* flag_dev, int exact_order, void* stream) {
  return mw_dk_sweep_ex(k, variant, coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so,
                        step_mag, flag_dev, exact_order, nullptr, nullptr, nullptr, stream);
}

extern "C" int64_t mw_dk_sweep_workspace(int k, int64_t i0, int64_t i1) {
  if (k < 2 || k > 4 || i1 < i0 || i0 < 0) return 0;
  return 4 * (int64_t)k * (i1 - i0);
}

// mw_dk_sweep with a caller workspace of mw_dk_sweep_workspace(k, i0, i1)
// doubles: the tree order then takes z^B and w^32 from a lane-per-root
// kernel (programmatic dependent launch).  Same results.
extern "C" int mw_dk_sweep_ws(int k, int variant, const double* coeffs, int64_t sc, int64_t n,
                              const double* zre, const double* zim, int64_t sz, int64_t i0,
                              int64_t i1, double* zre_out, double* zim_out, int64_t so,
                              double* step_mag, int* flag_dev, int exact_order, double* ws,
                              void* stream) {
  return mw_dk_sweep_ex(k, variant, coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so,
                        step_mag, flag_dev, exact_order, ws, nullptr, nullptr, stream);
}

// The sweep with explicit per-call tuning (NULL = defaults).  The collision
// key j*n + i is an int: n above 46340 would overflow it, so such sizes are
// rejected instead of silently losing a collision.
extern "C" int mw_dk_sweep_ex(int k, int variant, const double* coeffs, int64_t sc, int64_t n,
                              const double* zre, const double* zim, int64_t sz, int64_t i0,
                              int64_t i1, double* zre_out, double* zim_out, int64_t so,
                              double* step_mag, int* flag_dev, int exact_order, double* ws,
                              unsigned long long* max_mag_bits, const mw_tuning* tune,
                              void* stream) {
  mw_tuning t;
  if (!tuning_resolve(tune, &t)) return MW_ERR_INVALID;
  if (k < 2 || k > 4) return MW_ERR_INVALID;
  if (variant != 0 && variant != 1) return MW_ERR_INVALID;
  if (n < 1 || n > MW_DK_MAX_N || i0 < 0 || i1 < i0 || i1 > n) return MW_ERR_INVALID;
  if (i1 == i0) return MW_OK;
  if (!coeffs || !zre || !zim || !zre_out || !zim_out || !step_mag || !flag_dev)
    return MW_ERR_INVALID;
  if (sc < n || sz < n || so < n) return MW_ERR_INVALID;
  return dispatch<DkLaunch>(k, variant, coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out,
                            so, step_mag, flag_dev, exact_order ? 1 : 0, ws, t, max_mag_bits,
                            as_stream(stream));
}

// Root-sharded sweep with the state exchange fused in (peer stores over
// NVLink + per-source completion slots, see DkPeers).  state_in / the
// peer_out[rank] buffer hold (2K, n) planes (re planes, then im planes,
// plane stride n).  peer_out and peer_slot are DEVICE arrays of world
// pointers.  Roots [i0, i1) are this rank's shard.
extern "C" int mw_dk_sweep_peer(int k, int variant, const double* coeffs, int64_t sc, int64_t n,
                                const double* state_in, int64_t i0, int64_t i1,
                                double* const* peer_out, unsigned long long* const* peer_slot,
                                double* state_out_local, unsigned long long* my_slot,
                                unsigned int* done, unsigned long long* epoch, int* timeout,
                                int world, int rank, int sweep, int sweeps, long long spin_limit,
                                double* step_mag, int* flag_dev, int exact_order, double* ws,
                                void* stream) {
  if (k < 2 || k > 4) return MW_ERR_INVALID;
  if (variant != 0 && variant != 1) return MW_ERR_INVALID;
  if (n < 1 || n > MW_DK_MAX_N || i0 < 0 || i1 <= i0 || i1 > n) return MW_ERR_INVALID;
  if (world < 1 || rank < 0 || rank >= world || sweeps < 1 || sweep < 0 || sweep >= sweeps)
    return MW_ERR_INVALID;
  if (spin_limit < 1) return MW_ERR_INVALID;
  if (!coeffs || !state_in || !peer_out || !peer_slot || !state_out_local || !my_slot || !done ||
      !epoch || !timeout || !step_mag || !flag_dev)
    return MW_ERR_INVALID;
  if (sc < n) return MW_ERR_INVALID;
  DkPeers P{peer_out, peer_slot, my_slot, done, epoch, timeout, spin_limit, world, rank, sweep, sweeps};
  return dispatch<DkPeerLaunch>(k, variant, coeffs, sc, n, state_in, i0, i1, state_out_local,
                                step_mag, flag_dev, exact_order ? 1 : 0, P, ws,
                                as_stream(stream));
}

// Peer buffers: plain cudaMalloc allocations (zeroed) so one IPC handle
// covers exactly one buffer.
extern "C" int mw_peer_alloc(int64_t bytes, void** out) {
  if (bytes < 1 || !out) return MW_ERR_INVALID;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)bytes);
  if (e != cudaSuccess) return (int)e;
  e = cudaMemset(p, 0, (size_t)bytes);
  if (e != cudaSuccess) {
    cudaFree(p);
    return (int)e;
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return (int)e;
  *out = p;
  return MW_OK;
}

extern "C" int mw_peer_free(void* p) {
  if (!p) return MW_ERR_INVALID;
  return (int)cudaFree(p);
}

// 64-byte opaque handle (cudaIpcMemHandle_t) for a mw_peer_alloc buffer.
extern "C" int mw_ipc_get_handle(void* p, void* handle64) {
  if (!p || !handle64) return MW_ERR_INVALID;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) return (int)e;
  memcpy(handle64, &h, sizeof(h));
  return MW_OK;
}

extern "C" int mw_ipc_open_handle(const void* handle64, void** out) {
  if (!handle64 || !out) return MW_ERR_INVALID;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return (int)e;
  *out = p;
  return MW_OK;
}

extern "C" int mw_ipc_close_handle(void* p) {
  if (!p) return MW_ERR_INVALID;
  return (int)cudaIpcCloseMemHandle(p);
}
