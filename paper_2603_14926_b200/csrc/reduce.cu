// reduce.cu — dot, pairwise-tree fold and GEMV.
//
// Reference semantics (no dot/gemv function exists in the reference; both
// are defined from the naive matmul fold, linalg.py:284-314):
//   dot(x, y)  = fold_t add(acc, mul(x_t, y_t)), acc = exact zero, t asc.
//   gemv(A, x)_i = the same fold over row i.
// MW_ORDER_EXACT replays that fold on one thread per output (bit-exact).
// MW_ORDER_TREE is the throughput order; its tree is a pure function of n
// (never of grid shape or GPU count), so results are deterministic and
// identical on 1..8 GPUs:
//   dot:  block b covers elements [4096b, 4096b+4096); its partial p
//         (p = 0..255, global partial index 256b + p) folds the elements
//         4096b + p + 256j, j = 0..15, ascending from exact zero (coalesced:
//         consecutive lanes read consecutive elements).  Partial 256b + p
//         exists iff 4096b + p < n.  Partials combine by the in-place
//         pairwise tree (stride s = 1, 2, 4, ...: v[i] <- add(v[i], v[i+s])
//         for i % 2s == 0 when i+s < count; an unpaired tail passes through).
//   gemv: 128 partials per row; partial u folds t = u, u+128, ... ascending
//         from exact zero; the partials combine by the same pairwise tree.
#include <atomic>
#include "common.cuh"
#include "peer.cuh"

namespace mw {

constexpr int DOT_LEAF = 16;       // elements per partial
constexpr int DOT_BLOCK = 256;     // partials (threads) per block
constexpr int64_t DOT_PER_BLOCK = (int64_t)DOT_LEAF * DOT_BLOCK;  // 4096

// Pairwise tree over the block's 256 values v (one per thread) whose global
// in-place indices are base + tid, valid when < count.  Returns the subtree
// root in thread 0.
template <int K, int VAR>
__device__ __forceinline__ V<K> block_tree(V<K> v, int64_t base, int64_t count) {
  __shared__ double red[K][DOT_BLOCK / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t gi = base + tid;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    V<K> o = shfl_down<K>(v, s);
    if ((lane & (2 * s - 1)) == 0 && gi + s < count) v = Ops<K, VAR>::add(v, o);
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) red[c][warp] = v.c[c];
  }
  __syncthreads();
  if (warp == 0) {
    // level strides 32, 64, 128 act on warp roots w = 0..7 with strides 1, 2, 4
    V<K> w;
    const int nw = DOT_BLOCK / 32;
#pragma unroll
    for (int c = 0; c < K; ++c) w.c[c] = lane < nw ? red[c][lane] : 0.0;
#pragma unroll
    for (int s = 1; s < nw; s <<= 1) {
      V<K> o = shfl_down<K>(w, s);
      if ((lane & (2 * s - 1)) == 0 && lane + s < nw && base + (int64_t)(lane + s) * 32 < count)
        w = Ops<K, VAR>::add(w, o);
    }
    v = w;
  }
  return v;
}

// Number of dot partials for length n (see the order definition above).
__host__ __device__ __forceinline__ int64_t dot_partial_count(int64_t n) {
  if (n <= 0) return 0;
  const int64_t nb = (n + DOT_PER_BLOCK - 1) / DOT_PER_BLOCK;
  const int64_t last = n - (nb - 1) * DOT_PER_BLOCK;
  return (nb - 1) * DOT_BLOCK + (last < DOT_BLOCK ? last : DOT_BLOCK);
}

// Stage 1: block b folds its 256 strided partials and writes their tree root.
template <int K, int VAR>
__global__ void __launch_bounds__(DOT_BLOCK) dot_partials_kernel(
    const double* __restrict__ x, int64_t sx, const double* __restrict__ y, int64_t sy,
    int64_t n, double* __restrict__ partials, int64_t pstride) {
  const int64_t base = blockIdx.x * DOT_PER_BLOCK + threadIdx.x;
  V<K> acc = zero<K>();
  if (blockIdx.x * DOT_PER_BLOCK + DOT_PER_BLOCK <= n) {
    V<K> xs[DOT_LEAF], ys[DOT_LEAF];
#pragma unroll
    for (int j = 0; j < DOT_LEAF; ++j) {
      xs[j] = load<K>(x, sx, base + j * DOT_BLOCK);
      ys[j] = load<K>(y, sy, base + j * DOT_BLOCK);
    }
#pragma unroll
    for (int j = 0; j < DOT_LEAF; ++j)
      acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(xs[j], ys[j]));
  } else {
    for (int64_t t = base; t < n; t += DOT_BLOCK)
      acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(x, sx, t), load<K>(y, sy, t)));
  }
  V<K> r = block_tree<K, VAR>(acc, blockIdx.x * (int64_t)DOT_BLOCK, dot_partial_count(n));
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) partials[c * pstride + blockIdx.x] = r.c[c];
  }
}

// Single-launch tree dot for 1 < nb <= 256 blocks: every block writes its
// subtree root, the last block to finish (atomic ticket) folds the nb roots
// with the same pairwise tree and re-arms the ticket for the next call.
template <int K, int VAR>
__global__ void __launch_bounds__(DOT_BLOCK) dot_fused_kernel(
    const double* __restrict__ x, int64_t sx, const double* __restrict__ y, int64_t sy,
    int64_t n, double* __restrict__ partials, unsigned int* __restrict__ ticket,
    double* __restrict__ out) {
  __shared__ bool is_last;
  const int64_t base = blockIdx.x * DOT_PER_BLOCK + threadIdx.x;
  const int64_t nb = gridDim.x;
  V<K> acc = zero<K>();
  if (blockIdx.x * DOT_PER_BLOCK + DOT_PER_BLOCK <= n) {
    V<K> xs[DOT_LEAF], ys[DOT_LEAF];
#pragma unroll
    for (int j = 0; j < DOT_LEAF; ++j) {
      xs[j] = load<K>(x, sx, base + j * DOT_BLOCK);
      ys[j] = load<K>(y, sy, base + j * DOT_BLOCK);
    }
#pragma unroll
    for (int j = 0; j < DOT_LEAF; ++j)
      acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(xs[j], ys[j]));
  } else {
    for (int64_t t = base; t < n; t += DOT_BLOCK)
      acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(x, sx, t), load<K>(y, sy, t)));
  }
  V<K> r = block_tree<K, VAR>(acc, blockIdx.x * (int64_t)DOT_BLOCK, dot_partial_count(n));
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) partials[c * nb + blockIdx.x] = r.c[c];
    __threadfence();
    is_last = atomicAdd(ticket, 1u) == (unsigned)(nb - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  V<K> v = zero<K>();
  if (threadIdx.x < nb) {
#pragma unroll
    for (int c = 0; c < K; ++c) v.c[c] = __ldcg(partials + c * nb + threadIdx.x);
  }
  __syncthreads();  // block_tree reuses its shared buffer
  V<K> root = block_tree<K, VAR>(v, 0, nb);
  if (threadIdx.x == 0) {
    store<K>(out, 1, 0, root);
    *ticket = 0u;
  }
}

// Single-launch tree dot for 1 < nb <= 16 blocks (n <= 65536, config 1)
// as ONE thread-block cluster: each block's subtree root goes straight into
// the leader block's shared memory (distributed shared memory), one
// cluster barrier, and the leader folds the nb roots with the same
// pairwise tree -- no global partials, fences or atomic ticket on the
// latency path.  Same partials, same trees: bit-identical to
// dot_fused_kernel.
constexpr int DOT_CLUSTER_MAX = 16;
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
template <int K, int VAR>
__global__ void __launch_bounds__(DOT_BLOCK) dot_cluster_kernel(
    const double* __restrict__ x, int64_t sx, const double* __restrict__ y, int64_t sy,
    int64_t n, double* __restrict__ out) {
  __shared__ double roots[K][DOT_CLUSTER_MAX];
  const unsigned rank = cluster_ctarank();
  const int64_t nb = gridDim.x;
  const int64_t base = (int64_t)rank * DOT_PER_BLOCK + threadIdx.x;
  V<K> acc = zero<K>();
  if ((int64_t)rank * DOT_PER_BLOCK + DOT_PER_BLOCK <= n) {
    V<K> xs[DOT_LEAF], ys[DOT_LEAF];
#pragma unroll
    for (int j = 0; j < DOT_LEAF; ++j) {
      xs[j] = load<K>(x, sx, base + j * DOT_BLOCK);
      ys[j] = load<K>(y, sy, base + j * DOT_BLOCK);
    }
#pragma unroll
    for (int j = 0; j < DOT_LEAF; ++j)
      acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(xs[j], ys[j]));
  } else {
    for (int64_t t = base; t < n; t += DOT_BLOCK)
      acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(x, sx, t), load<K>(y, sy, t)));
  }
  V<K> r = block_tree<K, VAR>(acc, (int64_t)rank * DOT_BLOCK, dot_partial_count(n));
  if (threadIdx.x == 0) {
    const unsigned local = static_cast<unsigned>(__cvta_generic_to_shared(&roots[0][rank]));
    unsigned remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(local));
#pragma unroll
    for (int c = 0; c < K; ++c)
      asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote + c * DOT_CLUSTER_MAX * 8u),
                   "d"(r.c[c])
                   : "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank != 0) return;
  V<K> v = zero<K>();
  if (threadIdx.x < nb) {
#pragma unroll
    for (int c = 0; c < K; ++c) v.c[c] = roots[c][threadIdx.x];
  }
  __syncthreads();  // block_tree reuses its shared buffer
  V<K> root = block_tree<K, VAR>(v, 0, nb);
  if (threadIdx.x == 0) store<K>(out, 1, 0, root);
}

// Tree stage above the leaves: groups of 256 values -> one subtree root.
template <int K, int VAR>
__global__ void __launch_bounds__(DOT_BLOCK) tree_fold_kernel(const double* __restrict__ in,
                                                              int64_t istride, int64_t count,
                                                              double* __restrict__ out,
                                                              int64_t ostride) {
  const int64_t i = blockIdx.x * (int64_t)DOT_BLOCK + threadIdx.x;
  V<K> v = zero<K>();
  if (i < count) v = load<K>(in, istride, i);
  V<K> r = block_tree<K, VAR>(v, blockIdx.x * (int64_t)DOT_BLOCK, count);
  if (threadIdx.x == 0) store<K>(out, ostride, blockIdx.x, r);
}

// Exact reference order on one thread (parity path).
template <int K, int VAR>
__global__ void dot_exact_kernel(const double* __restrict__ x, int64_t sx,
                                 const double* __restrict__ y, int64_t sy, int64_t n,
                                 double* __restrict__ out) {
  V<K> acc = zero<K>();
  for (int64_t t = 0; t < n; ++t)
    acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(x, sx, t), load<K>(y, sy, t)));
  store<K>(out, 1, 0, acc);
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Folds `count` values (plane stride istride) in `in` down to one value
// written to out (plane stride 1).  ws holds the intermediate levels:
// needs ceil(count/256) * K doubles (+ the next levels, each 256x smaller).
template <int K, int VAR>
static int fold_levels(const double* in, int64_t istride, int64_t count, double* ws, double* out,
                       cudaStream_t st) {
  const double* cur = in;
  int64_t cstride = istride;
  while (true) {
    int64_t nb = ceil_div(count, DOT_BLOCK);
    double* dst = (nb == 1) ? out : ws;
    int64_t dstride = (nb == 1) ? 1 : nb;
    tree_fold_kernel<K, VAR><<<(unsigned)nb, DOT_BLOCK, 0, st>>>(cur, cstride, count, dst, dstride);
    int rc = launch_status();
    if (rc) return rc;
    if (nb == 1) return MW_OK;
    cur = ws;
    cstride = nb;
    count = nb;
    ws += nb * K;
  }
}

template <int K, int VAR>
struct DotLaunch {
  static int run(const double* x, int64_t sx, const double* y, int64_t sy, int64_t n, double* ws,
                 double* out, int order, int cluster, cudaStream_t st) {
    if (order == MW_ORDER_EXACT || n == 0) {
      dot_exact_kernel<K, VAR><<<1, 1, 0, st>>>(x, sx, y, sy, n, out);
      return launch_status();
    }
    int64_t nb = ceil_div(n, DOT_PER_BLOCK);
    if (nb == 1) {
      dot_partials_kernel<K, VAR><<<1, DOT_BLOCK, 0, st>>>(x, sx, y, sy, n, out, 1);
      return launch_status();
    }
    // ws[0] holds the single-launch ticket (zero before the first call,
    // left zero by every call, never overwritten); partials start at ws + 1
    unsigned int* ticket = reinterpret_cast<unsigned int*>(ws);
    double* part = ws + 1;
    if (nb <= DOT_CLUSTER_MAX && cluster) {
      auto kern = dot_cluster_kernel<K, VAR>;
      static std::atomic<bool> attr_set[64];  // lazy per-device init; idempotent, race-free
      int dev = 0;
      cudaGetDevice(&dev);
      if (dev < 0 || dev >= 64 || !attr_set[dev]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (dev >= 0 && dev < 64) attr_set[dev] = true;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)nb);
      cfg.blockDim = dim3(DOT_BLOCK);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = (unsigned)nb;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (cudaLaunchKernelEx(&cfg, kern, x, sx, y, sy, n, out) == cudaSuccess) return launch_status();
      (void)cudaGetLastError();  // cluster shape not available: the ticket form below
    }
    if (nb <= DOT_BLOCK) {
      dot_fused_kernel<K, VAR><<<(unsigned)nb, DOT_BLOCK, 0, st>>>(x, sx, y, sy, n, part, ticket,
                                                                  out);
      return launch_status();
    }
    dot_partials_kernel<K, VAR><<<(unsigned)nb, DOT_BLOCK, 0, st>>>(x, sx, y, sy, n, part, nb);
    int rc = launch_status();
    if (rc) return rc;
    return fold_levels<K, VAR>(part, nb, nb, part + nb * K, out, st);
  }
};

// Sharded tree dot with the all-gather-then-sum fused in (peer memory):
// rank r's slice covers global blocks [b0, b0 + nb_local); block b stores
// its subtree root into slot b0 + b of EVERY rank's root buffer (cudaIpc
// mapping), takes a ticket; the last block publishes and waits (peer.cuh),
// then folds all nbt block roots from the local buffer with the pairwise
// tree (<= 256: one block tree; <= 65536: two levels of 256, the tree_fold
// order) -- bit-identical to the 1-GPU tree dot on every rank.  Root
// buffers are double-buffered by call parity (epoch & 1) so a rank already
// in call c+1 never overwrites roots a slower rank is still folding.
template <int K, int VAR>
__global__ void __launch_bounds__(DOT_BLOCK) dot_peer_kernel(
    const double* __restrict__ x, int64_t sx, const double* __restrict__ y, int64_t sy,
    int64_t n_local, int64_t b0, int64_t nbt, double* const* peer_roots,
    unsigned long long* const* peer_slot, unsigned long long* my_slot, unsigned int* done,
    unsigned long long* epoch, int* timeout, int world, int rank, long long spin_limit,
    double* __restrict__ out) {
  __shared__ bool is_last;
  __shared__ double lvl[K][DOT_BLOCK];
  const int tid = threadIdx.x;
  const unsigned long long e = *(volatile unsigned long long*)epoch;  // before the ticket
  const int64_t par_off = (int64_t)(e & 1ull) * K * nbt;
  const int64_t nbl = n_local > 0 ? (n_local + DOT_PER_BLOCK - 1) / DOT_PER_BLOCK : 0;
  if (blockIdx.x < nbl) {
    const int64_t base = blockIdx.x * DOT_PER_BLOCK + tid;
    V<K> acc = zero<K>();
    if (blockIdx.x * DOT_PER_BLOCK + DOT_PER_BLOCK <= n_local) {
      V<K> xs[DOT_LEAF], ys[DOT_LEAF];
#pragma unroll
      for (int j = 0; j < DOT_LEAF; ++j) {
        xs[j] = load<K>(x, sx, base + j * DOT_BLOCK);
        ys[j] = load<K>(y, sy, base + j * DOT_BLOCK);
      }
#pragma unroll
      for (int j = 0; j < DOT_LEAF; ++j)
        acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(xs[j], ys[j]));
    } else {
      for (int64_t t = base; t < n_local; t += DOT_BLOCK)
        acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(x, sx, t), load<K>(y, sy, t)));
    }
    V<K> r = block_tree<K, VAR>(acc, blockIdx.x * (int64_t)DOT_BLOCK, dot_partial_count(n_local));
    if (tid == 0) {
      for (int p = 0; p < world; ++p) {
        double* dst = peer_roots[p] + par_off + b0 + blockIdx.x;
#pragma unroll
        for (int c = 0; c < K; ++c) dst[c * nbt] = r.c[c];
      }
    }
  }
  if (tid == 0) is_last = atom_add_acq_rel_gpu(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  if (tid == 0) {
    *(volatile unsigned*)done = 0u;
    peer_publish_wait(peer_slot, my_slot, world, rank, e + 1ull, spin_limit, timeout);
  }
  __syncthreads();
  const double* roots = peer_roots[rank] + par_off;
  const int64_t groups = (nbt + DOT_BLOCK - 1) / DOT_BLOCK;
  V<K> fin;
  for (int64_t g = 0; g < groups; ++g) {
    V<K> v = zero<K>();
    const int64_t i = g * DOT_BLOCK + tid;
    if (i < nbt) {
#pragma unroll
      for (int c = 0; c < K; ++c) v.c[c] = __ldcg(roots + c * nbt + i);
    }
    __syncthreads();  // block_tree reuses its shared buffer
    V<K> r = block_tree<K, VAR>(v, g * (int64_t)DOT_BLOCK, nbt);
    if (tid == 0) {
#pragma unroll
      for (int c = 0; c < K; ++c) lvl[c][g] = r.c[c];
    }
    fin = r;
  }
  if (groups > 1) {
    __syncthreads();
    V<K> v = zero<K>();
    if (tid < groups) {
#pragma unroll
      for (int c = 0; c < K; ++c) v.c[c] = lvl[c][tid];
    }
    __syncthreads();
    fin = block_tree<K, VAR>(v, 0, groups);
  }
  if (tid == 0) {
    store<K>(out, 1, 0, fin);
    *(volatile unsigned long long*)epoch = e + 1ull;
  }
}

template <int K, int VAR>
struct DotPeerLaunch {
  static int run(const double* x, int64_t sx, const double* y, int64_t sy, int64_t n_local,
                 int64_t b0, int64_t nbt, double* const* peer_roots,
                 unsigned long long* const* peer_slot, unsigned long long* my_slot,
                 unsigned int* done, unsigned long long* epoch, int* timeout, int world, int rank,
                 long long spin_limit, double* out, cudaStream_t st) {
    const int64_t nbl = n_local > 0 ? ceil_div(n_local, DOT_PER_BLOCK) : 0;
    dot_peer_kernel<K, VAR><<<(unsigned)(nbl > 0 ? nbl : 1), DOT_BLOCK, 0, st>>>(
        x, sx, y, sy, n_local, b0, nbt, peer_roots, peer_slot, my_slot, done, epoch, timeout,
        world, rank, spin_limit, out);
    return launch_status();
  }
};

template <int K, int VAR>
struct DotPartialsLaunch {
  static int run(const double* x, int64_t sx, const double* y, int64_t sy, int64_t n,
                 double* partials, int64_t pstride, cudaStream_t st) {
    int64_t nb = ceil_div(n, DOT_PER_BLOCK);
    dot_partials_kernel<K, VAR><<<(unsigned)nb, DOT_BLOCK, 0, st>>>(x, sx, y, sy, n, partials,
                                                                    pstride);
    return launch_status();
  }
};

template <int K, int VAR>
struct TreeFoldLaunch {
  static int run(const double* partials, int64_t pstride, int64_t count, double* ws, double* out,
                 cudaStream_t st) {
    return fold_levels<K, VAR>(partials, pstride, count, ws, out, st);
  }
};

// ------------------------------------------------------------------ GEMV
// Exact order: thread per row, t ascending.
template <int K, int VAR>
__global__ void __launch_bounds__(128) gemv_exact_kernel(const double* __restrict__ A, int64_t lda,
                                                         int64_t sA, const double* __restrict__ x,
                                                         int64_t sx, double* __restrict__ y,
                                                         int64_t sy, int64_t m, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  V<K> acc = zero<K>();
  const double* row = A + i * lda;
  for (int64_t t = 0; t < n; ++t)
    acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(row, sA, t), load<K>(x, sx, t)));
  store<K>(y, sy, i, acc);
}

// Tree order: GEMV_P = 128 partials per row, four warps per row.  Partial u
// (lane l of warp w, u = 32w + l) folds t = u, u+128, u+256, ... ascending
// from exact zero; the partials combine by the in-place pairwise tree
// (strides 1..64, pairs valid while the partner index < min(n, 128)).
// (Measured on B200 at 2048^2: 128 partials beat 32 and 256.)
// Four elements are loaded ahead of their arithmetic so HBM latency
// overlaps the FP64 chain.
constexpr int GEMV_WARPS = 4;
constexpr int GEMV_P = 32 * GEMV_WARPS;
constexpr int GEMV_ROWS_PER_CTA = 2;

template <int K, int VAR, int WARPS = GEMV_WARPS, int RPC = GEMV_ROWS_PER_CTA, int D = 4>
__global__ void __launch_bounds__(32 * WARPS * RPC)
    gemv_tree_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                     const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                     int64_t m, int64_t n) {
  constexpr int P = 32 * WARPS;
  __shared__ double red[RPC][K][WARPS];
  const int lane = threadIdx.x & 31;
  const int warp = (threadIdx.x >> 5) % WARPS;
  const int slot = (threadIdx.x >> 5) / WARPS;
  const int64_t i = blockIdx.x * (int64_t)RPC + slot;
  const bool live = i < m;
  const double* row = A + (live ? i : 0) * lda;
  const int u = warp * 32 + lane;
  V<K> acc = zero<K>();
  int64_t t = u;
  for (; t + (D - 1) * P < n; t += D * P) {
    V<K> a[D], xv[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      a[d] = load<K>(row, sA, t + d * P);
      xv[d] = load<K>(x, sx, t + d * P);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a[d], xv[d]));
  }
  for (; t < n; t += P)
    acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(row, sA, t), load<K>(x, sx, t)));
  const int64_t valid = n < P ? n : P;
  // The pairwise tree, executed level by level over all RPC x P partials of
  // the CTA in shared memory: each level's pairs are spread over the whole
  // CTA, so a level costs ceil(pairs/32) warp-adds instead of one masked
  // warp-add per warp and level (same pairs, same order, same bits).
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
  (void)red;
  if (warp == 0 && lane == 0 && live) {
    V<K> r0;
#pragma unroll
    for (int c = 0; c < K; ++c) r0.c[c] = part[slot][c][0];
    store<K>(y, sy, i, r0);
  }
}

template <int K, int VAR>
struct GemvLaunch {
  static int run(const double* A, int64_t lda, int64_t sA, const double* x, int64_t sx, double* y,
                 int64_t sy, int64_t m, int64_t n, int order, cudaStream_t st) {
    if (order == MW_ORDER_EXACT) {
      gemv_exact_kernel<K, VAR><<<(unsigned)ceil_div(m, 128), 128, 0, st>>>(A, lda, sA, x, sx, y,
                                                                            sy, m, n);
    } else {
      // rows per CTA: 2 for DD/TD from 1536 rows, else 1 -- with fewer rows
      // (a row-block shard at 4-8 GPUs) two-row CTAs leave SMs idle
      // (scripts/gemv_msweep.py: TD 296 rows 10.0 -> 8.5 us); 1 for QD.
      // Same partials and tree either way: same bits.
      if (K != 4 && m >= 1536)
        gemv_tree_kernel<K, VAR, GEMV_WARPS, GEMV_ROWS_PER_CTA>
            <<<(unsigned)ceil_div(m, GEMV_ROWS_PER_CTA), 32 * GEMV_WARPS * GEMV_ROWS_PER_CTA, 0, st>>>(
                A, lda, sA, x, sx, y, sy, m, n);
      else
        gemv_tree_kernel<K, VAR, GEMV_WARPS, 1><<<(unsigned)m, 32 * GEMV_WARPS, 0, st>>>(
            A, lda, sA, x, sx, y, sy, m, n);
    }
    return launch_status();
  }
};

}  // namespace mw

using namespace mw;

static int variant_ok(int k, int variant) {
  if (k < 2 || k > 4) return MW_ERR_INVALID;
  return (variant == 0 || variant == 1) ? MW_OK : MW_ERR_INVALID;
}

extern "C" int64_t mw_dot_workspace(int k, int64_t n) {
  if (k < 2 || k > 4 || n < 0) return 0;
  int64_t nb = ceil_div(n, DOT_PER_BLOCK);
  if (nb <= 1) return 0;
  // ws[0]: single-launch ticket; then nb*k partials (+ fold levels)
  if (nb <= DOT_BLOCK) return 1 + nb * k;
  return 1 + nb * k + mw_tree_fold_workspace(k, nb);
}

extern "C" int64_t mw_tree_fold_workspace(int k, int64_t count) {
  if (k < 2 || k > 4 || count < 1) return 0;
  int64_t total = 0;
  for (int64_t c = ceil_div(count, DOT_BLOCK); c > 1; c = ceil_div(c, DOT_BLOCK)) total += c * k;
  return total;
}

extern "C" int64_t mw_dot_num_partials(int64_t n) { return n <= 0 ? 0 : ceil_div(n, DOT_PER_BLOCK); }

extern "C" int mw_dot(int k, int variant, const double* x, int64_t sx, const double* y, int64_t sy,
                      int64_t n, double* ws, double* out_dev, int order, void* stream) {
  return mw_dot_ex(k, variant, x, sx, y, sy, n, ws, out_dev, order, nullptr, stream);
}

extern "C" int mw_dot_ex(int k, int variant, const double* x, int64_t sx, const double* y,
                         int64_t sy, int64_t n, double* ws, double* out_dev, int order,
                         const mw_tuning* tune, void* stream) {
  int rc = variant_ok(k, variant);
  if (rc) return rc;
  mw_tuning t;
  if (!tuning_resolve(tune, &t)) return MW_ERR_INVALID;
  if (n < 0 || !out_dev || (n > 0 && (!x || !y || sx < n || sy < n))) return MW_ERR_INVALID;
  if (order != MW_ORDER_EXACT && order != MW_ORDER_TREE) return MW_ERR_INVALID;
  if (order == MW_ORDER_TREE && mw_dot_workspace(k, n) > 0 && !ws) return MW_ERR_INVALID;
  return dispatch<DotLaunch>(k, variant, x, sx, y, sy, n, ws, out_dev, order, t.dot_cluster,
                             as_stream(stream));
}

extern "C" int mw_dot_partials(int k, int variant, const double* x, int64_t sx, const double* y,
                               int64_t sy, int64_t n, double* partials, int64_t pstride,
                               void* stream) {
  int rc = variant_ok(k, variant);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!x || !y || !partials || sx < n || sy < n))) return MW_ERR_INVALID;
  if (n == 0) return MW_OK;
  if (pstride < mw_dot_num_partials(n)) return MW_ERR_INVALID;
  return dispatch<DotPartialsLaunch>(k, variant, x, sx, y, sy, n, partials, pstride,
                                     as_stream(stream));
}

extern "C" int mw_tree_fold(int k, int variant, const double* partials, int64_t pstride,
                            int64_t count, double* ws, double* out_dev, void* stream) {
  int rc = variant_ok(k, variant);
  if (rc) return rc;
  if (count < 1 || !partials || !out_dev || pstride < count) return MW_ERR_INVALID;
  if (mw_tree_fold_workspace(k, count) > 0 && !ws) return MW_ERR_INVALID;
  return dispatch<TreeFoldLaunch>(k, variant, partials, pstride, count, ws, out_dev,
                                  as_stream(stream));
}

extern "C" int mw_gemv(int k, int variant, const double* A, int64_t lda, int64_t sA,
                       const double* x, int64_t sx, double* y, int64_t sy, int64_t m, int64_t n,
                       int order, void* stream) {
  int rc = variant_ok(k, variant);
  if (rc) return rc;
  if (m < 0 || n < 0) return MW_ERR_INVALID;
  if (order != MW_ORDER_EXACT && order != MW_ORDER_TREE) return MW_ERR_INVALID;
  if (m == 0) return MW_OK;
  if (!A || !x || !y || lda < n || sy < m || sx < n) return MW_ERR_INVALID;
  if (n > 0 && sA < (m - 1) * lda + n) return MW_ERR_INVALID;
  return dispatch<GemvLaunch>(k, variant, A, lda, sA, x, sx, y, sy, m, n, order,
                              as_stream(stream));
}

// Sharded tree dot, exchange fused in (dot_peer_kernel).  x, y: this
// rank's slice (n_local elements, starting at global element 4096 * b0;
// only the last rank's slice may end ragged).  nbt: block roots over all
// ranks (ceil(n_total / 4096), <= 65536).  peer_roots: device array of
// world pointers to each rank's root buffer (2 parities x k planes x nbt);
// peer_slot / my_slot / done / epoch / timeout as for mw_dk_sweep_peer.
// out_dev (k doubles) receives the full dot on every rank.
extern "C" int mw_dot_peer(int k, int variant, const double* x, int64_t sx, const double* y,
                           int64_t sy, int64_t n_local, int64_t b0, int64_t nbt,
                           double* const* peer_roots, unsigned long long* const* peer_slot,
                           unsigned long long* my_slot, unsigned int* done,
                           unsigned long long* epoch, int* timeout, int world, int rank,
                           long long spin_limit, double* out_dev, void* stream) {
  int rc = variant_ok(k, variant);
  if (rc) return rc;
  if (world < 1 || rank < 0 || rank >= world || spin_limit < 1) return MW_ERR_INVALID;
  if (nbt < 1 || nbt > (int64_t)DOT_BLOCK * DOT_BLOCK || b0 < 0 || n_local < 0) return MW_ERR_INVALID;
  if (b0 + ceil_div(n_local, DOT_PER_BLOCK) > nbt) return MW_ERR_INVALID;
  if (n_local > 0 && (!x || !y || sx < n_local || sy < n_local)) return MW_ERR_INVALID;
  if (!peer_roots || !peer_slot || !my_slot || !done || !epoch || !timeout || !out_dev)
    return MW_ERR_INVALID;
  return dispatch<DotPeerLaunch>(k, variant, x, sx, y, sy, n_local, b0, nbt, peer_roots, peer_slot,
                                 my_slot, done, epoch, timeout, world, rank, spin_limit, out_dev,
                                 as_stream(stream));
}
