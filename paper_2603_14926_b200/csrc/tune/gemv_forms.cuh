// gemv_forms.cuh -- tuning harness only (not in libmwgpu.so): the round-2
// alternative forms of the tree-order GEMV (persistent shuffle tree, per-warp
// cp.async.cg ring, two partials per thread, one warp per row, dynamic row
// tickets).  All keep gemv_tree_kernel's partials and tree (bit-identical);
// none beat it (profiles/r02_gemv_*.txt).
#pragma once
#include "../common.cuh"

namespace mw {

// Persistent form of the same tree order (bit-identical with
// gemv_tree_kernel): a CTA holds SLOTS row slots of four warps; each slot
// walks rows blockIdx.x * SLOTS + slot, += gridDim.x * SLOTS.  Per row the
// 128 partials fold exactly as above; the tree's strides 1..16 pair lanes of
// one warp and run as warp shuffles (no barrier); the four warp roots go to
// shared memory (double-buffered by row parity) and ONE named barrier per
// row and slot hands them to a combiner warp (rotating over the four warps,
// so no warp waits on the combine every row), which applies strides 32 and
// 64.  The next row's first D elements are requested before the shuffle
// tree runs, so its HBM latency hides behind the tree.  With PIPE, every
// group's loads are issued before the previous group's arithmetic
// (register double buffer).
__device__ __forceinline__ void gemv_bar_sync(int id) {
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}

template <int K, int VAR, int SLOTS, int D, bool XPF = true, int MINB = 1>
__global__ void __launch_bounds__(128 * SLOTS, MINB)
    gemv_ptree_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                      const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                      int64_t m, int64_t n) {
  constexpr int P = 128;
  __shared__ double roots[2][SLOTS][K][4];
  const int lane = threadIdx.x & 31;
  const int warp = (threadIdx.x >> 5) & 3;
  const int slot = threadIdx.x >> 7;
  const int u = warp * 32 + lane;
  const int64_t valid = n < P ? n : P;
  const int64_t step = (int64_t)gridDim.x * SLOTS;
  int64_t i = (int64_t)blockIdx.x * SLOTS + slot;
  const bool full = (int64_t)u + (D - 1) * P < n;  // row has >= 1 full group for this lane
  V<K> a[D], xv[D];
  if (XPF && i < m && full) {  // the first group of the first row, loaded ahead
#pragma unroll
    for (int d = 0; d < D; ++d) {
      a[d] = load<K>(A + i * lda, sA, u + d * P);
      xv[d] = load<K>(x, sx, u + d * P);
    }
  }
  for (int it = 0; i < m; i += step, ++it) {
    const double* row = A + i * lda;
    V<K> acc = zero<K>();
    int64_t t = u;
    if (XPF) {
      if (full) {
        for (;;) {
#pragma unroll
          for (int d = 0; d < D; ++d) acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a[d], xv[d]));
          t += D * P;
          if (t + (D - 1) * P >= n) break;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            a[d] = load<K>(row, sA, t + d * P);
            xv[d] = load<K>(x, sx, t + d * P);
          }
        }
      }
    } else {
      for (; t + (D - 1) * P < n; t += D * P) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
          a[d] = load<K>(row, sA, t + d * P);
          xv[d] = load<K>(x, sx, t + d * P);
        }
#pragma unroll
        for (int d = 0; d < D; ++d) acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a[d], xv[d]));
      }
    }
    for (; t < n; t += P)
      acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(load<K>(row, sA, t), load<K>(x, sx, t)));
    if (XPF) {  // next row's first group, in flight during the tree
      const int64_t inext = i + step;
      if (inext < m && full) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
          a[d] = load<K>(A + inext * lda, sA, u + d * P);
          xv[d] = load<K>(x, sx, u + d * P);
        }
      }
    }
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const V<K> o = shfl_down<K>(acc, s);
      if ((lane & (2 * s - 1)) == 0 && u + s < valid) acc = Ops<K, VAR>::add(acc, o);
    }
    const int buf = it & 1;
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < K; ++c) roots[buf][slot][c][warp] = acc.c[c];
    }
    gemv_bar_sync(1 + slot);
    if (warp == (it & 3) && lane == 0) {
      V<K> r[4];
#pragma unroll
      for (int w = 0; w < 4; ++w)
#pragma unroll
        for (int c = 0; c < K; ++c) r[w].c[c] = roots[buf][slot][c][w];
      if (32 < valid) r[0] = Ops<K, VAR>::add(r[0], r[1]);
      if (96 < valid) r[2] = Ops<K, VAR>::add(r[2], r[3]);
      if (64 < valid) r[0] = Ops<K, VAR>::add(r[0], r[2]);
      store<K>(y, sy, i, r[0]);
    }
  }
}

// Tree-order GEMV with A streamed through a per-WARP shared-memory ring by
// 16-byte cp.async.cg (L2 only: A never enters L1, so x stays L1-resident):
// every warp keeps S-1 chunks of D elements x K planes in flight while it
// folds the current chunk from shared memory, so the loads of chunk c+1..
// never wait behind the arithmetic of chunk c (the register-prefetch forms
// get their next loads sunk below the fold by the compiler).  Same partials
// (partial u folds t = u, u+128, ...), same tree: bit-identical.
// Requires n % (128 D) == 0 and 16-byte aligned rows/planes (else the caller
// uses gemv_tree_kernel).
template <int K, int VAR, int D, int S>
__global__ void __launch_bounds__(128)
    gemv_cg_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                   const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                   int64_t m, int64_t n) {
  constexpr int P = 128;
  constexpr int SEG = K * D;  // 256-byte segments per chunk per warp
  extern __shared__ double gcg_ring[];  // [warp][S][K*D][32]
  __shared__ double roots[K][4];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int u = warp * 32 + lane;
  const int64_t i = blockIdx.x;
  const double* row = A + i * lda;
  double* ring = gcg_ring + (size_t)warp * S * SEG * 32;
  const int64_t nch = n / (D * P);
  auto issue = [&](int64_t ch) {
    double* st = ring + (size_t)(ch % S) * SEG * 32;
    // SEG segments of 32 doubles; each lane copies 16 bytes of two of them
#pragma unroll
    for (int q = 0; q < SEG / 2; ++q) {
      const int seg = 2 * q + (lane >> 4);
      const int c = seg / D, d = seg % D;
      const int off = (lane & 15) * 2;
      const double* src = row + c * sA + ch * (D * P) + d * P + warp * 32 + off;
      cp_async16(st + seg * 32 + off, src, 16);
    }
    if (SEG & 1) {
      const int seg = SEG - 1;
      const int c = seg / D, d = seg % D;
      if (lane < 16)
        cp_async16(st + seg * 32 + lane * 2, row + c * sA + ch * (D * P) + d * P + warp * 32 + lane * 2, 16);
    }
  };
#pragma unroll
  for (int p = 0; p < S - 1; ++p) {
    if (p < nch) issue(p);
    cp_async_commit();
  }
  V<K> acc = zero<K>();
  for (int64_t ch = 0; ch < nch; ++ch) {
    V<K> xv[D];
#pragma unroll
    for (int d = 0; d < D; ++d) xv[d] = load<K>(x, sx, ch * (D * P) + d * P + u);
    cp_async_wait<S - 2>();
    __syncwarp();
    const double* st = ring + (size_t)(ch % S) * SEG * 32;
    V<K> a[D];
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int c = 0; c < K; ++c) a[d].c[c] = st[(c * D + d) * 32 + lane];
    __syncwarp();  // every lane has read the stage before it is refilled
    if (ch + S - 1 < nch) issue(ch + S - 1);
    cp_async_commit();
#pragma unroll
    for (int d = 0; d < D; ++d) acc = Ops<K, VAR>::add(acc, Ops<K, VAR>::mul(a[d], xv[d]));
  }
  const int64_t valid = n < P ? n : P;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const V<K> o = shfl_down<K>(acc, s);
    if ((lane & (2 * s - 1)) == 0 && u + s < valid) acc = Ops<K, VAR>::add(acc, o);
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) roots[c][warp] = acc.c[c];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    V<K> r[4];
#pragma unroll
    for (int w = 0; w < 4; ++w)
#pragma unroll
      for (int c = 0; c < K; ++c) r[w].c[c] = roots[c][w];
    if (32 < valid) r[0] = Ops<K, VAR>::add(r[0], r[1]);
    if (96 < valid) r[2] = Ops<K, VAR>::add(r[2], r[3]);
    if (64 < valid) r[0] = Ops<K, VAR>::add(r[0], r[2]);
    store<K>(y, sy, i, r[0]);
  }
}

// Same partials and tree as gemv_tree_kernel (bit-identical), 64 threads per
// row: thread t folds partials t and t + 64 as two interleaved independent
// chains (ILP 2 within a row; each thread lives twice as long, half as many
// threads per row).  D elements of each chain loaded ahead.  RPC rows per CTA.
template <int K, int VAR, int D, int RPC>
__global__ void __launch_bounds__(64 * RPC)
    gemv_u2_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                   const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                   int64_t m, int64_t n) {
  constexpr int P = 128;
  __shared__ double part[RPC][K][P];
  const int t = threadIdx.x & 63;
  const int slot = threadIdx.x >> 6;
  const int64_t i = blockIdx.x * (int64_t)RPC + slot;
  const bool live = i < m;
  const double* row = A + (live ? i : 0) * lda;
  V<K> acc0 = zero<K>(), acc1 = zero<K>();
  int64_t e = t;  // chain 0 at e, chain 1 at e + 64
  for (; e + 64 + (D - 1) * P < n; e += D * P) {
    V<K> a0[D], x0[D], a1[D], x1[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      a0[d] = load<K>(row, sA, e + d * P);
      x0[d] = load<K>(x, sx, e + d * P);
      a1[d] = load<K>(row, sA, e + 64 + d * P);
      x1[d] = load<K>(x, sx, e + 64 + d * P);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      acc0 = Ops<K, VAR>::add(acc0, Ops<K, VAR>::mul(a0[d], x0[d]));
      acc1 = Ops<K, VAR>::add(acc1, Ops<K, VAR>::mul(a1[d], x1[d]));
    }
  }
  for (int64_t f = e; f < n; f += P)
    acc0 = Ops<K, VAR>::add(acc0, Ops<K, VAR>::mul(load<K>(row, sA, f), load<K>(x, sx, f)));
  for (int64_t f = e + 64; f < n; f += P)
    acc1 = Ops<K, VAR>::add(acc1, Ops<K, VAR>::mul(load<K>(row, sA, f), load<K>(x, sx, f)));
  const int64_t valid = n < P ? n : P;
#pragma unroll
  for (int c = 0; c < K; ++c) {
    part[slot][c][t] = acc0.c[c];
    part[slot][c][t + 64] = acc1.c[c];
  }
  __syncthreads();
  const int tid = threadIdx.x;
#pragma unroll 1
  for (int s = 1; s < P; s <<= 1) {
    const int per_row = P / (2 * s);
    for (int w = tid; w < RPC * per_row; w += 64 * RPC) {
      const int r = w / per_row, idx = 2 * s * (w % per_row);
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
  if (t == 0 && live) {
    V<K> r0;
#pragma unroll
    for (int c = 0; c < K; ++c) r0.c[c] = part[slot][c][0];
    store<K>(y, sy, i, r0);
  }
}

// Same 128 partials and tree (bit-identical), ONE warp per row: lane l folds
// partials l, l + 32, l + 64, l + 96 as four interleaved independent chains
// (ILP 4), so 2048 rows are 2048 warps -- one resident wave on 148 SMs, no
// CTA turnover.  Tree: strides 1..16 by shuffles inside each chain, stride
// 32 pairs chains (0,1) and (2,3), stride 64 pairs the results -- all in
// registers of one lane.  D elements of every chain loaded ahead.
template <int K, int VAR, int D, int WPC>
__global__ void __launch_bounds__(32 * WPC)
    gemv_w1_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                   const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                   int64_t m, int64_t n) {
  constexpr int P = 128;
  const int lane = threadIdx.x & 31;
  const int64_t i = blockIdx.x * (int64_t)WPC + (threadIdx.x >> 5);
  if (i >= m) return;
  const double* row = A + i * lda;
  V<K> acc[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c] = zero<K>();
  int64_t t = lane;  // chain c at t + 32c
  for (; t + 96 + (D - 1) * P < n; t += D * P) {
    V<K> a[D][4], xv[D][4];
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        a[d][c] = load<K>(row, sA, t + 32 * c + d * P);
        xv[d][c] = load<K>(x, sx, t + 32 * c + d * P);
      }
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c] = Ops<K, VAR>::add(acc[c], Ops<K, VAR>::mul(a[d][c], xv[d][c]));
  }
#pragma unroll
  for (int c = 0; c < 4; ++c)
    for (int64_t f = t + 32 * c; f < n; f += P)
      acc[c] = Ops<K, VAR>::add(acc[c], Ops<K, VAR>::mul(load<K>(row, sA, f), load<K>(x, sx, f)));
  const int64_t valid = n < P ? n : P;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const V<K> o = shfl_down<K>(acc[c], s);
      if ((lane & (2 * s - 1)) == 0 && 32 * c + lane + s < valid) acc[c] = Ops<K, VAR>::add(acc[c], o);
    }
  }
  if (lane == 0) {
    if (32 < valid) acc[0] = Ops<K, VAR>::add(acc[0], acc[1]);
    if (96 < valid) acc[2] = Ops<K, VAR>::add(acc[2], acc[3]);
    if (64 < valid) acc[0] = Ops<K, VAR>::add(acc[0], acc[2]);
    store<K>(y, sy, i, acc[0]);
  }
}

// Tree-order GEMV (bit-identical) with DYNAMIC row assignment: a
// persistent grid of 4-warp CTAs takes rows from a global ticket
// (atomicAdd), the next ticket fetched while the current row folds, so CTAs
// that finish early take more rows (no wave tail) and drift out of phase
// (no convoy of load bursts).  ctr[0] is the row ticket, ctr[1] counts
// finished CTAs; the last CTA re-arms both (graph-replay safe).
template <int K, int VAR, int D, int MINB>
__global__ void __launch_bounds__(128, MINB)
    gemv_dyn_kernel(const double* __restrict__ A, int64_t lda, int64_t sA,
                    const double* __restrict__ x, int64_t sx, double* __restrict__ y, int64_t sy,
                    int64_t m, int64_t n, unsigned int* __restrict__ ctr) {
  constexpr int P = 128;
  __shared__ double roots[2][K][4];
  __shared__ unsigned int nxt[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int u = tid;
  const int64_t valid = n < P ? n : P;
  if (tid == 0) nxt[0] = atomicAdd(&ctr[0], 1u);
  __syncthreads();
  int64_t i = nxt[0];
  for (int it = 0; i < m; ++it) {
    if (tid == 0) nxt[(it + 1) & 1] = atomicAdd(&ctr[0], 1u);
    const double* row = A + i * lda;
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
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const V<K> o = shfl_down<K>(acc, s);
      if ((lane & (2 * s - 1)) == 0 && u + s < valid) acc = Ops<K, VAR>::add(acc, o);
    }
    const int buf = it & 1;
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < K; ++c) roots[buf][c][warp] = acc.c[c];
    }
    __syncthreads();
    if (warp == (it & 3) && lane == 0) {
      V<K> r[4];
#pragma unroll
      for (int w = 0; w < 4; ++w)
#pragma unroll
        for (int c = 0; c < K; ++c) r[w].c[c] = roots[buf][c][w];
      if (32 < valid) r[0] = Ops<K, VAR>::add(r[0], r[1]);
      if (96 < valid) r[2] = Ops<K, VAR>::add(r[2], r[3]);
      if (64 < valid) r[0] = Ops<K, VAR>::add(r[0], r[2]);
      store<K>(y, sy, i, r[0]);
    }
    i = nxt[(it + 1) & 1];
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&ctr[1], 1u) == gridDim.x - 1) {
      ctr[0] = 0u;
      ctr[1] = 0u;
    }
  }
}

}  // namespace mw
