// dk.cu — one Durand-Kerner sweep in complex K-word arithmetic.
//
// Reference: roots.dk_iterate (roots.py:240-315).  For every root i
// (Jacobi: all read the frozen previous state):
//   numerator   acc = (1, 0); for c = n-1..0: acc = c_mul(acc, z_i);
//               acc = c_add(acc, (coef_c, 0))                (271-276)
//   denominator den = (1, 0); for j = 0..n-1: f = c_sub(z_i, z_j), the
//               j == i factor pinned to (1, 0); den = c_mul(den, f) (278-293)
//   step        mag = dr^2 + di^2; num = acc * conj(den);
//               step = num / mag (Newton reciprocal)          (297-303)
//   update      z_i - step; |step| = hypot(step_re0, step_im0) (305-308)
// with the local 3M complex product (roots.py:258-267) in the exact order;
// the tree order uses the four-multiplication product c_mul4 (cheaper in
// K-word arithmetic, see below).
//
// exact_order = 1: the numerator and the denominator of root i run on two
// lanes of different warps (independent chains, no block barrier between
// them: the denominator warp stages z_j with warp-level syncs), each
// replaying the reference order op for op; the tail follows on the
// numerator lane.  Bit exact.  Each step is one dependent chain (8-cycle
// FP64 latency, measured), so a sweep costs ~n steps of ~700 cycles (TD).  The reciprocal of mag is computed once and applied to both
// parts, which is the identical op sequence the reference runs twice.
//
// exact_order = 0 (tree; order defined below): 64 strided partial products
// for the denominator, 64 Horner blocks for the numerator scaled by powers
// of z^B, pairwise trees, complex products in the four-multiplication
// form: reassociated, within the accuracy contract of
// tests/test_dk_accuracy.py.  Default kernel (with a workspace):
// dk_treem_kernel, 4 roots per CTA, one chain per lane, trees packed level
// by level across the CTA's roots; dk_tree_kernel (3 warps per root) is the
// workspace-free form.  Both give the same bits.
#pragma once
#include <atomic>
#include <climits>
#include <cstring>

#include "common.cuh"
#include "peer.cuh"

namespace mw {

template <int K, int VAR>
struct Cx {
  V<K> re, im;
};

template <int K, int VAR>
__device__ __forceinline__ Cx<K, VAR> c_mul(const Cx<K, VAR>& a, const Cx<K, VAR>& b) {
  using O = Ops<K, VAR>;
  V<K> p1 = O::mul(a.re, b.re);
  V<K> p2 = O::mul(a.im, b.im);
  V<K> p3 = O::mul(O::add(a.re, a.im), O::add(b.re, b.im));
  Cx<K, VAR> r;
  r.re = O::add(p1, neg(p2));
  r.im = O::add(O::add(p3, neg(p1)), neg(p2));
  return r;
}

// Out-of-line copy for the tree kernel: its many call sites (chains, trees,
// scans, powers) would otherwise inline ~30 copies of a 400-1000
// instruction body and thrash the instruction cache (ncu: stall
// "no_instructions" dominated).  Same ops, same bits.
template <int K, int VAR>
__device__ __noinline__ Cx<K, VAR> c_mul_ol(const Cx<K, VAR> a, const Cx<K, VAR> b) {
  return c_mul<K, VAR>(a, b);
}

// The TREE order's complex product: four multiplications, re = ar br -
// ai bi, im = ar bi + ai br.  In K-word arithmetic an add costs more FP64
// instructions than a mul (TD 57 vs 39; QD 103 vs 106, with five adds
// against two), so 4 mul + 2 add is 270 (TD) / 630 (QD) FP64 instructions
// against 402 / 833 for the reference's 3M product, on a dependent path of
// one mul + one add instead of one mul + three adds -- and it is the
// componentwise more accurate product.  Only the tree order uses it (held
// to the reference by the accuracy contract, tests/test_dk_accuracy.py, and
// restated in oracle/mw_oracle.c c_mul4); the exact order keeps c_mul.
template <int K, int VAR>
__device__ __forceinline__ Cx<K, VAR> c_mul4(const Cx<K, VAR>& a, const Cx<K, VAR>& b) {
  using O = Ops<K, VAR>;
  V<K> p1 = O::mul(a.re, b.re);
  V<K> p2 = O::mul(a.im, b.im);
  V<K> p3 = O::mul(a.re, b.im);
  V<K> p4 = O::mul(a.im, b.re);
  Cx<K, VAR> r;
  r.re = O::add(p1, neg(p2));
  r.im = O::add(p3, p4);
  return r;
}
template <int K, int VAR>
__device__ __noinline__ Cx<K, VAR> c_mul4_ol(const Cx<K, VAR> a, const Cx<K, VAR> b) {
  return c_mul4<K, VAR>(a, b);
}

template <int K, int VAR>
__device__ __forceinline__ Cx<K, VAR> c_one() {
  Cx<K, VAR> r;
  r.re = constant<K>(1.0);
  r.im = zero<K>();
  return r;
}

// Peer-memory exchange for the root-sharded sweep: every
// rank keeps the FULL (2K, n) state twice (read buffer / write buffer,
// swapped each sweep); the lane that finishes root i stores its new K-word
// (re, im) straight into the write buffer of EVERY rank over NVLink
// (cudaIpc-mapped peer pointers), so the exchange overlaps the other
// roots' arithmetic instead of following the kernel as an all-gather.
// Completion: after a warp/CTA sync over its storing threads, one thread
// per CTA takes a ticket with a gpu-scope acq_rel atomic (cumulative: it
// releases the CTA's peer stores); the last CTA has thereby acquired every
// CTA's stores and publishes "sweep s done" to every rank as a monotonic
// per-source slot value (epoch * sweeps + s + 1) with st.release.sys,
// which is cumulative over all it has observed
// and then waits (ld.acquire.sys, bounded) until every source's slot on
// THIS rank reached the same value.  The kernel therefore ends only when
// the full next state has landed locally, so the next sweep's kernel reads
// it after an ordinary stream boundary.  One slot per source takes plain
// release stores (no remote atomics) and only ever grows, so nothing is
// reset between runs.  A wait that exceeds spin_limit sets *timeout and
// returns instead of hanging the GPU.  tests/test_peer_protocol.py checks
// the protocol (with the host's run-parity rule, dist.DKPeerGraph) under
// random interleavings.
struct DkPeers {
  double* const* out;              // [world] peer write buffers, (2K, n) planes, stride n
  unsigned long long* const* slot; // [world] peer slot arrays ([world] u64 each)
  unsigned long long* my_slot;     // this rank's slot array
  unsigned int* done;              // CTA completion ticket (self-resetting)
  unsigned long long* epoch;       // completed replays (advanced by the last sweep)
  int* timeout;                    // set to 1 when a wait gave up
  long long spin_limit;
  int world, rank, sweep, sweeps;
  // optional (any sweep, not only the peer form): max_bits[0] is raised
  // atomically to the bit pattern of every step_mag written -- the sweep's
  // max update (roots.py:308) -- and max_bits[1] to that of every new
  // root's |z'| = hypot(re0, im0) (the max |z| of dk_solve's test,
  // roots.py:336), with no separate reduction; both are >= 0, so the
  // unsigned bit order is the value order (NaN, as np.max, dominates)
  unsigned long long* max_bits;
};

__device__ __forceinline__ void dk_note_max(unsigned long long* max_bits, double m) {
  if (max_bits) atomicMax(max_bits, (unsigned long long)__double_as_longlong(m));
}

// Called by exactly one thread per CTA, after a sync over the CTA's
// storing threads.
static __device__ __noinline__ void dk_peer_ticket(const DkPeers& P) {
  if (atom_add_acq_rel_gpu(P.done, 1u) != gridDim.x - 1) return;
  *(volatile unsigned*)P.done = 0;  // the next launch in the stream starts from zero
  const unsigned long long e = *(volatile unsigned long long*)P.epoch;
  const unsigned long long v = e * (unsigned long long)P.sweeps + (unsigned long long)P.sweep + 1ull;
  peer_publish_wait(P.slot, P.my_slot, P.world, P.rank, v, P.spin_limit, P.timeout);
  if (P.sweep == P.sweeps - 1) *(volatile unsigned long long*)P.epoch = e + 1;
}

// Shared tail: step = acc * conj(den) / |den|^2, z - step (roots.py:297-308).
// PEER: the new value also goes to every other rank's write buffer.
template <int K, int VAR, bool PEER = false>
__device__ __forceinline__ void dk_tail(const Cx<K, VAR>& acc, const Cx<K, VAR>& den,
                                        const Cx<K, VAR>& z, double* zre_out, double* zim_out,
                                        int64_t so, double* step_mag, int64_t i,
                                        const DkPeers* P = nullptr) {
  using O = Ops<K, VAR>;
  V<K> mag = O::add(O::mul(den.re, den.re), O::mul(den.im, den.im));
  V<K> num_re = O::add(O::mul(acc.re, den.re), O::mul(acc.im, den.im));
  V<K> num_im = O::add(O::mul(acc.im, den.re), neg(O::mul(acc.re, den.im)));
  V<K> rcp = recip_newton<K, VAR>(mag);
  V<K> step_re = O::mul(num_re, rcp);
  V<K> step_im = O::mul(num_im, rcp);
  const V<K> nre = O::add(z.re, neg(step_re));
  const V<K> nim = O::add(z.im, neg(step_im));
  store<K>(zre_out, so, i, nre);
  store<K>(zim_out, so, i, nim);
  const double smag = hypot(step_re.c[0], step_im.c[0]);
  step_mag[i] = smag;
  if (P && P->max_bits) {
    dk_note_max(P->max_bits, smag);
    dk_note_max(P->max_bits + 1, hypot(nre.c[0], nim.c[0]));
  }
  if constexpr (PEER) {
    for (int p = 0; p < P->world; ++p) {
      if (p == P->rank) continue;
      store<K>(P->out[p], so, i, nre);
      store<K>(P->out[p] + (int64_t)K * so, so, i, nim);
    }
  }
}

constexpr int DK_EXACT_ROOTS = 32;  // lanes per role warp (two warps: num + den)
// Roots handled per CTA (mw_tuning.dk_exact_roots, <= 32; lanes beyond it
// idle; default 32, 16 and 8 measured 0.5-5 % slower).  Fewer roots per
// CTA spread the 2n sequential chains over more SM sub-partitions.
// mw_tuning.dk_exact_split = 1: split-pair exact kernel (dk_exact2_kernel)
// for TD and QD, 0: single-warp chains everywhere.  Measured (config 5,
// us/sweep, eager, single -> split): TD 353 -> 295 (one hand-off per step),
// QD 745 -> 575 (XP: p1, p2 handed over too); DD 165 -> 173, so DD stays
// single-warp.
constexpr int DK_SPLIT_MIN_K = 3;
constexpr int DK_CH = 128;          // roots staged in smem per chunk

template <int K, int VAR, bool PEER = false>
__global__ void __launch_bounds__(2 * DK_EXACT_ROOTS)
    dk_exact_kernel(const double* __restrict__ coeffs, int64_t sc, int64_t n,
                    const double* __restrict__ zre, const double* __restrict__ zim, int64_t sz,
                    int64_t i0, int64_t i1, double* __restrict__ zre_out,
                    double* __restrict__ zim_out, int64_t so, double* __restrict__ step_mag,
                    int* __restrict__ flag, int roots_per_cta, DkPeers peers = DkPeers{}) {
  using O = Ops<K, VAR>;
  __shared__ double zs[2][K][DK_CH];
  __shared__ double dx[2][K][DK_EXACT_ROOTS];
  const int lane = threadIdx.x & 31;
  const bool is_den = threadIdx.x >= 32;
  const int64_t i = i0 + (int64_t)blockIdx.x * roots_per_cta + lane;
  const bool live = lane < roots_per_cta && i < i1;

  Cx<K, VAR> z;
  z.re = live ? load<K>(zre, sz, i) : zero<K>();
  z.im = live ? load<K>(zim, sz, i) : zero<K>();
  Cx<K, VAR> acc = c_one<K, VAR>();

  // unroll 2 lets the scheduler overlap consecutive steps (TD: 1.15x);
  // QD's larger body does better rolled (register pressure)
  constexpr int UNR = K < 4 ? 2 : 1;
  if (!is_den) {
#pragma unroll UNR
    for (int64_t c = n - 1; c >= 0; --c) {
      acc = c_mul(acc, z);
      Cx<K, VAR> ci;
      ci.re = load<K>(coeffs, sc, c);
      ci.im = zero<K>();
      acc.re = O::add(acc.re, ci.re);
      acc.im = O::add(acc.im, ci.im);
    }
  }
  // denominator: the den warp alone stages z_j chunks (warp-level syncs, so
  // the numerator warp's Horner chain runs concurrently instead of waiting
  // at block barriers)
  if (is_den) {
    for (int64_t j0 = 0; j0 < n; j0 += DK_CH) {
      const int cnt = (int)((n - j0) < DK_CH ? (n - j0) : DK_CH);
      __syncwarp();
      for (int e = lane; e < K * cnt; e += 32) {
        const int c = e / cnt, jj = e % cnt;
        zs[0][c][jj] = zre[c * sz + j0 + jj];
        zs[1][c][jj] = zim[c * sz + j0 + jj];
      }
      __syncwarp();
#pragma unroll UNR
      for (int jj = 0; jj < cnt; ++jj) {
        const int64_t j = j0 + jj;
        Cx<K, VAR> zj, f;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          zj.re.c[c] = zs[0][c][jj];
          zj.im.c[c] = zs[1][c][jj];
        }
        f.re = O::add(z.re, neg(zj.re));
        f.im = O::add(z.im, neg(zj.im));
        if (j == i) f = c_one<K, VAR>();
        if (live && fabs(f.re.c[0]) + fabs(f.im.c[0]) == 0.0) {
          const long long key = (long long)j * n + i;
          atomicMin(flag, key > INT_MAX ? INT_MAX : (int)key);
        }
        acc = c_mul(acc, f);
      }
    }
  }
  __syncthreads();
  if (is_den) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      dx[0][c][lane] = acc.re.c[c];
      dx[1][c][lane] = acc.im.c[c];
    }
  }
  __syncthreads();
  if (!is_den && live) {
    Cx<K, VAR> den;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      den.re.c[c] = dx[0][c][lane];
      den.im.c[c] = dx[1][c][lane];
    }
    dk_tail<K, VAR, PEER>(acc, den, z, zre_out, zim_out, so, step_mag, i, &peers);
  }
  if constexpr (PEER) {
    if (!is_den) {
      __syncwarp();
      if (lane == 0) dk_peer_ticket(peers);
    }
  }
}

// ------------------------------------------------ exact order, split pairs
// The single-warp exact kernel above issues every op of a step from one
// warp; one warp sustains only ~1 FP64 instruction per 2.6-3.5 cycles on
// this code (csrc/tune/mw_latency.cu), so a QD step (~1000 instructions)
// is issue-bound well above its dependent-chain latency.  Here each chain
// runs on a PAIR of warps, lanes = roots, same ops in the same order
// (bit-exact), with ONE hand-off per step:
//   warp A (imaginary part): s = re + im, p3 = s * bsum, p1 = re * b.re,
//           p2 = im * b.im, im' = (p3 - p1) - p2 [+ 0]
//   warp B (real part):      p1, p2 (the same products, recomputed),
//           re' = (p1 - p2) [+ coef]
//   both write their new half to a step-parity slot, one 64-thread named
//   barrier, each reads the other's half.
// XP (QD): B hands p1, p2 to A through a second barrier instead (A's QD
// issue load would otherwise exceed the chain latency).
// Numerator pair = warps 0/1 (b = z, plus the reference's (coef, 0) add),
// denominator pair = warps 2/3 (b = f_j = z_i - z_j, j == i pinned to
// (1, 0); B forms f_{j+1} and bsum = f.re + f.im one step ahead and hands
// them to A through the slot).  Tail on warp 0 as before.
__device__ __forceinline__ void named_sync(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void named_arrive(int id) {
  asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory");
}

template <int K>
__device__ __forceinline__ void sm_put(double (*buf)[32], int lane, const V<K>& v) {
#pragma unroll
  for (int c = 0; c < K; ++c) buf[c][lane] = v.c[c];
}
template <int K>
__device__ __forceinline__ V<K> sm_get(const double (*buf)[32], int lane) {
  V<K> v;
#pragma unroll
  for (int c = 0; c < K; ++c) v.c[c] = buf[c][lane];
  return v;
}

template <int K, int VAR, bool PEER = false, bool XP = (K == 4)>
__global__ void __launch_bounds__(128)
    dk_exact2_kernel(const double* __restrict__ coeffs, int64_t sc, int64_t n,
                     const double* __restrict__ zre, const double* __restrict__ zim, int64_t sz,
                     int64_t i0, int64_t i1, double* __restrict__ zre_out,
                     double* __restrict__ zim_out, int64_t so, double* __restrict__ step_mag,
                     int* __restrict__ flag, int roots_per_cta, DkPeers peers = DkPeers{}) {
  using O = Ops<K, VAR>;
  // [pair][parity][K][lane]
  __shared__ double s_re[2][2][K][32], s_im[2][2][K][32];
  // denominator factor for the next step: f.re, f.im, f.re + f.im
  __shared__ double s_fr[2][K][32], s_fi[2][K][32], s_fs[2][K][32];
  // XP: B hands its p1, p2 to A (A skips two products, one more barrier)
  __shared__ double s_p1[2][K][32], s_p2[2][K][32];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int pair = warp >> 1;  // 0 numerator, 1 denominator
  const bool is_b = warp & 1;  // B: real part, A: imaginary part
  const int64_t i = i0 + (int64_t)blockIdx.x * roots_per_cta + lane;
  const bool live = lane < roots_per_cta && i < i1;
  const int bar = 1 + pair, bar_x = 3 + pair;

  Cx<K, VAR> z;
  z.re = live ? load<K>(zre, sz, i) : zero<K>();
  z.im = live ? load<K>(zim, sz, i) : zero<K>();

  // acc = (1, 0): B owns re, A owns im; the other half is read per step
  V<K> re = constant<K>(1.0), im = zero<K>();

  if (pair == 0) {
    // ---------------- numerator: for c = n-1..0: acc = acc*z; acc += (a_c, 0)
    const V<K> zsum = O::add(z.re, z.im);
    V<K> coef = load<K>(coeffs, sc, n - 1);
#pragma unroll 1
    for (int64_t st = 0; st < n; ++st) {
      const int q = (int)(st & 1);
      const int64_t c = n - 1 - st;
      if (is_b) {
        const V<K> ci = coef;
        if (c > 0) coef = load<K>(coeffs, sc, c - 1);
        const V<K> p1 = O::mul(re, z.re);
        const V<K> p2 = O::mul(im, z.im);
        if constexpr (XP) {
          sm_put<K>(s_p1[0], lane, p1);
          sm_put<K>(s_p2[0], lane, p2);
          named_arrive(bar_x);
        }
        re = O::add(O::add(p1, neg(p2)), ci);
        sm_put<K>(s_re[0][q], lane, re);
      } else {
        const V<K> p3 = O::mul(O::add(re, im), zsum);
        V<K> p1, p2;
        if constexpr (XP) {
          named_sync(bar_x);
          p1 = sm_get<K>(s_p1[0], lane);
          p2 = sm_get<K>(s_p2[0], lane);
        } else {
          p1 = O::mul(re, z.re);
          p2 = O::mul(im, z.im);
        }
        im = O::add(O::add(O::add(p3, neg(p1)), neg(p2)), zero<K>());
        sm_put<K>(s_im[0][q], lane, im);
      }
      named_sync(bar);
      if (is_b) im = sm_get<K>(s_im[0][q], lane);
      else re = sm_get<K>(s_re[0][q], lane);
    }
  } else {
    // ---------------- denominator: for j = 0..n-1: acc = acc * f_j
    auto factor = [&](int64_t j, const Cx<K, VAR>& zj) {
      Cx<K, VAR> g;
      g.re = O::add(z.re, neg(zj.re));
      g.im = O::add(z.im, neg(zj.im));
      if (j == i) g = c_one<K, VAR>();
      if (live && fabs(g.re.c[0]) + fabs(g.im.c[0]) == 0.0) {
        const long long key = (long long)j * n + i;
        atomicMin(flag, key > INT_MAX ? INT_MAX : (int)key);
      }
      return g;
    };
    Cx<K, VAR> f, zn;  // B: current factor and z_{j+1} (loaded a step ahead)
    V<K> fs;
    if (is_b) {
      zn.re = load<K>(zre, sz, 0);
      zn.im = load<K>(zim, sz, 0);
      f = factor(0, zn);
      fs = O::add(f.re, f.im);
      sm_put<K>(s_fr[0], lane, f.re);
      sm_put<K>(s_fi[0], lane, f.im);
      sm_put<K>(s_fs[0], lane, fs);
      if (n > 1) {
        zn.re = load<K>(zre, sz, 1);
        zn.im = load<K>(zim, sz, 1);
      }
    }
    named_sync(bar);
#pragma unroll 1
    for (int64_t j = 0; j < n; ++j) {
      const int q = (int)(j & 1);
      if (is_b) {
        const Cx<K, VAR> zj1 = zn;
        if (j + 2 < n) {
          zn.re = load<K>(zre, sz, j + 2);
          zn.im = load<K>(zim, sz, j + 2);
        }
        const V<K> p1 = O::mul(re, f.re);
        const V<K> p2 = O::mul(im, f.im);
        if constexpr (XP) {
          sm_put<K>(s_p1[1], lane, p1);
          sm_put<K>(s_p2[1], lane, p2);
          named_arrive(bar_x);
        }
        re = O::add(p1, neg(p2));
        sm_put<K>(s_re[1][q], lane, re);
        if (j + 1 < n) {
          f = factor(j + 1, zj1);
          sm_put<K>(s_fr[q ^ 1], lane, f.re);
          sm_put<K>(s_fi[q ^ 1], lane, f.im);
          sm_put<K>(s_fs[q ^ 1], lane, O::add(f.re, f.im));
        }
      } else {
        const V<K> fsum = sm_get<K>(s_fs[q], lane);
        const V<K> p3 = O::mul(O::add(re, im), fsum);
        V<K> p1, p2;
        if constexpr (XP) {
          named_sync(bar_x);
          p1 = sm_get<K>(s_p1[1], lane);
          p2 = sm_get<K>(s_p2[1], lane);
        } else {
          p1 = O::mul(re, sm_get<K>(s_fr[q], lane));
          p2 = O::mul(im, sm_get<K>(s_fi[q], lane));
        }
        im = O::add(O::add(p3, neg(p1)), neg(p2));
        sm_put<K>(s_im[1][q], lane, im);
      }
      named_sync(bar);
      if (is_b) im = sm_get<K>(s_im[1][q], lane);
      else re = sm_get<K>(s_re[1][q], lane);
    }
  }
  __syncthreads();
  if (warp == 0) {
    const int q = (int)((n - 1) & 1);
    if (live) {
      Cx<K, VAR> acc, den;
      acc.re = re;
      acc.im = im;
      den.re = sm_get<K>(s_re[1][q], lane);
      den.im = sm_get<K>(s_im[1][q], lane);
      dk_tail<K, VAR, PEER>(acc, den, z, zre_out, zim_out, so, step_mag, i, &peers);
    }
    if constexpr (PEER) {
      __syncwarp();
      if (lane == 0) dk_peer_ticket(peers);
    }
  }
}

// ----------------------------------------------------------- tree order
// DK_P = 64 partials per role.
//  denominator: partial u (u < 64) folds the factors
//    j = u, u+64, ... ascending from (1, 0) (j == i pinned to (1, 0));
//    with V = min(n, 64) partials: first v_l <- v_l * v_{l+32} (l < 32,
//    l + 32 < V), then the in-place pairwise tree over v_0..v_31 (strides
//    1..16, pair valid while the partner index < min(V, 32)).
//  numerator: the monic coefficients a_0..a_n (a_n = 1) split
//    into blocks of B = ceil((n+1)/64); block u = [uB, (u+1)B) is evaluated
//    by Horner from its top coefficient, scaled by w^u with w = z^B; the
//    terms combine like the denominator (t_l + t_{l+32} first, then the
//    pairwise tree over 32, validity against the number of blocks).
//    w = z^B by right-to-left square-and-multiply; w^u for u < 32 by a
//    Hillis-Steele product scan over the warp (x_l <- x_l * x_{l-s} for
//    s = 1, 2, 4, 8, 16 from x_0 = 1, x_l = w), and for u >= 32 as
//    (the same scan) * w^32, w^32 = five squarings of w.
constexpr int DK_P = 64;

template <int K, int VAR>
__device__ __forceinline__ Cx<K, VAR> shfl_cx(const Cx<K, VAR>& v, int s, bool up) {
  Cx<K, VAR> r;
#pragma unroll
  for (int c = 0; c < K; ++c) {
    r.re.c[c] = up ? __shfl_up_sync(0xffffffffu, v.re.c[c], s) : __shfl_down_sync(0xffffffffu, v.re.c[c], s);
    r.im.c[c] = up ? __shfl_up_sync(0xffffffffu, v.im.c[c], s) : __shfl_down_sync(0xffffffffu, v.im.c[c], s);
  }
  return r;
}

// Mapping: one CTA of three warps per root, one role each, so the three
// dependency chains run on different schedulers:
//   warp 0  denominator: lane l owns partials l and l+32 (two product chains)
//   warp 1  numerator:   lane l owns blocks l and l+32 (two Horner chains)
//   warp 2  powers:      w = z^B, w^32, the scan x_l = w^l and x_l * w^32,
//                        handed to warp 1 through shared memory.
// w = z^B by right-to-left square-and-multiply from (1, 0); w32 = five
// squarings of w (the tree order's definition, see above).
template <int K, int VAR>
__device__ __forceinline__ void dk_powers(const Cx<K, VAR>& z, int64_t B, Cx<K, VAR>& w,
                                          Cx<K, VAR>& w32, bool with_w32 = true) {
  w = c_one<K, VAR>();
  Cx<K, VAR> sq = z;
  for (int64_t e = B; e > 0; e >>= 1) {
    if (e & 1) w = c_mul4_ol(w, sq);
    if (e > 1) sq = c_mul4_ol(sq, sq);
  }
  w32 = w;
  if (!with_w32) return;
#pragma unroll 1
  for (int r = 0; r < 5; ++r) w32 = c_mul4_ol(w32, w32);
}

// One thread per root: w = z^B and (with_w32) w^32 for the tree sweep that
// follows (programmatic dependent launch: the sweep starts as soon as every
// CTA here has issued launch_dependents, and only its powers warps wait).
template <int K, int VAR>
__global__ void __launch_bounds__(128)
    dk_pow_kernel(const double* __restrict__ zre, const double* __restrict__ zim, int64_t sz,
                  int64_t n, int64_t i0, int64_t i1, double* __restrict__ wbuf, int64_t ws,
                  int with_w32) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= i1) return;
  const int64_t B = (n + 1 + DK_P - 1) / DK_P;
  Cx<K, VAR> z, w, w32;
  z.re = load<K>(zre, sz, i);
  z.im = load<K>(zim, sz, i);
  dk_powers<K, VAR>(z, B, w, w32, with_w32 != 0);
  const int64_t r = i - i0;
  store<K>(wbuf, ws, r, w.re);
  store<K>(wbuf + (int64_t)K * ws, ws, r, w.im);
  store<K>(wbuf + (int64_t)2 * K * ws, ws, r, w32.re);
  store<K>(wbuf + (int64_t)3 * K * ws, ws, r, w32.im);
}

// EXTPOW: w = z^B and w^32 come from dk_pow_kernel (lane = root, so no
// warp spends 10 complex products per root on a value all 32 lanes
// duplicate); the powers warp waits for it with griddepcontrol.wait while
// the denominator and Horner warps already run (programmatic dependent
// launch).  wbuf: 4K planes (w.re, w.im, w32.re, w32.im), plane stride
// ws, indexed by i - i0.
template <int K, int VAR, bool PEER = false, bool EXTPOW = false>
__global__ void __launch_bounds__(96)
    dk_tree_kernel(const double* __restrict__ coeffs, int64_t sc, int64_t n,
                   const double* __restrict__ zre, const double* __restrict__ zim, int64_t sz,
                   int64_t i0, int64_t i1, double* __restrict__ zre_out,
                   double* __restrict__ zim_out, int64_t so, double* __restrict__ step_mag,
                   int* __restrict__ flag, DkPeers peers, const double* __restrict__ wbuf,
                   int64_t ws) {
  using O = Ops<K, VAR>;
  __shared__ double den_s[2][K];
  __shared__ double pw[2][2][K][32];  // [lo/hi][re/im][c][lane]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t i = i0 + blockIdx.x;
  const int64_t B = (n + 1 + DK_P - 1) / DK_P;
  const int64_t nblocks = (n + 1 + B - 1) / B;
  Cx<K, VAR> z;
  z.re = load<K>(zre, sz, i);
  z.im = load<K>(zim, sz, i);
  Cx<K, VAR> p[2];
  if (warp == 0) {
    // ---- denominator partials u = lane and u = lane + 32
    Cx<K, VAR> v[2] = {c_one<K, VAR>(), c_one<K, VAR>()};
    for (int64_t j0 = lane; j0 < n; j0 += DK_P) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t j = j0 + 32 * h;
        if (j < n) {
          Cx<K, VAR> f;
          f.re = O::add(z.re, neg(load<K>(zre, sz, j)));
          f.im = O::add(z.im, neg(load<K>(zim, sz, j)));
          if (j == i) f = c_one<K, VAR>();
          if (fabs(f.re.c[0]) + fabs(f.im.c[0]) == 0.0) {
            const long long key = (long long)j * n + i;
            atomicMin(flag, key > INT_MAX ? INT_MAX : (int)key);
          }
          v[h] = c_mul4_ol(v[h], f);
        }
      }
    }
    const int64_t valid = n < DK_P ? n : DK_P;
    if (lane + 32 < valid) v[0] = c_mul4_ol(v[0], v[1]);
    const int64_t v32 = valid < 32 ? valid : 32;
#pragma unroll 1
    for (int s = 1; s < 32; s <<= 1) {
      Cx<K, VAR> o = shfl_cx(v[0], s, false);
      if ((lane & (2 * s - 1)) == 0 && lane + s < v32) v[0] = c_mul4_ol(v[0], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < K; ++c) {
        den_s[0][c] = v[0].re.c[c];
        den_s[1][c] = v[0].im.c[c];
      }
    }
  } else if (warp == 1) {
    // ---- numerator blocks u = lane and u = lane + 32 (two Horner chains)
    const int64_t lo0 = lane * B, lo1 = (lane + 32) * B;
    const int64_t hi0 = (lo0 + B < n + 1) ? lo0 + B : n + 1;
    const int64_t hi1 = (lo1 + B < n + 1) ? lo1 + B : n + 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t lo = h ? lo1 : lo0, hi = h ? hi1 : hi0;
      p[h].re = zero<K>();
      p[h].im = zero<K>();
      if (lo < hi) p[h].re = (hi - 1 == n) ? constant<K>(1.0) : load<K>(coeffs, sc, hi - 1);
    }
    for (int64_t d = 2; d <= B; ++d) {
      const int64_t c0 = hi0 - d, c1 = hi1 - d;
      if (c0 >= lo0) {
        p[0] = c_mul4_ol(p[0], z);
        p[0].re = O::add(p[0].re, load<K>(coeffs, sc, c0));
      }
      if (c1 >= lo1) {
        p[1] = c_mul4_ol(p[1], z);
        p[1].re = O::add(p[1].re, load<K>(coeffs, sc, c1));
      }
    }
  } else {
    // ---- powers: w = z^B, w^32, x_l = w^l (scan), x_l * w^32
    Cx<K, VAR> w, w32;
    if constexpr (EXTPOW) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      const int64_t r = i - i0;
      w.re = load<K>(wbuf, ws, r);
      w.im = load<K>(wbuf + (int64_t)K * ws, ws, r);
      w32.re = load<K>(wbuf + (int64_t)2 * K * ws, ws, r);
      w32.im = load<K>(wbuf + (int64_t)3 * K * ws, ws, r);
    } else {
      dk_powers<K, VAR>(z, B, w, w32);
    }
    Cx<K, VAR> x = lane == 0 ? c_one<K, VAR>() : w;
#pragma unroll 1
    for (int s = 1; s < 32; s <<= 1) {
      Cx<K, VAR> o = shfl_cx(x, s, true);
      if (lane >= s) x = c_mul4_ol(x, o);
    }
    Cx<K, VAR> xh = c_mul4_ol(x, w32);
#pragma unroll
    for (int c = 0; c < K; ++c) {
      pw[0][0][c][lane] = x.re.c[c];
      pw[0][1][c][lane] = x.im.c[c];
      pw[1][0][c][lane] = xh.re.c[c];
      pw[1][1][c][lane] = xh.im.c[c];
    }
  }
  __syncthreads();
  if (warp != 1) return;
  Cx<K, VAR> t[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    Cx<K, VAR> x;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      x.re.c[c] = pw[h][0][c][lane];
      x.im.c[c] = pw[h][1][c][lane];
    }
    t[h] = c_mul4_ol(p[h], x);
  }
  if (lane + 32 < nblocks) {
    t[0].re = O::add(t[0].re, t[1].re);
    t[0].im = O::add(t[0].im, t[1].im);
  }
  const int64_t b32 = nblocks < 32 ? nblocks : 32;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    Cx<K, VAR> o = shfl_cx(t[0], s, false);
    if ((lane & (2 * s - 1)) == 0 && lane + s < b32) {
      t[0].re = O::add(t[0].re, o.re);
      t[0].im = O::add(t[0].im, o.im);
    }
  }
  if (lane == 0) {
    Cx<K, VAR> den;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      den.re.c[c] = den_s[0][c];
      den.im.c[c] = den_s[1][c];
    }
    dk_tail<K, VAR, PEER>(t[0], den, z, zre_out, zim_out, so, step_mag, i, &peers);
    if constexpr (PEER) dk_peer_ticket(peers);
  }
}

// ------------------------------------------- tree order, R roots per CTA
// The same tree order (and the same bits) as dk_tree_kernel, mapped for
// throughput: a CTA owns R roots and 5R warps —
//   warps [0, 2R)   denominator: warp (r, h), lane l folds partial l + 32h
//   warps [2R, 4R)  numerator:   warp (r, h), lane l runs block l + 32h
//   warps [4R, 5R)  powers:      the scan x_l = w^l and x_l * w^32 of root r
// so every lane carries ONE chain (4 chain warps per root instead of 2
// two-chain warps: more warps to hide the FP64 latency, half the registers
// per chain), and the pairwise trees run level by level over all R roots
// of the CTA in shared memory: a level costs ceil(R * pairs / 32) warp
// products instead of one 32-lane product per root in which most lanes are
// masked.  The per-root tail runs on lane r of warp 2R.
template <int K>
__host__ __device__ constexpr size_t dk_treem_smem(int R) {
  // den + num partials [R][64] complex, powers [R][2][2][K][32], and for
  // R = 1 the w^32 hand-off [2K][64] (slot 0)
  return (size_t)R * 64 * 2 * K * sizeof(double) * 2 + (size_t)R * 2 * 2 * K * 32 * sizeof(double) +
         (R == 1 ? (size_t)2 * K * 64 * sizeof(double) : 0);
}

template <int K, int VAR>
__device__ __forceinline__ void cx_put(double* base, int idx, const Cx<K, VAR>& v) {
  // layout [re/im][c][64] per root
#pragma unroll
  for (int c = 0; c < K; ++c) {
    base[c * 64 + idx] = v.re.c[c];
    base[(K + c) * 64 + idx] = v.im.c[c];
  }
}
template <int K, int VAR>
__device__ __forceinline__ Cx<K, VAR> cx_get(const double* base, int idx) {
  Cx<K, VAR> v;
#pragma unroll
  for (int c = 0; c < K; ++c) {
    v.re.c[c] = base[c * 64 + idx];
    v.im.c[c] = base[(K + c) * 64 + idx];
  }
  return v;
}

// Warps per CTA: 5R, plus (R = 1) a w^32 warp, so that the five squarings
// w -> w^32 run beside the scan instead of before it: with one root per
// CTA the powers path, not the FP64 pipe, bounds the sweep (measured,
// scripts/time_dk_shard.py: TD 18.6 -> 17.2, QD 36.4 -> 32.5 us at 64
// roots; with 2 roots per CTA the extra warps cost more than they save).
template <int R>
__host__ __device__ constexpr int dk_treem_warps() { return R == 1 ? 8 : 5 * R; }

// Phase timestamps for the tuning harness only (csrc/tune/dk_phase.cu
// defines MW_DK_PROFILE); compiled out of the product.
#ifdef MW_DK_PROFILE
__device__ unsigned long long g_dk_prof[4096][12];
#define MW_DK_MARK(slot)                                                              \
  do {                                                                                \
    unsigned long long t_;                                                            \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
    if (blockIdx.x < 4096) g_dk_prof[blockIdx.x][slot] = t_;                          \
  } while (0)
#else
#define MW_DK_MARK(slot) \
  do {                   \
  } while (0)
#endif

__device__ __forceinline__ void bar_sync_n(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
template <int K, int VAR>
__device__ __forceinline__ V<K> shfl_v(const V<K>& v, int src) {
  V<K> r;
#pragma unroll
  for (int c = 0; c < K; ++c) r.c[c] = __shfl_sync(0xffffffffu, v.c[c], src);
  return r;
}
template <int K>
__device__ __forceinline__ V<K> sel(bool t, const V<K>& a, const V<K>& b) {
  V<K> r;
#pragma unroll
  for (int c = 0; c < K; ++c) r.c[c] = t ? a.c[c] : b.c[c];
  return r;
}
// One complex product of a denominator tree level on FOUR adjacent lanes:
// b[idx] <- b[idx] * b[idx + s] with idx = 2 s pair (pair < 0: lanes idle;
// pairs whose partner index is >= v32 pass through).  Lane roles 0..3 form
// p1 = a.re c.re, p2 = a.im c.im, p3 = a.re c.im, p4 = a.im c.re (one SIMD
// mul), then role 0 forms re = p1 - p2 and role 2 im = p3 + p4 (one SIMD
// add): c_mul4's operations on c_mul4's operands.
template <int K, int VAR>
__device__ __forceinline__ void dk_den_pair4(double* b, int s, int pair, int v32) {
  using O = Ops<K, VAR>;
  const int lane = threadIdx.x & 31, role = lane & 3;
  const int idx = pair < 0 ? 0 : 2 * s * pair;
  const bool act = pair >= 0 && idx + s < v32;
  // this role's factor of a (re for roles 0, 2) and of c (re for roles 0, 3)
  const double* pa = b + ((role & 1) ? K : 0) * 64 + idx;
  const double* pc = b + ((role == 0 || role == 3) ? 0 : K) * 64 + idx + s;
  V<K> fa, fc;
#pragma unroll
  for (int c = 0; c < K; ++c) {
    fa.c[c] = pa[c * 64];
    fc.c[c] = pc[c * 64];
  }
  const V<K> p = O::mul(fa, fc);
  const V<K> nxt = shfl_v<K, VAR>(p, lane + 1);
  const V<K> q = O::add(p, sel<K>(role == 0, neg(nxt), nxt));
  __syncwarp();  // every lane has read its operands before b[idx] is replaced
  if (act && (role == 0 || role == 2)) {
#pragma unroll
    for (int c = 0; c < K; ++c) b[((role >> 1) * K + c) * 64 + idx] = q.c[c];
  }
}

template <int K, int VAR, int R, bool PEER = false>
__global__ void __launch_bounds__(32 * dk_treem_warps<R>(), R == 2 ? 2 : 1)
    dk_treem_kernel(const double* __restrict__ coeffs, int64_t sc, int64_t n,
                    const double* __restrict__ zre, const double* __restrict__ zim, int64_t sz,
                    int64_t i0, int64_t i1, double* __restrict__ zre_out,
                    double* __restrict__ zim_out, int64_t so, double* __restrict__ step_mag,
                    int* __restrict__ flag, DkPeers peers, const double* __restrict__ wbuf,
                    int64_t ws) {
  using O = Ops<K, VAR>;
  extern __shared__ __align__(16) double dsm[];
  double* den_s = dsm;                             // [R][2K][64]
  double* num_s = den_s + (size_t)R * 2 * K * 64;  // [R][2K][64]
  double* pw = num_s + (size_t)R * 2 * K * 64;     // [R][2 (lo/hi)][2K][32]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t B = (n + 1 + DK_P - 1) / DK_P;
  const int64_t nblocks = (n + 1 + B - 1) / B;
  const int64_t valid = n < DK_P ? n : DK_P;
  const int v32 = (int)(valid < 32 ? valid : 32);
  const int b32 = (int)(nblocks < 32 ? nblocks : 32);
  const int64_t rbase = i0 + (int64_t)blockIdx.x * R;
  // role of this warp in the first phase; with one root per CTA the powers
  // and w^32 warps sit on sub-partitions 2 and 3 (warps 6, 7; 4 and 5 idle)
  // so the denominator warps (sub-partitions 0, 1: the longest chains)
  // issue alone
  const int rw = R == 1 ? (warp < 4 ? warp : warp == 6 ? 4 : warp == 7 ? 5 : 99) : warp;
  if (threadIdx.x == 0) MW_DK_MARK(0);

  if (rw < 2 * R) {
    // ---- denominator partial u = lane + 32h of root r
    const int r = warp >> 1, h = warp & 1;
    const int64_t i = rbase + r;
    const int u = lane + 32 * h;
    Cx<K, VAR> v = c_one<K, VAR>();
    if (i < i1) {
      Cx<K, VAR> z;
      z.re = load<K>(zre, sz, i);
      z.im = load<K>(zim, sz, i);
      for (int64_t j = u; j < n; j += DK_P) {
        Cx<K, VAR> f;
        f.re = O::add(z.re, neg(load<K>(zre, sz, j)));
        f.im = O::add(z.im, neg(load<K>(zim, sz, j)));
        if (j == i) f = c_one<K, VAR>();
        if (fabs(f.re.c[0]) + fabs(f.im.c[0]) == 0.0) {
          const long long key = (long long)j * n + i;
          atomicMin(flag, key > INT_MAX ? INT_MAX : (int)key);
        }
        v = c_mul4<K, VAR>(v, f);  // inlined: the two chain sites are the hot loops
      }
    }
    cx_put<K, VAR>(den_s + (size_t)r * 2 * K * 64, u, v);
    if (threadIdx.x == 0) MW_DK_MARK(1);
  } else if (rw < 4 * R) {
    // ---- numerator block u = lane + 32h of root r (Horner from its top)
    const int r = (warp - 2 * R) >> 1, h = warp & 1;
    const int64_t i = rbase + r;
    const int u = lane + 32 * h;
    Cx<K, VAR> p;
    p.re = zero<K>();
    p.im = zero<K>();
    if (i < i1) {
      Cx<K, VAR> z;
      z.re = load<K>(zre, sz, i);
      z.im = load<K>(zim, sz, i);
      const int64_t lo = u * B;
      const int64_t hi = (lo + B < n + 1) ? lo + B : n + 1;
      if (lo < hi) p.re = (hi - 1 == n) ? constant<K>(1.0) : load<K>(coeffs, sc, hi - 1);
      for (int64_t c = hi - 2; c >= lo; --c) {
        p = c_mul4<K, VAR>(p, z);
        p.re = O::add(p.re, load<K>(coeffs, sc, c));
        // (the real coefficient is added to the real part only: the tree
        // order does not add the reference's (coef, 0) zero imaginary part)
      }
    }
    cx_put<K, VAR>(num_s + (size_t)r * 2 * K * 64, u, p);
    if (threadIdx.x == 64 * R) MW_DK_MARK(2);
  } else if (rw < 5 * R) {
    // ---- powers of root r: x_l = w^l (Hillis-Steele scan), x_l * w^32
    const int r = rw - 4 * R;
    const int64_t i = rbase + r;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (rw == 4 * R && lane == 0) MW_DK_MARK(3);
    Cx<K, VAR> w = c_one<K, VAR>(), w32 = c_one<K, VAR>();
    if (i < i1) {
      const int64_t q = i - i0;
      w.re = load<K>(wbuf, ws, q);
      w.im = load<K>(wbuf + (int64_t)K * ws, ws, q);
      if constexpr (R > 1) {
        w32.re = load<K>(wbuf + (int64_t)2 * K * ws, ws, q);
        w32.im = load<K>(wbuf + (int64_t)3 * K * ws, ws, q);
      }
    }
    Cx<K, VAR> x = lane == 0 ? c_one<K, VAR>() : w;
#pragma unroll 1
    for (int s = 1; s < 32; s <<= 1) {
      Cx<K, VAR> o = shfl_cx(x, s, true);
      if (lane >= s) x = c_mul4_ol(x, o);
    }
    if constexpr (R == 1) {
      named_sync(1 + r);  // w^32 from warp 5R + r
      w32 = cx_get<K, VAR>(pw + (size_t)R * 2 * 2 * K * 32 + (size_t)r * 2 * K * 64, 0);
    }
    const Cx<K, VAR> xh = c_mul4_ol(x, w32);
    if (rw == 4 * R && lane == 0) MW_DK_MARK(4);
    double* pr = pw + (size_t)r * 2 * 2 * K * 32;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      pr[(0 * 2 * K + c) * 32 + lane] = x.re.c[c];
      pr[(0 * 2 * K + K + c) * 32 + lane] = x.im.c[c];
      pr[(1 * 2 * K + c) * 32 + lane] = xh.re.c[c];
      pr[(1 * 2 * K + K + c) * 32 + lane] = xh.im.c[c];
    }
  } else if (R == 1 && rw == 5) {
    // ---- w^32 of root r: five squarings of w (beside the scan)
    const int r = rw - 5 * R;
    const int64_t i = rbase + r;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    Cx<K, VAR> w32 = c_one<K, VAR>();
    if (i < i1) {
      const int64_t q = i - i0;
      w32.re = load<K>(wbuf, ws, q);
      w32.im = load<K>(wbuf + (int64_t)K * ws, ws, q);
#pragma unroll 1
      for (int t = 0; t < 5; ++t) w32 = c_mul4_ol(w32, w32);
    }
    if (lane == 0) cx_put<K, VAR>(pw + (size_t)R * 2 * 2 * K * 32 + (size_t)r * 2 * K * 64, 0, w32);
    named_sync(1 + r);
  }
  __syncthreads();

  if (threadIdx.x == 0) MW_DK_MARK(5);
  // t_u = p_u * x_u (numerator warps); denominator level A (v_l * v_{l+32})
  if (warp < 2 * R) {
    const int tau = threadIdx.x;  // < 64R: first 32R threads act
    if (tau < 32 * R) {
      const int r = tau >> 5, l = tau & 31;
      if (l + 32 < valid) {
        double* b = den_s + (size_t)r * 2 * K * 64;
        cx_put<K, VAR>(b, l, c_mul4_ol(cx_get<K, VAR>(b, l), cx_get<K, VAR>(b, l + 32)));
      }
    }
  } else if (warp < 4 * R) {
    const int r = (warp - 2 * R) >> 1, h = warp & 1;
    const int u = lane + 32 * h;
    double* b = num_s + (size_t)r * 2 * K * 64;
    const double* pr = pw + ((size_t)r * 2 + h) * 2 * K * 32;
    Cx<K, VAR> x;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      x.re.c[c] = pr[c * 32 + lane];
      x.im.c[c] = pr[(K + c) * 32 + lane];
    }
    cx_put<K, VAR>(b, u, c_mul4_ol(cx_get<K, VAR>(b, u), x));
  }
  __syncthreads();

  if (threadIdx.x == 0) MW_DK_MARK(6);
  // The two trees run decoupled and almost barrier-free.
  //  denominator (32 values per root after level A): every complex product
  //    runs on FOUR adjacent lanes (dk_den_pair4: the muls p1..p4 of c_mul4
  //    as one SIMD mul, then re = p1 - p2 and im = p3 + p4 as one SIMD add
  //    -- the same operations on the same operands, so the same bits).
  //    Stride 1 has 16 pairs per root = 64 lanes = the root's two
  //    denominator warps; one named barrier over the denominator warps;
  //    strides 2..16 have <= 8 pairs = one warp per root, so they follow
  //    each other under warp-level syncs only.
  //  numerator (64 terms per root): one warp per root adds t_l + t_{l+32}
  //    from shared memory and runs strides 1..16 as warp shuffles.
  if (warp < 2 * R) {
    const int r = warp >> 1;
    double* b = den_s + (size_t)r * 2 * K * 64;
    dk_den_pair4<K, VAR>(b, 1, (warp & 1) * 8 + (lane >> 2), v32);
    bar_sync_n(14, 64 * R);
    // (the one warp per root is picked so that the CTA's tree warps --
    // denominator and numerator -- spread over the four sub-partitions:
    // they are latency bound and would otherwise share two of them)
    if ((warp & 1) == ((r >> 1) & 1)) {
#pragma unroll 1
      for (int s = 2; s < 32; s <<= 1) {
        dk_den_pair4<K, VAR>(b, s, (lane >> 2) < 16 / s ? (lane >> 2) : -1, v32);
        __syncwarp();
      }
    }
  } else if (warp < 4 * R && (warp & 1) == 1 - ((((warp - 2 * R) >> 1) >> 1) & 1)) {
    const int r = (warp - 2 * R) >> 1;
    double* b = num_s + (size_t)r * 2 * K * 64;
    const int lim = (int)(nblocks < 64 ? nblocks : 64);
    Cx<K, VAR> t = cx_get<K, VAR>(b, lane);
    if (lane + 32 < lim) {
      const Cx<K, VAR> o = cx_get<K, VAR>(b, lane + 32);
      t.re = O::add(t.re, o.re);
      t.im = O::add(t.im, o.im);
    }
#pragma unroll 1
    for (int s = 1; s < 32; s <<= 1) {
      const Cx<K, VAR> o = shfl_cx(t, s, false);
      if ((lane & (2 * s - 1)) == 0 && lane + s < b32) {
        t.re = O::add(t.re, o.re);
        t.im = O::add(t.im, o.im);
      }
    }
    if (lane == 0) cx_put<K, VAR>(b, 0, t);
  }
  __syncthreads();

  if (threadIdx.x == 0) MW_DK_MARK(7);
  // Tail (dk_tail's ops, roots.py:297-308) split over two warps, lane r =
  // root r: warp 2R forms |den|^2 and its Newton reciprocal (the dependent
  // chain), warp 2R+1 meanwhile forms the numerator acc * conj(den); after
  // one hand-off each applies the reciprocal to its half and stores it.
  if (warp == 2 * R || warp == 2 * R + 1) {
    const bool chain = warp == 2 * R;
    const int64_t i = rbase + lane;
    const bool act = lane < R && i < i1;
    double* my = pw + (size_t)(lane < R ? lane : 0) * (3 * K + 2);  // num_re, num_im, rcp, step_im0, z'_im0
    double nz0 = 0.0;
    Cx<K, VAR> z, acc, den;
    V<K> num, step;
    if (act) {
      z.re = load<K>(zre, sz, i);
      z.im = load<K>(zim, sz, i);
      acc = cx_get<K, VAR>(num_s + (size_t)lane * 2 * K * 64, 0);
      den = cx_get<K, VAR>(den_s + (size_t)lane * 2 * K * 64, 0);
      if (chain) {
        const V<K> mag = O::add(O::mul(den.re, den.re), O::mul(den.im, den.im));
        const V<K> rcp = recip_newton<K, VAR>(mag);
#pragma unroll
        for (int c = 0; c < K; ++c) my[2 * K + c] = rcp.c[c];
      } else {
        const V<K> num_re = O::add(O::mul(acc.re, den.re), O::mul(acc.im, den.im));
        const V<K> num_im = O::add(O::mul(acc.im, den.re), neg(O::mul(acc.re, den.im)));
#pragma unroll
        for (int c = 0; c < K; ++c) {
          my[c] = num_re.c[c];
          my[K + c] = num_im.c[c];
        }
      }
    }
    bar_sync_n(12, 64);
    if (act) {
      V<K> rcp;
#pragma unroll
      for (int c = 0; c < K; ++c) {
        rcp.c[c] = my[2 * K + c];
        num.c[c] = my[(chain ? 0 : K) + c];
      }
      step = O::mul(num, rcp);
      const V<K> nz = O::add(chain ? z.re : z.im, neg(step));
      nz0 = nz.c[0];
      double* outp = chain ? zre_out : zim_out;
      store<K>(outp, so, i, nz);
      if constexpr (PEER) {
        for (int p = 0; p < peers.world; ++p) {
          if (p == peers.rank) continue;
          store<K>(peers.out[p] + (chain ? 0 : (int64_t)K * so), so, i, nz);
        }
      }
      if (!chain) {
        my[3 * K] = step.c[0];
        my[3 * K + 1] = nz0;
      }
    }
    bar_sync_n(12, 64);
    if (chain) {
      if (act) {
        const double smag = hypot(step.c[0], my[3 * K]);
        step_mag[i] = smag;
        if (peers.max_bits) {
          dk_note_max(peers.max_bits, smag);
          dk_note_max(peers.max_bits + 1, hypot(nz0, my[3 * K + 1]));
        }
      }
      if (lane == 0) MW_DK_MARK(8);
      if constexpr (PEER) {
        __syncwarp();
        if (lane == 0) dk_peer_ticket(peers);
      }
    }
  }
}

// Roots per CTA of the tree sweep (mw_tuning.dk_tree_roots): 0 = the
// 3-warp single-root kernel (dk_tree_kernel), 1, 2 or 4 =
// dk_treem_kernel<R>, -1 (default) = by shard size (4 from 512 roots, 2
// from 256, else 1).  Results are identical.

// dk_treem_kernel<R> as a programmatic dependent launch after dk_pow_kernel
// (plain stream order where that is unsupported).
template <int K, int VAR, bool PEER, int R>
static int dk_treem_launch(const double* coeffs, int64_t sc, int64_t n, const double* zre,
                           const double* zim, int64_t sz, int64_t i0, int64_t i1, double* zre_out,
                           double* zim_out, int64_t so, double* step_mag, int* flag, DkPeers peers,
                           double* ws, cudaStream_t st) {
  const int64_t cnt = i1 - i0;
  const size_t smem = dk_treem_smem<K>(R);
  auto kern = dk_treem_kernel<K, VAR, R, PEER>;
  static std::atomic<bool> attr_set[64];  // per instantiation and device; idempotent, race-free
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  const unsigned grid = (unsigned)((cnt + R - 1) / R);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32 * dk_treem_warps<R>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, coeffs, sc, n, zre, zim, sz, i0, i1, zre_out,
                                     zim_out, so, step_mag, flag, peers, (const double*)ws, cnt);
  if (e == cudaErrorNotSupported) {
    (void)cudaGetLastError();
    kern<<<grid, 32 * dk_treem_warps<R>(), smem, st>>>(coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so,
                                      step_mag, flag, peers, (const double*)ws, cnt);
    return launch_status();
  }
  if (e != cudaSuccess) return (int)e;
  return launch_status();
}

// Tree sweep launch: with a workspace (4K doubles per root) the powers come
// from dk_pow_kernel and the sweep is a programmatic dependent launch;
// without one the powers warp computes them itself.  Same bits.
template <int K, int VAR, bool PEER>
int dk_tree_launch(const double* coeffs, int64_t sc, int64_t n, const double* zre,
                          const double* zim, int64_t sz, int64_t i0, int64_t i1, double* zre_out,
                          double* zim_out, int64_t so, double* step_mag, int* flag, DkPeers peers,
                          double* ws, mw_tuning tune, cudaStream_t st) {
  const int64_t cnt = i1 - i0;
  if (!ws) {
    dk_tree_kernel<K, VAR, PEER, false><<<(unsigned)cnt, 96, 0, st>>>(
        coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so, step_mag, flag, peers,
        (const double*)nullptr, (int64_t)0);
    return launch_status();
  }
  int roots = tune.dk_tree_roots;
  if (roots < 0) roots = cnt >= 512 ? 4 : cnt >= 256 ? 2 : 1;  // auto: ~128+ CTAs when possible
  // R = 1 squares w -> w^32 inside the sweep (beside the scan)
  dk_pow_kernel<K, VAR><<<(unsigned)((cnt + 127) / 128), 128, 0, st>>>(zre, zim, sz, n, i0, i1, ws,
                                                                       cnt, roots == 1 ? 0 : 1);
  int rc = launch_status();
  if (rc) return rc;
  if (roots == 1) return dk_treem_launch<K, VAR, PEER, 1>(coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so, step_mag, flag, peers, ws, st);
  if (roots == 2) return dk_treem_launch<K, VAR, PEER, 2>(coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so, step_mag, flag, peers, ws, st);
  if (roots == 4) return dk_treem_launch<K, VAR, PEER, 4>(coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so, step_mag, flag, peers, ws, st);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cnt);
  cfg.blockDim = dim3(96);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, dk_tree_kernel<K, VAR, PEER, true>, coeffs, sc, n, zre,
                                     zim, sz, i0, i1, zre_out, zim_out, so, step_mag, flag, peers,
                                     (const double*)ws, cnt);
  if (e == cudaErrorNotSupported) {
    // no programmatic launch here: plain stream order (griddepcontrol.wait
    // is then a no-op and the powers are complete before the sweep starts)
    (void)cudaGetLastError();
    dk_tree_kernel<K, VAR, PEER, true><<<(unsigned)cnt, 96, 0, st>>>(
        coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so, step_mag, flag, peers,
        (const double*)ws, cnt);
    return launch_status();
  }
  if (e != cudaSuccess) return (int)e;
  return launch_status();
}

// Exact-order sweep launch (dk_exact2_kernel for TD/QD when split, else
// dk_exact_kernel).  ws is unused.
template <int K, int VAR, bool PEER>
int dk_exact_launch(const double* coeffs, int64_t sc, int64_t n, const double* zre,
                    const double* zim, int64_t sz, int64_t i0, int64_t i1, double* zre_out,
                    double* zim_out, int64_t so, double* step_mag, int* flag, DkPeers peers,
                    double* ws, mw_tuning tune, cudaStream_t st) {
  (void)ws;
  const int64_t cnt = i1 - i0;
  const int r = tune.dk_exact_roots;
  const int64_t blocks = (cnt + r - 1) / r;
  if (tune.dk_exact_split && K >= DK_SPLIT_MIN_K)
    dk_exact2_kernel<K, VAR, PEER><<<(unsigned)blocks, 128, 0, st>>>(
        coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so, step_mag, flag, r, peers);
  else
    dk_exact_kernel<K, VAR, PEER><<<(unsigned)blocks, 2 * DK_EXACT_ROOTS, 0, st>>>(
        coeffs, sc, n, zre, zim, sz, i0, i1, zre_out, zim_out, so, step_mag, flag, r, peers);
  return launch_status();
}

// The sweep launchers are instantiated in dk_exact_k*.cu / dk_tree_k*.cu
// (one translation unit per K and family, compiled in parallel); other
// units see only these declarations.
#define MW_DK_LAUNCH_SIG(FN, K, VAR, PEER)                                                    \
  int FN<K, VAR, PEER>(const double*, int64_t, int64_t, const double*, const double*, int64_t, \
                       int64_t, int64_t, double*, double*, int64_t, double*, int*, DkPeers,    \
                       double*, mw_tuning, cudaStream_t)
#define MW_DK_FOR_K(PREFIX, FN, K)             \
  PREFIX MW_DK_LAUNCH_SIG(FN, K, 0, false);    \
  PREFIX MW_DK_LAUNCH_SIG(FN, K, 1, false);    \
  PREFIX MW_DK_LAUNCH_SIG(FN, K, 0, true);     \
  PREFIX MW_DK_LAUNCH_SIG(FN, K, 1, true);

}  // namespace mw
