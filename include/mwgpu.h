/* mwgpu.h — C-ABI of the B200 branch-free DD/TD/QD kernels.
 *
 * This is the drop-in boundary for the reference's array-level dispatch
 * (K, Variant) -> f(a_comps, b_comps) -> out_comps
 * (pkg/src/mwfloat/batch.py:178-194) and the lane/row/point folds built on
 * it (linalg.py:284-297, poly.py:89-96, roots.py:240-315).
 *
 * Conventions (all entry points):
 *  - A K-word array is K planes of float64 in device memory; plane c of an
 *    operand starts at  base + c * plane_stride  (strides in elements).
 *    Matrices are row-major inside a plane with leading dimension ld.
 *  - k is the word count (2 = DD, 3 = TD, 4 = QD); variant is
 *    MW_VARIANT_STANDARD (0, the reference's default: dw_add_accurate /
 *    dw_mul and the renormalising tw_/qw_ add/mul, multiword.py:118-145,
 *    164-513) or MW_VARIANT_BRANCH_FREE (1, multiword.py:129-156,
 *    361-402, 516-588).  Both exist for every k.
 *  - Pointers are caller-owned device pointers; nothing is allocated.
 *    `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous and stream-ordered; results are valid after the stream
 *    synchronises.
 *  - Return value: 0 on success, a negative MW_ERR_* for argument errors
 *    (nothing launched), or a positive cudaError_t from the launch.
 *    Non-finite values propagate, never trap (multiword.py:18-20).
 */
#ifndef MWGPU_H
#define MWGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MW_VARIANT_STANDARD 0
#define MW_VARIANT_BRANCH_FREE 1

#define MW_OK 0
#define MW_ERR_INVALID -1     /* bad k / size / stride / pointer            */
#define MW_ERR_UNSUPPORTED -2 /* reserved: (k, variant) without a kernel     */

/* Largest DK degree: the collision key j*n + i must stay below INT32_MAX
 * (the "no collision" sentinel), so every collision is reported. */
#define MW_DK_MAX_N 46340

#define MW_ORDER_EXACT 0 /* reference fold order: bit-exact, one thread/output */
#define MW_ORDER_TREE 1  /* fixed split + pairwise tree: within n*2^-p bound   */

/* Library version string and a static message for a status code. */
const char* mw_version(void);
const char* mw_status_string(int status);

/* Named kernels outside the (K, Variant) dispatch, over component planes
 * (plane strides sa / sb / so, n lanes):
 *   MW_NAMED_DW_ADD_SLOPPY  DD, replaces multiword.dw_add_sloppy
 *                           (multiword.py:104-115)
 *   MW_NAMED_TW_MUL_CLEANED TD, replaces multiword.tw_mul_cleaned
 *                           (multiword.py:325-358)                       */
#define MW_NAMED_DW_ADD_SLOPPY 0
#define MW_NAMED_TW_MUL_CLEANED 1
int mw_named_op(int op, const double* a, int64_t sa, const double* b, int64_t sb,
                double* out, int64_t so, int64_t n, void* stream);

/* Renormalisation of raw expansions (replaces multiword.tw_renormalize /
 * qw_renormalize, multiword.py:191-241, and normalize 710-719): k = 2 reads
 * 2 planes (quick_two_sum), k = 3 reads 4 planes (s0, s1, s2, t0), k = 4
 * reads 5 planes (x0..x4); writes k planes.  Value-dependent branches per
 * lane, as in the reference. */
int mw_renormalize(int k, const double* in, int64_t si, double* out, int64_t so,
                   int64_t n, void* stream);

/* Correctly rounded a*b + c per element (replaces eft.fma, eft.py:33-48 /
 * _fmaext.c:16-40). */
int mw_fma(const double* a, const double* b, const double* c, double* out, int64_t n,
           void* stream);

/* The error-free transformations over arrays (eft.py:51-83): op 0
 * quick_two_sum (requires |a| >= |b|), 1 two_sum, 2 two_prod (one FMA);
 * s[i] + e[i] == a[i] op b[i] exactly (within the EFT contracts). */
int mw_eft(int op, const double* a, const double* b, double* s, double* e,
           int64_t n, void* stream);

/* out = a (+) b lane-wise.  Replaces batch.batch_add -> _BATCH_ADD[(k,v)]
 * (batch.py:204-207, 178-185).  Bit-exact with the reference. */
int mw_ew_add(int k, int variant, const double* a, int64_t sa, const double* b,
              int64_t sb, double* out, int64_t so, int64_t n, void* stream);

/* out = a (-) b = a (+) (-b).  Replaces mw_sub / linalg._ew_sub
 * (multiword.py:629-630, linalg.py:200-201).  Bit-exact. */
int mw_ew_sub(int k, int variant, const double* a, int64_t sa, const double* b,
              int64_t sb, double* out, int64_t so, int64_t n, void* stream);

/* out = a (*) b.  Replaces batch.batch_mul -> _BATCH_MUL[(k,v)]
 * (batch.py:210-213, 187-194).  Bit-exact. */
int mw_ew_mul(int k, int variant, const double* a, int64_t sa, const double* b,
              int64_t sb, double* out, int64_t so, int64_t n, void* stream);

/* out = a / b by the shared Newton reciprocal sequence.  Replaces
 * batch.batch_div -> _newton_div (batch.py:216-231, multiword.py:639-658).
 * Zero lanes of b give inf/nan.  Bit-exact. */
int mw_ew_div(int k, int variant, const double* a, int64_t sa, const double* b,
              int64_t sb, double* out, int64_t so, int64_t n, void* stream);

/* y <- alpha (*) x (+) y, alpha a host array of k doubles.  Defined by
 * batch_mul then batch_add (batch.py:204-213).  Bit-exact. */
int mw_axpy(int k, int variant, const double* alpha_host, const double* x,
            int64_t sx, double* y, int64_t sy, int64_t n, void* stream);

/* Workspace (in doubles) mw_dot needs for length n (0 when n <= 4096).
 * For 4096 < n <= 2^20 the tree dot is one launch whose last block folds
 * the block partials; its ticket lives in ws[0], which must be zero before
 * the first call (every call leaves it zero and never writes it
 * otherwise, whatever n).  Do not share one workspace between concurrently
 * running calls. */
int64_t mw_dot_workspace(int k, int64_t n);

/* out_dev[0..k) = sum_t x_t (*) y_t.  The definition is the naive-matmul
 * fold (linalg.py:300-314) for 1xn . nx1.  MW_ORDER_EXACT replays it
 * bit-exactly on one thread.  MW_ORDER_TREE: block b covers elements
 * [4096b, 4096b+4096); its partial p (p < 256) folds elements
 * 4096b + p + 256j (j = 0..15) ascending from exact zero (and exists iff
 * 4096b + p < n); all partials combine by a fixed in-place pairwise tree
 * (stride 1, 2, 4, ...; an unpaired tail passes through) -- a function of n
 * only, so the result does not depend on launch shape or GPU count.
 * ws: mw_dot_workspace(k, n) doubles (may be NULL when that is 0). */
int mw_dot(int k, int variant, const double* x, int64_t sx, const double* y,
           int64_t sy, int64_t n, double* ws, double* out_dev, int order,
           void* stream);

/* Tree-dot first stage for sharded dots: writes mw_dot_num_partials(n) =
 * ceil(n/4096) block partials (each the tree root of its 256 partials) to
 * partials[c*pstride + b].  Shards that split x, y at multiples of 4096
 * elements produce partials that, concatenated in shard order and folded
 * with mw_tree_fold, equal the single-GPU mw_dot bit for bit. */
int64_t mw_dot_num_partials(int64_t n);
int mw_dot_partials(int k, int variant, const double* x, int64_t sx,
                    const double* y, int64_t sy, int64_t n, double* partials,
                    int64_t pstride, void* stream);

/* out_dev[0..k) = pairwise-tree fold of count K-word values (plane stride
 * pstride), the tree mw_dot uses above the block level.
 * ws: mw_tree_fold_workspace(k, count) doubles (NULL when 0). */
int64_t mw_tree_fold_workspace(int k, int64_t count);
int mw_tree_fold(int k, int variant, const double* partials, int64_t pstride,
                 int64_t count, double* ws, double* out_dev, void* stream);

/* y = A x, A m x n.  Definition: y_i = fold_t add(acc, mul(A_it, x_t)) from
 * exact zero, t ascending = matmul(A, x as n x 1, naive) (linalg.py:284-297).
 * MW_ORDER_EXACT: one thread per row, bit-exact.  MW_ORDER_TREE: 128
 * partials per row (four warps); partial u folds t = u, u+128, ... from
 * exact zero, then an in-place pairwise tree over min(n, 128) partials. */
int mw_gemv(int k, int variant, const double* A, int64_t lda, int64_t sA,
            const double* x, int64_t sx, double* y, int64_t sy, int64_t m,
            int64_t n, int order, void* stream);

/* C = A B, A m x kd, B kd x n.  Each C_ij folds t ascending from exact zero
 * exactly as _rows_kernel_simd / _rows_kernel_scalar (linalg.py:284-314),
 * so the result is bit-exact with matmul(..., MatMulPlan("naive", v)). */
int mw_gemm(int k, int variant, const double* A, int64_t lda, int64_t sA,
            const double* B, int64_t ldb, int64_t sB, double* C, int64_t ldc,
            int64_t sC, int64_t m, int64_t n, int64_t kd, void* stream);

/* Batched / accumulating form of mw_gemm: for b < batch,
 *   C_b = Cin_b + A_b B_b   (every C_ij folds t ascending starting from
 *                            Cin_ij, or from exact zero when Cin == NULL),
 * operand b at base + b * bs (elements), planes at + c * s.  The Strassen
 * scheme (linalg.py:390-546) runs its 7^L leaf products and its odd-size
 * peel folds (which start from a product, linalg.py:470-500) through it. */
int mw_gemm_batched(int k, int variant, const double* A, int64_t lda,
                    int64_t sA, int64_t bsA, const double* B, int64_t ldb,
                    int64_t sB, int64_t bsB, double* C, int64_t ldc,
                    int64_t sC, int64_t bsC, const double* Cin, int64_t ldci,
                    int64_t sCi, int64_t bsCi, int64_t m, int64_t n,
                    int64_t kd, int64_t batch, void* stream);

/* y_p = Horner(coeffs, x_p) for npts points: acc = a_deg; acc = acc (*) x
 * (+) a_i for i = deg-1..0 (poly.py:89-96).  coeffs: k planes of deg+1
 * doubles (a_i multiplies x^i).  Bit-exact with horner_eval per point.
 * QD branch-free points whose low words are all +0.0 (plain doubles) take a
 * shortened product (63 instead of 106 FP64 instructions) that is
 * bit-identical for finite values; a non-finite result re-runs the full
 * product, so the result is horner_eval's in every case. */
int mw_horner(int k, int variant, const double* coeffs, int64_t sc,
              int64_t degree, const double* x, int64_t sx, double* y,
              int64_t sy, int64_t npts, void* stream);

/* Batched polynomial evaluation, one point per thread:
 * method 0 = Horner, 1 = Estrin (coefficients zero-padded to a power of
 * two, level-by-level pairwise combine, x squared between levels;
 * poly.estrin_eval / estrin_eval_batched, poly.py:106-153).  xim == NULL:
 * real points x (k planes, stride sx) -> y; xim != NULL: complex points
 * (xre, xim) -> (yre, yim) with the 3M product and (a_i, 0) coefficients
 * (poly.eval_complex, poly.py:156-178).  Bit-exact per point. */
int mw_poly_eval(int k, int variant, const double* coeffs, int64_t sc,
                 int64_t degree, const double* xre, const double* xim,
                 int64_t sx, double* yre, double* yim, int64_t sy,
                 int64_t npts, int method, void* stream);

/* One Durand-Kerner sweep (roots.py:240-315) for roots i in [i0, i1) of
 * the monic degree-n polynomial z^n + sum c_j z^j.  Reads the frozen full
 * state (zre, zim: k planes of n doubles each, plane stride sz), writes
 * updated roots i into zre_out/zim_out at index i (plane stride so) and
 * |step| = hypot(step_re0, step_im0) into step_mag[i].  The caller sets
 * *flag_dev = INT32_MAX first; a vanishing denominator factor lowers it to
 * min over (j*n + i) of the colliding pairs, and the caller raises
 * CollisionError (roots.py:289-292).  exact_order = 1 replays the
 * reference order bit for bit; 0 is the tree order: 64 partial products and
 * 64 Horner blocks per root combined by pairwise trees, complex products
 * in the four-multiplication form -- within the stated accuracy contract
 * of the reference, not bitwise.  1 <= n <=
 * MW_DK_MAX_N. */
int mw_dk_sweep(int k, int variant, const double* coeffs, int64_t sc,
                int64_t n, const double* zre, const double* zim, int64_t sz,
                int64_t i0, int64_t i1, double* zre_out, double* zim_out,
                int64_t so, double* step_mag, int* flag_dev, int exact_order,
                void* stream);

/* Root-sharded DK sweep with the per-sweep state exchange fused into the
 * kernel (replaces the all-gather that follows mw_dk_sweep
 * in dist.dk_sweeps_sharded, the reference's thread-pool join over the
 * shared state, roots.py:240-315).  Every rank holds the full state
 * twice, as (2k, n) planes (re planes then im planes, plane stride n):
 * state_in is read; the lane finishing root i (i in [i0, i1)) writes it
 * to state_out_local and to peer_out[p] for every other rank p (device
 * array of world pointers, cudaIpc-mapped) -- the transfer overlaps the
 * remaining roots' arithmetic.  The last CTA then stores the value
 * epoch*sweeps + sweep + 1 into slot [rank] of every peer_slot[p] (device
 * array of world pointers to world-u64 slot arrays; st.release.sys) and
 * waits, at most spin_limit polls of ~0.25 us, until every entry of
 * my_slot reaches it; on expiry it sets *timeout = 1 and returns (no
 * hang).  done (u32, zero-initialised) is a self-resetting CTA ticket;
 * epoch (u64) counts completed runs and is advanced by the sweep
 * == sweeps - 1 launch.  ws: optional workspace as for mw_dk_sweep_ws
 * (NULL allowed).  Arithmetic and order are those of mw_dk_sweep
 * (exact_order as there), so results are bitwise independent of world. */
int mw_dk_sweep_peer(int k, int variant, const double* coeffs, int64_t sc,
                     int64_t n, const double* state_in, int64_t i0, int64_t i1,
                     double* const* peer_out,
                     unsigned long long* const* peer_slot,
                     double* state_out_local, unsigned long long* my_slot,
                     unsigned int* done, unsigned long long* epoch, int* timeout,
                     int world, int rank, int sweep, int sweeps,
                     long long spin_limit, double* step_mag, int* flag_dev,
                     int exact_order, double* ws, void* stream);

/* Sharded tree dot with the all-gather-then-sum fused into one kernel per
 * rank ("dot products by a custom multi-component
 * all-gather-then-sum, since NCCL's sum is not error-free"; replaces
 * mw_dot_partials + all-gather + mw_tree_fold of dist.dot_allgather).
 * x, y: this rank's slice (n_local elements) starting at global element
 * 4096*b0 (slices cut at multiples of 4096; only the last may be ragged).
 * nbt = ceil(n_total/4096) <= 65536 block roots over all ranks.  Each block
 * stores its root into slot b0 + b of every rank's root buffer
 * (peer_roots: device array of world pointers; buffer = 2 parities x k
 * planes x nbt doubles, parity = *epoch & 1); the last block publishes
 * *epoch + 1 into peer_slot (as mw_dk_sweep_peer), waits (bounded by
 * spin_limit, then *timeout = 1), folds the nbt roots with the pairwise
 * tree and writes k doubles to out_dev; *epoch is then incremented.
 * Bit-identical to mw_dot(order TREE) over the full vectors. */
int mw_dot_peer(int k, int variant, const double* x, int64_t sx,
                const double* y, int64_t sy, int64_t n_local, int64_t b0,
                int64_t nbt, double* const* peer_roots,
                unsigned long long* const* peer_slot,
                unsigned long long* my_slot, unsigned int* done,
                unsigned long long* epoch, int* timeout, int world, int rank,
                long long spin_limit, double* out_dev, void* stream);

/* Peer buffers for mw_dk_sweep_peer / mw_dot_peer: a zeroed cudaMalloc allocation (one
 * IPC handle covers exactly one buffer), its 64-byte cudaIpcMemHandle_t,
 * and open/close of a peer's handle (cudaIpcMemLazyEnablePeerAccess). */
int mw_peer_alloc(int64_t bytes, void** out);
int mw_peer_free(void* p);
int mw_ipc_get_handle(void* p, void* handle64);
int mw_ipc_open_handle(const void* handle64, void** out);
int mw_ipc_close_handle(void* p);

/* mw_dk_sweep with a caller workspace of mw_dk_sweep_workspace(k, i0, i1)
 * doubles (device memory, stream-ordered, not shared between concurrent
 * calls).  Tree order: w = z^B and w^32 of every root are then computed
 * by a lane-per-root kernel and the sweep kernel is a programmatic
 * dependent launch whose powers warp waits for them (griddepcontrol), so
 * no warp computes a value its 32 lanes duplicate.  Identical results;
 * ignored for the exact order. */
int64_t mw_dk_sweep_workspace(int k, int64_t i0, int64_t i1);
int mw_dk_sweep_ws(int k, int variant, const double* coeffs, int64_t sc,
                   int64_t n, const double* zre, const double* zim, int64_t sz,
                   int64_t i0, int64_t i1, double* zre_out, double* zim_out,
                   int64_t so, double* step_mag, int* flag_dev, int exact_order,
                   double* ws, void* stream);

/* Per-call tuning of the launch shape (no global state: the library is
 * stateless and reentrant).  Results never depend on it:
 * every choice runs the same ops in the same order.  NULL = defaults.
 *   gemm_tile      0 (default) picks the CTA tile per call from the shape
 *                  (smaller tiles for row-block shards, where the large
 *                  tile leaves SMs unevenly loaded); 1..3 force slot 0..2.
 *   dot_cluster    1 (default) runs dots of 2..16 blocks of 4096 elements
 *                  as one thread-block cluster (block roots folded through
 *                  distributed shared memory); 0 the single-launch ticket
 *                  form.
 *   dk_tree_roots  tree-order sweep with a workspace: roots per CTA, 1, 2
 *                  or 4 (one chain per lane, trees packed level by level
 *                  over the CTA's roots); -1 (default) by shard size (4
 *                  from 512 roots, 2 from 256, else 1); 0 the 3-warp
 *                  single-root kernel.
 *   dk_exact_roots exact-order sweep: roots per CTA, 1..32 (default 32).
 *   dk_exact_split exact-order sweep: 1 (default) splits each TD/QD
 *                  root's chains over a pair of warps (real / imaginary
 *                  halves of the 3M product), 0 one warp per chain.      */
typedef struct mw_tuning {
  int gemm_tile;
  int dot_cluster;
  int dk_tree_roots;
  int dk_exact_roots;
  int dk_exact_split;
} mw_tuning;

/* Fills *t with the defaults; returns MW_OK (MW_ERR_INVALID for NULL). */
int mw_tuning_defaults(mw_tuning* t);

/* mw_gemm / mw_dot / mw_dk_sweep_ws with explicit tuning (NULL = the
 * defaults the plain entry points use); MW_ERR_INVALID for a value out of
 * range.  mw_dk_sweep_ex: if max_mag_bits != NULL (two device u64 the
 * caller zeroes first), [0] is atomically raised to the bit pattern of
 * every step_mag written and [1] to that of every new root's
 * hypot(re0, im0), so after the sweep they hold the sweep's max update
 * (RootState.last_max_update, roots.py:308) and the max |z| of dk_solve's
 * convergence test (roots.py:336) with no separate reduction; both are
 * >= 0, so the bit order is the value order. */
int mw_gemm_ex(int k, int variant, const double* A, int64_t lda, int64_t sA,
               const double* B, int64_t ldb, int64_t sB, double* C, int64_t ldc,
               int64_t sC, int64_t m, int64_t n, int64_t kd,
               const mw_tuning* tune, void* stream);
int mw_dot_ex(int k, int variant, const double* x, int64_t sx, const double* y,
              int64_t sy, int64_t n, double* ws, double* out_dev, int order,
              const mw_tuning* tune, void* stream);
int mw_dk_sweep_ex(int k, int variant, const double* coeffs, int64_t sc,
                   int64_t n, const double* zre, const double* zim, int64_t sz,
                   int64_t i0, int64_t i1, double* zre_out, double* zim_out,
                   int64_t so, double* step_mag, int* flag_dev, int exact_order,
                   double* ws, unsigned long long* max_mag_bits,
                   const mw_tuning* tune, void* stream);

/* FP64 pipe microbenchmark: 8 independent DFMA (op = 0) or DADD (op = 1)
 * chains per thread, 8 unrolled steps per iteration: executes
 * blocks * threads * iters * 64 FP64 ops, no memory traffic; the caller
 * times it.  sink receives one double per thread (threads <= 256). */
int mw_fp64_peak_kernel(int op, int blocks, int threads, int iters,
                        double* sink, void* stream);

/* Multiprocessor count of the current device (grid sizing helper). */
int mw_device_sm_count(void);

#ifdef __cplusplus
}
#endif

#endif /* MWGPU_H */
