"""Generate golden fixtures for the DD/TD/QD hot path FROM THE REFERENCE.

Run in the build container (the reference is not on the GPU box):

    python tests/golden/make_golden.py [--ref /path/to/built/pkg/src]

It copies /root/reference/pkg to a scratch dir, builds its C extension
(`python setup.py build_ext --inplace`, the reference's own recipe), imports
`mwfloat` from there and records inputs + outputs of the reference's own
public functions on small seeded cases:

  ew.npz      batch_add / batch_mul / batch_div / linalg._ew_sub
              (batch.py:204-231, linalg.py:200-201)
  dot.npz     scalar fold mw_add(acc, mw_mul(x_t, y_t)) == matmul(1xn, nx1, naive)
  axpy.npz    batch_mul(alpha, x) then batch_add(., y)
  gemv.npz    matmul(A, x as n x 1, naive)                (linalg.py:549-569)
  gemm.npz    matmul(A, B, naive), blocked checked equal    (linalg.py:284-349)
  horner.npz  horner_eval per point                         (poly.py:89-96)
  dk.npz      aberth_init + dk_iterate (one sweep), and the config-5
              degree-512 problem expanded with Fractions +
              from_oracle, one sweep from the near-root start and one from
              the R0 = 1.5 Aberth circle                     (roots.py:188-315)
  cgemm.npz   cmatmul (3M) on gen_complex_test_matrices     (linalg.py:247-276, 572-590)
  strassen.npz matmul(scheme="strassen") with even splits and odd peels (linalg.py:390-546)
  testmats.npz gen_test_matrices(16, k) and chebyshev_coeffs(12, k) (linalg.py:224-244, roots.py:343-368)
  dksolve.npz dk_solve from the reference's Aberth start (final roots and
              sweep count) on chebyshev_coeffs(16 / 64)   (roots.py:318-368)
  named.npz   dw_add_sloppy, tw_mul_cleaned, tw_/qw_renormalize, normalize,
              eft.fma, strassen_pad_policy (multiword.py:104-358, 710-719)
  polyx.npz   estrin_eval per point (== estrin_eval_batched) and
              eval_complex Horner / Estrin                   (poly.py:106-178)

Every array is stored component-planar (K x ...).  The fixtures are small
(< 1 MB total) and committed; tests/test_oracle_golden.py pins the C
oracle to them on CPU, and the GPU parity tests compare against them too.
"""

from __future__ import annotations

import argparse
import math
import os
import shutil
import subprocess
import sys
import time
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from paper_2603_14926_b200 import gen  # noqa: E402


def build_reference(dst="/tmp/mwfloat_ref_build") -> str:
    src = "/root/reference/pkg"
    if not os.path.exists(os.path.join(dst, "src", "mwfloat")):
        shutil.rmtree(dst, ignore_errors=True)
        shutil.copytree(src, dst)
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=dst, check=True,
                   stdout=subprocess.DEVNULL)
    return os.path.join(dst, "src")


def rand_mw(rng, k, w, e_lo=-100, e_hi=100):
    """Wide-exponent K-word values (the reference tests' generator,
    pkg/tests/conftest.py:127-133)."""
    c0 = rng.uniform(1.0, 2.0, w) * np.exp2(rng.integers(e_lo, e_hi + 1, w))
    c0 *= np.where(rng.random(w) < 0.5, -1.0, 1.0)
    comps = [c0]
    for _ in range(1, k):
        comps.append(comps[-1] * 2.0**-53 * rng.uniform(-0.49, 0.49, w))
    return np.stack(comps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=None, help="path containing the built mwfloat package")
    ap.add_argument("--skip-dk512", action="store_true")
    ap.add_argument("--only", default="", help="comma list of fixture names to (re)generate")
    args = ap.parse_args()
    sys.path.insert(0, args.ref or build_reference())
    import mwfloat
    from mwfloat import batch, linalg, multiword, poly, roots
    from mwfloat.multiword import Variant, from_oracle
    from mwfloat.oracle import BigFloat, oracle_cos, oracle_pi, oracle_sin

    BF, STD = Variant.BRANCH_FREE, Variant.STANDARD
    cases = [(2, BF), (3, BF), (4, BF), (2, STD), (3, STD), (4, STD)]
    tag = {BF: "bf", STD: "std"}
    t0 = time.time()

    only = set(filter(None, args.only.split(",")))

    def want(name):
        return not only or name in only

    # ------------------------------------------------------------- ew
    out = {}
    rng = np.random.default_rng(20240809)
    W = 257
    for k, v in cases:
        a = rand_mw(rng, k, W)
        b = rand_mw(rng, k, W)
        # special lanes: exact cancellation, zero operand, identical, one
        a[:, 0] = -b[:, 0]
        b[:, 1] = 0.0
        a[:, 2] = b[:, 2]
        b[:, 3] = 0.0
        b[0, 3] = 1.0
        la, lb = batch.LaneBatch(tuple(a)), batch.LaneBatch(tuple(b))
        p = f"k{k}_{tag[v]}"
        out[p + "_a"] = a
        out[p + "_b"] = b
        out[p + "_add"] = np.stack(batch.batch_add(la, lb, v).comps)
        out[p + "_mul"] = np.stack(batch.batch_mul(la, lb, v).comps)
        out[p + "_sub"] = np.stack(linalg._ew_sub(la.comps, lb.comps, v))
        bz = b.copy()
        bz[:, 5] = 0.0  # zero divisor lane propagates inf/nan (batch.py:216-219)
        out[p + "_bz"] = bz
        out[p + "_div"] = np.stack(batch.batch_div(la, batch.LaneBatch(tuple(bz)), v).comps)
        # scalar path agrees per lane (test_batch.py:86-122 property)
        for lane in (7, 100):
            sa = tuple(float(c) for c in a[:, lane])
            sb = tuple(float(c) for c in b[:, lane])
            assert multiword.mw_add(sa, sb, v) == tuple(out[p + "_add"][:, lane])
            assert multiword.mw_mul(sa, sb, v) == tuple(out[p + "_mul"][:, lane])
    if want("ew"):
        np.savez_compressed(os.path.join(HERE, "ew.npz"), **out)
    print(f"ew done {time.time() - t0:.1f}s")

    # ------------------------------------------------------------- dot
    out = {}
    for k, v in cases:
        n = 300
        rng = np.random.default_rng(100 + k)
        x = gen.g_k(rng, k, n)
        y = gen.g_k(rng, k, n)
        acc = (0.0,) * k
        for t in range(n):
            acc = multiword.mw_add(acc, multiword.mw_mul(tuple(x[:, t]), tuple(y[:, t]), v), v)
        mm = linalg.matmul(
            linalg.MWMatrix(tuple(c.reshape(1, n) for c in x)),
            linalg.MWMatrix(tuple(c.reshape(n, 1) for c in y)),
            linalg.MatMulPlan(scheme="naive", variant=v),
        )
        assert tuple(float(c[0, 0]) for c in mm.comps) == acc
        p = f"k{k}_{tag[v]}"
        out[p + "_x"] = x
        out[p + "_y"] = y
        out[p + "_out"] = np.array(acc)
    if want("dot"):
        np.savez_compressed(os.path.join(HERE, "dot.npz"), **out)

    # ------------------------------------------------------------- axpy
    out = {}
    for k, v in cases:
        n = 1000
        rng = np.random.default_rng(200 + k)
        x = gen.g_k(rng, k, n)
        y = gen.g_k(rng, k, n)
        alpha = gen.g_k(rng, k, 1)[:, 0]
        la = batch.LaneBatch(tuple(np.full(n, alpha[c]) for c in range(k)))
        prod = batch.batch_mul(la, batch.LaneBatch(tuple(x)), v)
        r = batch.batch_add(prod, batch.LaneBatch(tuple(y)), v)
        p = f"k{k}_{tag[v]}"
        out[p + "_alpha"] = alpha
        out[p + "_x"] = x
        out[p + "_y"] = y
        out[p + "_out"] = np.stack(r.comps)
    if want("axpy"):
        np.savez_compressed(os.path.join(HERE, "axpy.npz"), **out)
    print(f"dot/axpy done {time.time() - t0:.1f}s")

    # ------------------------------------------------------------- gemv
    out = {}
    for k, v in cases:
        m, n = 40, 67
        rng = np.random.default_rng(300 + k)
        a = gen.g_k(rng, k, (m, n))
        x = gen.g_k(rng, k, n)
        r = linalg.matmul(
            linalg.MWMatrix(tuple(a)),
            linalg.MWMatrix(tuple(c.reshape(n, 1) for c in x)),
            linalg.MatMulPlan(scheme="naive", variant=v),
        )
        p = f"k{k}_{tag[v]}"
        out[p + "_a"] = a
        out[p + "_x"] = x
        out[p + "_out"] = np.stack([c[:, 0] for c in r.comps])
    if want("gemv"):
        np.savez_compressed(os.path.join(HERE, "gemv.npz"), **out)

    # ------------------------------------------------------------- gemm
    out = {}
    for k, v in cases:
        m, kd, n = 19, 23, 29
        rng = np.random.default_rng(400 + k)
        a = gen.g_k(rng, k, (m, kd))
        b = gen.g_k(rng, k, (kd, n))
        A, B = linalg.MWMatrix(tuple(a)), linalg.MWMatrix(tuple(b))
        r = linalg.matmul(A, B, linalg.MatMulPlan(scheme="naive", variant=v))
        rb = linalg.matmul(A, B, linalg.MatMulPlan(scheme="blocked", variant=v, strassen_cutoff=8))
        assert r.bitwise_equal(rb)
        p = f"k{k}_{tag[v]}"
        out[p + "_a"] = a
        out[p + "_b"] = b
        out[p + "_out"] = np.stack(r.comps)
    if want("gemm"):
        np.savez_compressed(os.path.join(HERE, "gemm.npz"), **out)
    print(f"gemv/gemm done {time.time() - t0:.1f}s")

    # ------------------------------------------------------------- horner
    out = {}
    for k, v, deg, npts in [(4, BF, 1024, 24), (3, BF, 100, 40), (2, BF, 100, 40), (2, STD, 100, 40),
                            (3, STD, 100, 40), (4, STD, 200, 24)]:
        coeffs, x = gen.config4_horner(npts=npts, degree=deg, k=k, seed=500 + k)
        # half the points carry full K-word values
        rng = np.random.default_rng(550 + k)
        x[:, npts // 2:] = gen.g_k(rng, k, npts - npts // 2)
        p_ = poly.MWPolynomial(tuple(coeffs))
        y = np.zeros((k, npts))
        for i in range(npts):
            y[:, i] = poly.horner_eval(p_, tuple(float(c) for c in x[:, i]), v)
        p = f"k{k}_{tag[v]}"
        out[p + "_coeffs"] = coeffs
        out[p + "_x"] = x
        out[p + "_out"] = y
    if want("horner"):
        np.savez_compressed(os.path.join(HERE, "horner.npz"), **out)
    print(f"horner done {time.time() - t0:.1f}s")

    # ------------------------------------------------------------- dk
    out = {}
    for k, v in cases:
        q = roots.chebyshev_coeffs(16, k)
        st = roots.aberth_init(q, v)
        nxt = roots.dk_iterate(q, st, v)
        p = f"k{k}_{tag[v]}"
        out[p + "_coeffs"] = np.stack(q.comps)
        out[p + "_zre"] = np.stack(st.re)
        out[p + "_zim"] = np.stack(st.im)
        out[p + "_new_re"] = np.stack(nxt.re)
        out[p + "_new_im"] = np.stack(nxt.im)
        out[p + "_maxupd"] = np.array([nxt.last_max_update])
    if not args.skip_dk512 and want("dk"):
        n = 512
        r = gen.config5_roots(n, 0)
        for k in (3, 4):
            # exact expansion in Fractions via quadratic factors
            coeffs_fr = [Fraction(1)]
            for root in r[: n // 2]:
                a1 = Fraction(-2) * Fraction(float(root.real))
                a0 = Fraction(float(root.real)) ** 2 + Fraction(float(root.imag)) ** 2
                newc = [Fraction(0)] * (len(coeffs_fr) + 2)
                for i, c in enumerate(coeffs_fr):
                    newc[i] += c * a0
                    newc[i + 1] += c * a1
                    newc[i + 2] += c
                coeffs_fr = newc
            rows = [from_oracle(coeffs_fr[i], k) for i in range(n)]
            q = roots.MonicPoly(tuple(np.array([row[c] for row in rows]) for c in range(k)))
            zre, zim = gen.config5_init(k, n)
            st = roots.RootState(re=tuple(zre), im=tuple(zim))
            nxt = roots.dk_iterate(q, st, BF)
            p = f"c5_k{k}"
            out[p + "_coeffs"] = np.stack(q.comps)
            out[p + "_zre"] = zre
            out[p + "_zim"] = zim
            out[p + "_new_re"] = np.stack(nxt.re)
            out[p + "_new_im"] = np.stack(nxt.im)
            out[p + "_maxupd"] = np.array([nxt.last_max_update])
            # Aberth circle with the reference's centre and angles, R0 = 1.5
            cen = multiword.mw_neg(multiword.mw_div(q.coeff(n - 1), multiword.from_basefloat(float(n), k), BF))
            pi = oracle_pi()
            two_over_n = BigFloat.from_fraction(Fraction(2, n))
            offset = BigFloat.from_fraction(Fraction(3, 2 * n))
            cre = np.zeros((k, n))
            cim = np.zeros((k, n))
            for j in range(1, n + 1):
                theta = BigFloat.from_int(j - 1).mul(two_over_n).mul(pi).add(offset)
                cre[:, j - 1] = from_oracle(oracle_cos(theta), k)
                cim[:, j - 1] = from_oracle(oracle_sin(theta), k)
            add, mul = batch._BATCH_ADD[k, BF], batch._BATCH_MUL[k, BF]
            rad = tuple(np.full(n, c) for c in multiword.from_basefloat(1.5, k))
            cenb = tuple(np.full(n, cen[c]) for c in range(k))
            are = np.stack(add(cenb, mul(rad, tuple(cre))))
            aim = np.stack(mul(rad, tuple(cim)))
            st2 = roots.RootState(re=tuple(are), im=tuple(aim))
            nxt2 = roots.dk_iterate(q, st2, BF)
            out[p + "_ab_zre"] = are
            out[p + "_ab_zim"] = aim
            out[p + "_ab_new_re"] = np.stack(nxt2.re)
            out[p + "_ab_new_im"] = np.stack(nxt2.im)
            out[p + "_ab_maxupd"] = np.array([nxt2.last_max_update])
            print(f"dk512 k={k} done {time.time() - t0:.1f}s")
    if want("dk"):
        np.savez_compressed(os.path.join(HERE, "dk.npz"), **out)
    # ------------------------------------------------------------- estrin / complex eval
    out = {}
    for k, v, deg, npts in [(4, BF, 1024, 16), (3, BF, 100, 33), (2, BF, 37, 33), (2, STD, 37, 33), (4, BF, 0, 3),
                            (3, BF, 1, 5), (3, STD, 20, 9), (4, STD, 20, 9)]:
        rng = np.random.default_rng(700 + k + deg)
        coeffs = gen.g_k(rng, k, deg + 1)
        x = gen.g_k(rng, k, npts) * 1.1
        zr = gen.g_k(rng, k, npts) * 0.9
        zi = gen.g_k(rng, k, npts) * 0.9
        p_ = poly.MWPolynomial(tuple(coeffs))
        est = np.zeros((k, npts))
        hre = np.zeros((k, npts)); him = np.zeros((k, npts))
        ere = np.zeros((k, npts)); eim = np.zeros((k, npts))
        for i in range(npts):
            est[:, i] = poly.estrin_eval(p_, tuple(float(c) for c in x[:, i]), v)
            z = (tuple(float(c) for c in zr[:, i]), tuple(float(c) for c in zi[:, i]))
            r = poly.eval_complex(p_, z, "horner", v)
            hre[:, i], him[:, i] = r[0], r[1]
            r = poly.eval_complex(p_, z, "estrin", v)
            ere[:, i], eim[:, i] = r[0], r[1]
        bat = np.stack(poly.estrin_eval_batched(p_, batch.LaneBatch(tuple(x)), v).comps)
        assert np.array_equal(bat.view(np.int64), est.view(np.int64))
        p = f"k{k}_{tag[v]}_d{deg}"
        out[p + "_coeffs"] = coeffs
        out[p + "_x"] = x
        out[p + "_estrin"] = est
        out[p + "_zre"] = zr
        out[p + "_zim"] = zi
        out[p + "_ch_re"] = hre
        out[p + "_ch_im"] = him
        out[p + "_ce_re"] = ere
        out[p + "_ce_im"] = eim
    if want("polyx"):
        np.savez_compressed(os.path.join(HERE, "polyx.npz"), **out)
    print(f"polyx done {time.time() - t0:.1f}s")

    # ------------------------------------------------------------- 3M complex GEMM
    out = {}
    for k, v, n in [(2, BF, 24), (3, BF, 17), (4, BF, 16), (2, STD, 24), (3, STD, 12), (4, STD, 10)]:
        a, b = linalg.gen_complex_test_matrices(n, 20240806 + k, k)
        c = linalg.cmatmul(a, b, linalg.MatMulPlan(scheme="naive", variant=v))
        p = f"k{k}_{tag[v]}"
        for nm, m in (("a", a), ("b", b), ("c", c)):
            out[f"{p}_{nm}_re"] = np.stack(m.re.comps)
            out[f"{p}_{nm}_im"] = np.stack(m.im.comps)
    if want("cgemm"):
        np.savez_compressed(os.path.join(HERE, "cgemm.npz"), **out)
    print(f"cgemm done {time.time() - t0:.1f}s")

    # ------------------------------------------------------------- Strassen
    out = {}
    for k, v, n, cut in [(2, BF, 37, 8), (3, BF, 48, 8), (4, BF, 35, 4), (2, STD, 37, 8), (3, STD, 20, 4),
                         (4, STD, 18, 4), (2, BF, 64, 32)]:
        rng = np.random.default_rng(900 + k + n)
        a = gen.g_k(rng, k, (n, n))
        b = gen.g_k(rng, k, (n, n))
        c = linalg.matmul(linalg.MWMatrix(tuple(a)), linalg.MWMatrix(tuple(b)),
                          linalg.MatMulPlan(scheme="strassen", variant=v, strassen_cutoff=cut))
        p = f"k{k}_{tag[v]}_n{n}_c{cut}"
        out[p + "_a"] = a
        out[p + "_b"] = b
        out[p + "_out"] = np.stack(c.comps)
        out[p + "_steps"] = np.array([len(linalg.strassen_pad_policy(n, cut))])
    if want("strassen"):
        np.savez_compressed(os.path.join(HERE, "strassen.npz"), **out)
    print(f"strassen done {time.time() - t0:.1f}s")

    # ------------------------------------------------------------- accuracy inputs
    out = {}
    for k in (2, 3, 4):
        a, b = linalg.gen_test_matrices(16, k)
        out[f"k{k}_a"] = np.stack(a.comps)
        out[f"k{k}_b"] = np.stack(b.comps)
        q = roots.chebyshev_coeffs(12, k)
        out[f"k{k}_cheb12"] = np.stack(q.comps)
    if want("testmats"):
        np.savez_compressed(os.path.join(HERE, "testmats.npz"), **out)

    # ------------------------------------------------------------- named kernels
    # multiword's kernels outside the dispatch tables and its helpers:
    # dw_add_sloppy (104-115; arrays), tw_mul_cleaned (325-358) and the
    # renormalisers tw_/qw_renormalize (191-241) + normalize (710-719)
    # (scalar-only in the reference: data-dependent branches, so per lane),
    # eft.fma (eft.py:33-48) and linalg.strassen_pad_policy (390-406).
    if want("named"):
        from mwfloat import eft as reft

        out = {}
        rng = np.random.default_rng(20240810)
        W = 193
        a, b = rand_mw(rng, 2, W), rand_mw(rng, 2, W)
        a[:, 0] = -b[:, 0]
        b[:, 1] = 0.0
        out["sloppy_a"], out["sloppy_b"] = a, b
        out["sloppy_out"] = np.stack(multiword.dw_add_sloppy(tuple(a), tuple(b)))
        a, b = rand_mw(rng, 3, W), rand_mw(rng, 3, W)
        b[:, 1] = 0.0
        b[:, 2] = 1.0
        a[:, 3] = 0.0
        out["cleaned_a"], out["cleaned_b"] = a, b
        out["cleaned_out"] = np.array([multiword.tw_mul_cleaned(tuple(a[:, i]), tuple(b[:, i]))
                                       for i in range(W)]).T
        # raw expansions: decreasing terms, zeros placed to reach every branch
        for k, m in ((3, 4), (4, 5)):
            raw = np.zeros((m, W))
            raw[0] = rng.uniform(-1, 1, W) * np.exp2(rng.integers(-60, 60, W))
            for j in range(1, m):
                raw[j] = raw[j - 1] * 2.0**-52 * rng.uniform(-1.0, 1.0, W)
            for i in range(W):
                mask = (i * 2654435761) % (1 << m)
                for j in range(1, m):
                    if mask >> j & 1:
                        raw[j, i] = 0.0
            raw[0, 0] = np.inf
            raw[:, 1] = 0.0
            fn = multiword.tw_renormalize if k == 3 else multiword.qw_renormalize
            out[f"renorm{k}_in"] = raw
            out[f"renorm{k}_out"] = np.array([fn(*(float(v) for v in raw[:, i])) for i in range(W)]).T
        for k in (2, 3, 4):
            c = rand_mw(rng, k, W)
            c[1:] *= rng.uniform(0.5, 300.0, (k - 1, W))  # overlapping components
            out[f"normalize{k}_in"] = c
            out[f"normalize{k}_out"] = np.array([multiword.normalize(tuple(float(v) for v in c[:, i]))
                                                 for i in range(W)]).T
        fa = rng.uniform(-1, 1, W) * np.exp2(rng.integers(-40, 40, W))
        fb = rng.uniform(-1, 1, W) * np.exp2(rng.integers(-40, 40, W))
        fc = -(fa * fb) * (1.0 + rng.uniform(-1e-15, 1e-15, W))  # cancellation
        fc[::3] = rng.uniform(-1, 1, len(fc[::3]))
        out["fma_a"], out["fma_b"], out["fma_c"] = fa, fb, fc
        out["fma_out"] = np.asarray(reft.fma(fa, fb, fc))
        pads = []
        for n, cut in ((1, 32), (32, 32), (33, 32), (64, 32), (100, 8), (129, 16), (4096, 128), (2047, 64)):
            for kind, size in linalg.strassen_pad_policy(n, cut):
                pads.append((n, cut, {"blocked": 0, "peel": 1, "split": 2}[kind], size))
        out["strassen_pad"] = np.array(pads, dtype=np.int64)
        np.savez_compressed(os.path.join(HERE, "named.npz"), **out)
        print(f"named done {time.time() - t0:.1f}s")

    # ------------------------------------------------------------ dk_solve
    # the full solve loop (roots.py:318-340) from the reference's own Aberth
    # start: final roots and the sweep count, on the Chebyshev test
    # polynomials (roots.py:343-368) at n = 16 for all six (K, Variant)
    # pairs and at the paper's n = 64 for TD and QD
    if want("dksolve"):
        out = {}
        cases_s = [(k, v, 16) for k, v in cases] + [(3, BF, 64), (4, BF, 64)]
        for k, v, n in cases_s:
            q = roots.chebyshev_coeffs(n, k)
            st, iters = roots.dk_solve(q, v)
            p = f"k{k}_{tag[v]}_n{n}"
            out[p + "_coeffs"] = np.stack(q.comps)
            out[p + "_re"] = np.stack(st.re)
            out[p + "_im"] = np.stack(st.im)
            out[p + "_iters"] = np.array([iters])
            out[p + "_maxupd"] = np.array([st.last_max_update])
        np.savez_compressed(os.path.join(HERE, "dksolve.npz"), **out)
        print(f"dksolve done {time.time() - t0:.1f}s")

    print(f"all done {time.time() - t0:.1f}s  (mwfloat {getattr(mwfloat, '__version__', '?')})")


if __name__ == "__main__":
    main()
