"""Small invocations of every kernel family (for compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__ as g
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import blas, gen, poly, linalg
g.smoke()
rng = np.random.default_rng(0)
BF, STD = mw.Variant.BRANCH_FREE, mw.Variant.STANDARD
for k in (2, 3, 4):
    for v in (BF, STD):
        a, b = gen.g_k(rng, k, (37, 29)), gen.g_k(rng, k, (29, 41))
        mw.matmul(mw.MWMatrix(a), mw.MWMatrix(b), mw.MatMulPlan(scheme="naive", variant=v))
        s = gen.g_k(rng, k, (37, 37))
        mw.matmul(mw.MWMatrix(s), mw.MWMatrix(s), mw.MatMulPlan(scheme="strassen", variant=v, strassen_cutoff=8))
        x = mw.LaneBatch(gen.g_k(rng, k, 5001)); y = mw.LaneBatch(gen.g_k(rng, k, 5001))
        for fn in (mw.batch_add, mw.batch_sub, mw.batch_mul, mw.batch_div):
            fn(x, y, v)
        blas.dot(x, y, v); blas.dot(x, y, v, order="exact"); blas.axpy((1.0,) + (0.0,) * (k - 1), x, y, v)
        A = mw.MWMatrix(gen.g_k(rng, k, (33, 5001)))
        blas.gemv(A, x, v); blas.gemv(A, x, v, order="exact")
        P = mw.MWPolynomial(gen.g_k(rng, k, 300))
        mw.horner_eval_batched(P, x, v); poly.estrin_eval_batched(P, x, v)
        poly.eval_complex_batched(P, x, y, "horner", v); poly.eval_complex_batched(P, x, y, "estrin", v)
        q = mw.MonicPoly(gen.g_k(rng, k, 40) * 0.5)
        ang = 2 * np.pi * np.arange(40) / 40 + 0.1
        zr = np.zeros((k, 40)); zi = np.zeros((k, 40)); zr[0] = 1.3 * np.cos(ang); zi[0] = 1.3 * np.sin(ang)
        st = mw.RootState(re=zr, im=zi)
        mw.dk_iterate(q, st, v, exact_order=True); mw.dk_iterate(q, st, v, exact_order=False)
        linalg.cmatmul(*linalg.gen_complex_test_matrices(9, 1, k), mw.MatMulPlan(scheme="naive", variant=v))
xs = mw.LaneBatch(gen.g_k(rng, 2, 70000)); blas.dot(xs, xs, BF)
torch.cuda.synchronize()
print("sanitize run ok")
