"""One launch of each hot kernel at its benchmark size (for ncu captures).

    python scripts/prof_kernels.py [--only gemm_dd,horner,...] [--warm N]

Inputs are created on the device (this is a profiling driver, not the
benchmark); each kernel runs `--warm` untimed launches then one more.
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_14926_b200 as mw  # noqa: E402
from paper_2603_14926_b200 import blas, gen  # noqa: E402
from paper_2603_14926_b200.linalg import gemm_into  # noqa: E402
from paper_2603_14926_b200.poly import horner_into  # noqa: E402

BF = mw.Variant.BRANCH_FREE


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--warm", type=int, default=1)
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))

    def want(name):
        return not only or name in only

    torch.cuda.set_device(0)
    jobs = []
    for k, n, name in ((2, 4096, "gemm_dd"), (3, 2048, "gemm_td"), (4, 2048, "gemm_qd")):
        if want(name):
            a, b = gen.config3_gemm(k, n)
            A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
            C = torch.empty_like(A)
            jobs.append((name, lambda A=A, B=B, C=C: gemm_into(A, B, C, BF)))
    if want("horner"):
        coeffs, x = gen.config4_horner()
        c, xd = torch.from_numpy(coeffs).cuda(), torch.from_numpy(x).cuda()
        y = torch.empty_like(xd)
        jobs.append(("horner", lambda: horner_into(c, xd, y, BF)))
    if want("dot") or want("axpy"):
        x, yv, alpha = gen.config1_dot()
        X, Y = mw.LaneBatch(x), mw.LaneBatch(yv)
        out = torch.empty(2, dtype=torch.float64, device="cuda")
        if want("dot"):
            jobs.append(("dot", lambda X=X, Y=Y, out=out: blas.dot_tensor(X, Y, BF, out=out)))
        if want("axpy"):
            jobs.append(("axpy", lambda X=X, Y=Y: blas.axpy_(tuple(alpha), X, Y, BF)))
    for k in (3, 4):
        name = f"gemv_{'td' if k == 3 else 'qd'}"
        if want(name):
            a, x = gen.config2_gemv(k)
            A, X = mw.MWMatrix(a), mw.LaneBatch(x)
            jobs.append((name, lambda A=A, X=X: blas.gemv(A, X, BF, order="tree")))
    for k in (3, 4):
        name = f"dk_{'td' if k == 3 else 'qd'}"
        if want(name) or want(name + "_exact"):
            q = mw.MonicPoly(gen.config5_poly(k))
            zre, zim = gen.config5_init(k)
            st = mw.RootState(re=zre, im=zim)
            if want(name):
                jobs.append((name, lambda q=q, st=st: mw.dk_sweeps(q, st, 1, BF, exact_order=False, check=False)))
            if want(name + "_exact"):
                jobs.append((name + "_exact", lambda q=q, st=st: mw.dk_sweeps(q, st, 1, BF, exact_order=True, check=False)))
    if want("dk_td_peer"):
        from paper_2603_14926_b200 import dist as mwdist

        coeffs = torch.from_numpy(gen.config5_poly(3)).cuda()
        zre, zim = (torch.from_numpy(t).cuda() for t in gen.config5_init(3))
        pg = mwdist.DKPeerGraph(coeffs, zre, zim, 2, BF, exact_order=False)
        jobs.append(("dk_td_peer", pg.replay))
    if want("estrin_qd"):
        coeffs, x = gen.config4_horner(npts=1 << 20)
        P, X = mw.MWPolynomial(coeffs), mw.LaneBatch(x)
        jobs.append(("estrin_qd", lambda P=P, X=X: mw.estrin_eval_batched(P, X, BF)))
    if want("ew_qd_mul"):
        rng = np.random.default_rng(0)
        a, b = mw.LaneBatch(gen.g_k(rng, 4, 1 << 24)), mw.LaneBatch(gen.g_k(rng, 4, 1 << 24))
        jobs.append(("ew_qd_mul", lambda a=a, b=b: mw.batch_mul(a, b, BF)))
    for name, fn in jobs:
        for _ in range(args.warm):
            fn()
        fn()
        torch.cuda.synchronize()
        print("ran", name, flush=True)


if __name__ == "__main__":
    main()
