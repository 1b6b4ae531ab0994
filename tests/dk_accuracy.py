"""Accuracy contract of the tree-order Durand-Kerner sweep (test helper).

The reference sweep (``dk_iterate``, roots.py:240-315) computes, for every
root i from the frozen state z,

    z_i' = z_i - q(z_i) / prod_{j != i} (z_i - z_j)

with the numerator by Horner (272-276) and the denominator as an ordered
product (279-293).  The tree order regroups both folds, so its rounding
errors differ.  The bound used here is condition-aware: a K-word fold of n
terms perturbs q(z_i) by at most ~ n 2^-p sum_j |c_j| |z_i|^j (c_n = 1) and
the product by a relative ~ n 2^-p, so the step moves by at most

    B_i = n 2^-p (sum_j |c_j| |z_i|^j) / |prod_{j != i} (z_i - z_j)|

plus the final subtraction's rounding, 2^(1-p) |z_i|.  SURVEY §8(d)(i)'s
size-only bound n 2^(-p+4) |step| + 2^-p |z| is NOT met on the config-5
polynomial by the reference itself (|q'(r_i)| spans 1e-102 .. 1e20: the
reference's own step differs from the exact step by far more than
n 2^-p |step| on the ill-conditioned roots), so the contract is stated
against B_i with a constant C_TREE.

``exact_step`` evaluates the same update with mpmath at ``prec`` bits (the
north star's mpmath oracle); at 2400 bits its own error is negligible
against 2^-212 times any condition number of this problem.
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

P_BITS = {2: 106, 3: 159, 4: 212}
C_TREE = 2.0  # stated constant: |z_tree - z_ref| <= C_TREE * B_i + 2^(1-p) |z_i|
EXACT_FACTOR = 10.0  # tree error vs the exact step <= 10 x the reference's own error


def leading_complex(zre, zim) -> np.ndarray:
    return np.asarray(zre)[0] + 1j * np.asarray(zim)[0]


def cond_bound(coeffs, zre, zim) -> np.ndarray:
    """B_i for every root (float64, evaluated in log space: the sums and
    products over- and underflow binary64 at n = 512)."""
    coeffs = np.asarray(coeffs)
    k, n = coeffs.shape
    p = P_BITS[k]
    c_abs = np.abs(coeffs.sum(axis=0))  # |c_j| from its K words (enough for a bound)
    z = leading_complex(zre, zim)
    logz = np.log(np.abs(z))
    with np.errstate(divide="ignore"):
        logc = np.concatenate([np.log(c_abs), [0.0]])  # c_n = 1 (monic)
    j = np.arange(n + 1)
    terms = logc[None, :] + j[None, :] * logz[:, None]  # (n roots, n+1 terms)
    mx = terms.max(axis=1)
    log_num = mx + np.log(np.exp(terms - mx[:, None]).sum(axis=1))
    d = np.abs(z[:, None] - z[None, :])
    np.fill_diagonal(d, 1.0)
    log_den = np.log(d).sum(axis=1)
    return np.exp(math.log(n) - p * math.log(2.0) + log_num - log_den)


def kword_value(planes, i) -> Fraction:
    return sum((Fraction(float(c)) for c in np.asarray(planes)[:, i]), Fraction(0))


def diff_mag(are, aim, bre, bim) -> np.ndarray:
    """|a_i - b_i| per root, a and b K-word complex planes, differences exact."""
    n = np.asarray(are).shape[1]
    out = np.empty(n)
    for i in range(n):
        dr = kword_value(are, i) - kword_value(bre, i)
        di = kword_value(aim, i) - kword_value(bim, i)
        out[i] = math.hypot(float(dr), float(di))
    return out


def contract_ratio(coeffs, zre, zim, tre, tim, rre, rim):
    """Per root |z_tree - z_ref| / (B_i + 2^(1-p)|z_i|); returns (ratios, B)."""
    k = np.asarray(coeffs).shape[0]
    b = cond_bound(coeffs, zre, zim)
    z = np.abs(leading_complex(rre, rim))
    floor = math.ldexp(1.0, 1 - P_BITS[k]) * z
    d = diff_mag(tre, tim, rre, rim)
    with np.errstate(invalid="ignore", divide="ignore"):
        ratio = np.where(d == 0.0, 0.0, d / (b + floor))
    return ratio, b


def exact_step(coeffs, zre, zim, i, prec=2400):
    """z_i - q(z_i) / prod_{j != i}(z_i - z_j) at ``prec`` bits (mpmath);
    inputs taken exactly from their K words.  Returns an mpc."""
    import mpmath

    ctx = mpmath.MPContext()
    ctx.prec = prec
    coeffs = np.asarray(coeffs)
    zre, zim = np.asarray(zre), np.asarray(zim)
    k, n = coeffs.shape

    def val(planes, idx):
        return ctx.fsum(ctx.mpf(float(c)) for c in planes[:, idx])

    zs = [ctx.mpc(val(zre, j), val(zim, j)) for j in range(n)]
    cs = [val(coeffs, j) for j in range(n)]
    zi = zs[i]
    acc = ctx.mpc(1)
    for j in range(n - 1, -1, -1):
        acc = acc * zi + cs[j]
    den = ctx.mpc(1)
    for j in range(n):
        if j != i:
            den *= zi - zs[j]
    return zi - acc / den, ctx


def exact_errors(coeffs, zre, zim, tre, tim, rre, rim, idx, prec=2400):
    """For roots idx: (|z_tree - z_exact|, |z_ref - z_exact|, |z_exact|)."""
    out = []
    for i in idx:
        ex, ctx = exact_step(coeffs, zre, zim, int(i), prec)

        def err(re, im):
            v = ctx.mpc(ctx.fsum(ctx.mpf(float(c)) for c in np.asarray(re)[:, i]),
                        ctx.fsum(ctx.mpf(float(c)) for c in np.asarray(im)[:, i]))
            return float(abs(v - ex))

        out.append((err(tre, tim), err(rre, rim), float(abs(ex))))
    return out
