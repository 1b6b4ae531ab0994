"""Seeded synthetic inputs for the benchmark configurations.

The reference publishes no datasets; every config in BASELINE.json is a
seeded synthetic draw, restated here once so the GPU path, the CPU oracle
and the reference itself see identical arrays.

``g_k(rng, k, shape)``  (input generator G_K):
    c0 = U[-1, 1); c_j = c0 * 2^(-53 j) * U[-1, 1) for j = 1..K-1, drawn in
    that order; then one bottom-up quick_two_sum pass
    (c_{K-2}, c_{K-1}) = qts(c_{K-2}, c_{K-1}), ..., (c0, c1) = qts(c0, c1)
    -- for DD exactly config 1's QuickTwoSum(hi, lo); the same first phase
    as qw_renormalize (multiword.py:204-207).
Arrays are K x shape float64, component-planar.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

__all__ = [
    "g_k",
    "config1_dot",
    "config2_gemv",
    "config3_gemm",
    "config4_horner",
    "config5_roots",
    "config5_poly",
    "config5_init",
    "round_fraction",
]


def _qts(a, b):
    s = a + b
    e = b - (s - a)
    return s, e


def g_k(rng: np.random.Generator, k: int, shape) -> np.ndarray:
    shape = (shape,) if isinstance(shape, int) else tuple(shape)
    c0 = rng.uniform(-1.0, 1.0, shape)
    comps = [c0]
    for j in range(1, k):
        comps.append(c0 * 2.0 ** (-53 * j) * rng.uniform(-1.0, 1.0, shape))
    for j in range(k - 2, -1, -1):
        comps[j], comps[j + 1] = _qts(comps[j], comps[j + 1])
    return np.ascontiguousarray(np.stack(comps))


def config1_dot(n: int = 65536, seed: int = 0):
    """DD x, y = G_2(n) drawn x then y; alpha = G_2(1) drawn after."""
    rng = np.random.default_rng(seed)
    x = g_k(rng, 2, n)
    y = g_k(rng, 2, n)
    alpha = g_k(rng, 2, 1)[:, 0].copy()
    return x, y, alpha


def config2_gemv(k: int, n: int = 2048, seed: int = 0):
    """A = G_K(n x n), then x = G_K(n)."""
    rng = np.random.default_rng(seed)
    a = g_k(rng, k, (n, n))
    x = g_k(rng, k, n)
    return a, x


def config3_gemm(k: int, n: int, seed: int = 0):
    """A = G_K(n x n), then B = G_K(n x n)."""
    rng = np.random.default_rng(seed)
    a = g_k(rng, k, (n, n))
    b = g_k(rng, k, (n, n))
    return a, b


def config4_horner(npts: int = 1 << 24, degree: int = 1024, k: int = 4, seed: int = 0):
    """QD coefficients G_4(degree+1) (a_i low to high), then points
    x ~ U[-1.1, 1.1) as (x, 0, 0, 0)."""
    rng = np.random.default_rng(seed)
    coeffs = g_k(rng, k, degree + 1)
    x0 = rng.uniform(-1.1, 1.1, npts)
    x = np.zeros((k, npts))
    x[0] = x0
    return coeffs, x


# ------------------------------------------------------------ config 5
def config5_roots(n: int = 512, seed: int = 0) -> np.ndarray:
    """256 roots uniform in the upper half disk plus their conjugates
    (SURVEY §8(d) config 5): rad = sqrt(U[0,1)), then th = U[0, pi)."""
    if n % 2:
        raise ValueError("n must be even (conjugate pairs)")
    rng = np.random.default_rng(seed)
    half = n // 2
    rad = np.sqrt(rng.uniform(0.0, 1.0, half))
    th = rng.uniform(0.0, np.pi, half)
    r = rad * np.exp(1j * th)
    return np.concatenate([r, np.conj(r)])


def _dyadic(x: float):
    """x = m * 2^e exactly, m an int."""
    num, den = float(x).as_integer_ratio()
    return num, -(den.bit_length() - 1)


def round_fraction(value: Fraction, k: int):
    """Greedy nearest-double K-word rounding (multiword.from_oracle,
    multiword.py:760-775)."""
    out = []
    fr = Fraction(value)
    for _ in range(k):
        c = float(fr)  # correctly rounded
        out.append(c)
        fr -= Fraction(c)
    return tuple(out)


def config5_poly(k: int, n: int = 512, seed: int = 0) -> np.ndarray:
    """Monic coefficients c_0..c_{n-1} of prod (z^2 - 2 Re r z + |r|^2) over
    the upper-half roots, expanded exactly and rounded per coefficient to K
    words.  Exact arithmetic uses integers on a common power-of-two scale
    (the roots are binary64, so every coefficient is dyadic)."""
    roots = config5_roots(n, seed)[: n // 2]
    # every quadratic coefficient as an integer times 2^E with one shared E
    quads = []
    emin = 0
    for r in roots:
        a1 = -2.0 * r.real  # exact (power-of-two scaling)
        re_m, re_e = _dyadic(r.real)
        im_m, im_e = _dyadic(r.imag)
        # |r|^2 = re^2 + im^2 exactly: (re_m^2 2^(2re_e) + im_m^2 2^(2im_e))
        e2 = min(2 * re_e, 2 * im_e)
        m2 = (re_m * re_m << (2 * re_e - e2)) + (im_m * im_m << (2 * im_e - e2))
        m1, e1 = _dyadic(a1)
        quads.append(((m2, e2), (m1, e1)))
        emin = min(emin, e2, e1)
    E = emin
    # With u = 2^scale, every a_j = int_j / u exactly, and
    # P(z) = prod (z^2 + a1 z + a0) = U(z) / u^m where
    # U(z) = prod (u z^2 + int1 z + int0) has integer coefficients.
    scale = -E
    qi = [(m2 << (e2 - E), m1 << (e1 - E)) for (m2, e2), (m1, e1) in quads]
    poly = [1]  # U coefficients, low to high
    for a0, a1 in qi:
        u = 1 << scale
        newp = [0] * (len(poly) + 2)
        for i, c in enumerate(poly):
            if c == 0:
                continue
            newp[i] += c * a0
            newp[i + 1] += c * a1
            newp[i + 2] += c * u
        poly = newp
    m = len(qi)
    den = 1 << (scale * m)
    coeffs = np.zeros((k, n))
    for i in range(n):
        comps = round_fraction(Fraction(poly[i], den), k)
        for c in range(k):
            coeffs[c, i] = comps[c]
    return coeffs


def config5_init(k: int, n: int = 512, seed: int = 0, noise_seed: int = 1):
    """Near-root start z_j = r_j (1 + 1e-3 (u_j + i v_j)) with
    g = default_rng(1), u then v ~ U[-1, 1) (SURVEY §8(d) recipe (ii)),
    rounded to K words as (value, 0, ...).  Returns (re, im) K x n."""
    r = config5_roots(n, seed)
    g = np.random.default_rng(noise_seed)
    u = g.uniform(-1.0, 1.0, n)
    v = g.uniform(-1.0, 1.0, n)
    z = r * (1.0 + 1e-3 * (u + 1j * v))
    re = np.zeros((k, n))
    im = np.zeros((k, n))
    re[0] = z.real
    im[0] = z.imag
    return re, im
