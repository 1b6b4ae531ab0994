"""GPU numerics beyond bit-parity: the reference's own accuracy and
behaviour tests, run through this package's API on the device.

Mirrors pkg/tests/test_multiword.py (error-bound sweeps, BF vs Standard),
test_linalg.py / verify.py (matmul digit floors on the paper's sqrt(5)/
sqrt(3) matrices), test_poly.py (degree-15 Horner vs the
exact value) and test_roots.py (residual decrease, clustered roots,
determinism, NoConvergence, Standard/BF iteration parity).
"""

import math
from fractions import Fraction

import numpy as np
import pytest
import torch

from conftest import assert_bitwise, rand_mw
from paper_2603_14926_b200 import (
    LaneBatch,
    MatMulPlan,
    MonicPoly,
    MWPolynomial,
    Variant,
    batch_add,
    batch_div,
    batch_mul,
    horner_eval,
    matmul,
    random_polynomial,
)
from paper_2603_14926_b200 import linalg, roots

pytestmark = pytest.mark.gpu

BITS = {2: 106, 3: 159, 4: 212}
CASES = [(k, v) for k in (2, 3, 4) for v in (Variant.BRANCH_FREE, Variant.STANDARD)]
IDS = [f"k{k}_{v.value}" for k, v in CASES]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def exact(comps) -> Fraction:
    return sum(Fraction(float(c)) for c in comps)


def rel_err(got, want: Fraction) -> float:
    if want == 0:
        return abs(float(exact(got)))
    return abs(float((exact(got) - want) / want))


@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_error_bound_sweep(k, v):
    """add / mul / div within 2^(-b+4) of the exact result
    (test_multiword.py:107-113, 172-178; acceptance bound sweeps)."""
    rng = np.random.default_rng(4242 + k)
    w = 1500
    a, b = rand_mw(rng, k, w), rand_mw(rng, k, w)
    la, lb = LaneBatch(a), LaneBatch(b)
    s, p, q = batch_add(la, lb, v).numpy(), batch_mul(la, lb, v).numpy(), batch_div(la, lb, v).numpy()
    bound = 2.0 ** (-BITS[k] + 4)
    for i in range(0, w, 7):
        ea, eb = exact(a[:, i]), exact(b[:, i])
        assert rel_err(s[:, i], ea + eb) <= bound
        assert rel_err(p[:, i], ea * eb) <= bound
        assert rel_err(q[:, i], ea / eb) <= bound * 4


@pytest.mark.parametrize("k", [2, 3, 4])
def test_bf_vs_standard_within_bound(k):
    """test_multiword.py:189-204: BF and Standard agree to 2^(-b+5)."""
    rng = np.random.default_rng(99 + k)
    a, b = rand_mw(rng, k, 3000), rand_mw(rng, k, 3000)
    la, lb = LaneBatch(a), LaneBatch(b)
    for fn in (batch_add, batch_mul):
        x = fn(la, lb, Variant.BRANCH_FREE).numpy()
        y = fn(la, lb, Variant.STANDARD).numpy()
        for i in range(0, 3000, 11):
            ey = exact(y[:, i])
            if ey:
                assert abs(float((exact(x[:, i]) - ey) / ey)) <= 2.0 ** (-BITS[k] + 5)


def _exact_matmul(a: np.ndarray, b: np.ndarray):
    """Exact product of K-word matrices on a common power-of-two scale."""
    def to_int(m):
        fr = [[sum(Fraction(float(c)) for c in m[:, i, j]) for j in range(m.shape[2])] for i in range(m.shape[1])]
        den = 1
        for row in fr:
            for x in row:
                den = max(den, x.denominator)
        return np.array([[int(x * den) for x in row] for row in fr], dtype=object), den

    ai, ad = to_int(a)
    bi, bd = to_int(b)
    return ai.dot(bi), ad * bd


REAL_FLOORS = {2: 29.0, 3: 45.5, 4: 61.7}  # verify.py:285


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("variant", ["std", "bf"])
@pytest.mark.parametrize("scheme", ["naive", "strassen"])
def test_matmul_digit_floors(k, variant, scheme):
    """The paper's accuracy benchmark at n = 64: significant decimal digits
    of every entry of A B vs the exact product stay above the reference's
    floors 29.0 / 45.5 / 61.7 (verify.check_matmul_digit_floors)."""
    n = 64
    a, b = linalg.gen_test_matrices(n, k)
    c = matmul(a, b, MatMulPlan(scheme=scheme, variant=variant)).numpy()
    num, den = _exact_matmul(a.numpy(), b.numpy())
    worst = math.inf
    for i in range(0, n, 3):
        for j in range(0, n, 5):
            ex = Fraction(int(num[i, j]), den)
            d = abs(exact(c[:, i, j]) - ex)
            digits = 80.0 if d == 0 else -math.log10(float(d / abs(ex)))
            worst = min(worst, digits)
    assert worst >= REAL_FLOORS[k], worst


def test_gen_test_matrices_match_reference(golden):
    g = golden("testmats")
    for k in (2, 3, 4):
        a, b = linalg.gen_test_matrices(16, k)
        assert_bitwise(a.numpy(), g[f"k{k}_a"])
        assert_bitwise(b.numpy(), g[f"k{k}_b"])


@pytest.mark.parametrize("k", [2, 3, 4])
def test_horner_degree15_vs_exact(k):
    """test_poly.py:44-58: relative error <= 15 * 2^(-53K+4)."""
    p = random_polynomial(15, 333, k)
    coeffs = [exact(p.coeff(i)) for i in range(16)]
    rng = np.random.default_rng(5)
    for _ in range(20):
        xv = float(rng.uniform(-1, 1))
        got = horner_eval(p, (xv,) + (0.0,) * (k - 1), Variant.BRANCH_FREE)
        ref = Fraction(0)
        for c in reversed(coeffs):
            ref = ref * Fraction(xv) + c
        if ref:
            assert rel_err(got, ref) <= 15 * 2.0 ** (-53 * k + 4)


def test_chebyshev_coeffs_match_reference(golden):
    g = golden("testmats")
    for k in (2, 3, 4):
        assert_bitwise(roots.chebyshev_coeffs(12, k).planes.cpu().numpy(), g[f"k{k}_cheb12"])


def test_residuals_decrease_on_separated_roots():
    """test_roots.py:130-139."""
    q = roots.chebyshev_coeffs(8, 2)
    state = roots.aberth_init(q, Variant.BRANCH_FREE)
    res = []
    for _ in range(10):
        state = roots.dk_iterate(q, state, Variant.BRANCH_FREE)
        res.append(roots.residual_check(q, state.roots()))
    for a, b in zip(res[3:], res[4:]):
        assert b <= a or b < 1e-30


def test_triple_root_cluster():
    """test_roots.py:152-162: (z-1)^3 converges loosely."""
    q = MonicPoly.from_coeffs([(-1.0, 0.0), (3.0, 0.0), (-3.0, 0.0)])
    try:
        state, _ = roots.dk_solve(q, Variant.BRANCH_FREE, tol=1e-14, max_iter=400)
    except roots.NoConvergence as err:
        state = err.state
    assert roots.residual_check(q, state.roots()) <= 1e-29
    for zre, zim in state.roots():
        assert abs(zre[0] - 1.0) < 1e-8 and abs(zim[0]) < 1e-8


@pytest.mark.parametrize("exact_order", [True, False])
def test_deterministic_rerun(exact_order):
    q = roots.chebyshev_coeffs(16, 3)
    s1, i1 = roots.dk_solve(q, Variant.BRANCH_FREE, exact_order=exact_order)
    s2, i2 = roots.dk_solve(q, Variant.BRANCH_FREE, exact_order=exact_order)
    assert i1 == i2
    assert_bitwise(s1.re.cpu().numpy(), s2.re.cpu().numpy())
    assert_bitwise(s1.im.cpu().numpy(), s2.im.cpu().numpy())


def test_no_convergence_carries_state():
    q = roots.chebyshev_coeffs(8, 2)
    with pytest.raises(roots.NoConvergence) as info:
        roots.dk_solve(q, Variant.BRANCH_FREE, max_iter=2)
    assert info.value.state.iteration == 2


def test_iteration_parity_std_bf():
    q = roots.chebyshev_coeffs(16, 3)
    _, it_std = roots.dk_solve(q, Variant.STANDARD)
    _, it_bf = roots.dk_solve(q, Variant.BRANCH_FREE)
    assert abs(it_std - it_bf) <= 1


def test_tree_dk_converges_like_exact():
    """The reordered (tree) sweep reaches the same roots to working
    precision on a well-separated problem."""
    q = roots.chebyshev_coeffs(16, 4)
    se, _ = roots.dk_solve(q, Variant.BRANCH_FREE, exact_order=True)
    st, _ = roots.dk_solve(q, Variant.BRANCH_FREE, exact_order=False)
    # (sorted on keys rounded well above the noise: parts that are zero come
    # out as +-1e-60-size values whose sign is not reproducible across orders)
    key = lambda r: (round(r[0], 10) + 0.0, round(r[1], 10) + 0.0)
    a = sorted(((r[0][0], r[1][0]) for r in se.roots()), key=key)
    b = sorted(((r[0][0], r[1][0]) for r in st.roots()), key=key)
    for (x0, y0), (x1, y1) in zip(a, b):
        assert abs(x0 - x1) < 1e-14 and abs(y0 - y1) < 1e-14


def _exact_pair_ok(a, b, s, e, op):
    fa, fb, fs, fe = (Fraction(float(v)) for v in (a, b, s, e))
    return (fa + fb if op == "add" else fa * fb) == fs + fe


def test_eft_exactness_wide_exponent_sweep():
    """two_sum / two_prod exactness through the device kernels
    (test_eft.py:60-72, 85-89): DD add/mul of (a, 0) and (b, 0) must return
    s + e == a + b and p + e == a * b exactly, over a wide exponent sweep."""
    rng = np.random.default_rng(20240809)
    n = 20000
    def draw(lo, hi):
        m = rng.uniform(1, 2, n) * np.exp2(rng.integers(lo, hi, n))
        return m * np.where(rng.random(n) < 0.5, -1, 1)
    a, b = draw(-500, 501), draw(-500, 501)
    A = np.stack([a, np.zeros(n)])
    B = np.stack([b, np.zeros(n)])
    s = batch_add(LaneBatch(A), LaneBatch(B), Variant.BRANCH_FREE).numpy()
    for i in range(0, n, 13):
        assert _exact_pair_ok(a[i], b[i], s[0, i], s[1, i], "add")
    a, b = draw(-140, 141), draw(-140, 141)  # two_prod contract: |ab| well above subnormal
    A = np.stack([a, np.zeros(n)])
    B = np.stack([b, np.zeros(n)])
    p = batch_mul(LaneBatch(A), LaneBatch(B), Variant.BRANCH_FREE).numpy()
    for i in range(0, n, 13):
        assert _exact_pair_ok(a[i], b[i], p[0, i], p[1, i], "mul")


def _dk_solve_stepwise(q, variant, tol, max_iter, exact_order):
    """The reference loop (roots.py:318-340): one dk_iterate per sweep and
    the convergence test after each."""
    state = roots.aberth_init(q, variant)
    for _ in range(max_iter):
        state = roots.dk_iterate(q, state, variant, exact_order)
        zmag = float(torch.max(torch.hypot(state.re[0], state.im[0])).item())
        if state.last_max_update <= tol * max(zmag, 1e-300):
            return state, state.iteration
    raise roots.NoConvergence("", state)


@pytest.mark.parametrize("exact_order", [True, False])
@pytest.mark.parametrize("k,deg", [(2, 8), (3, 16), (4, 12)])
def test_dk_solve_chunked_equals_stepwise_loop(k, deg, exact_order):
    """dk_solve's chunked device loop returns exactly the state and sweep
    count of the sweep-by-sweep reference loop."""
    q = roots.chebyshev_coeffs(deg, k)
    tol = roots.default_tolerance(k)
    want, wi = _dk_solve_stepwise(q, Variant.BRANCH_FREE, tol, 200, exact_order)
    got, gi = roots.dk_solve(q, Variant.BRANCH_FREE, tol=tol, exact_order=exact_order)
    assert gi == wi and got.converged
    assert_bitwise(got.re.cpu().numpy(), want.re.cpu().numpy())
    assert_bitwise(got.im.cpu().numpy(), want.im.cpu().numpy())
    assert got.last_max_update == want.last_max_update
    # a budget that ends mid-chunk: NoConvergence carries the last state
    cut = max(1, wi - 2)
    with pytest.raises(roots.NoConvergence) as info:
        roots.dk_solve(q, Variant.BRANCH_FREE, tol=tol, max_iter=cut, exact_order=exact_order)
    ref = roots.dk_sweeps(q, roots.aberth_init(q, Variant.BRANCH_FREE), cut, Variant.BRANCH_FREE, exact_order)
    assert info.value.state.iteration == cut
    assert_bitwise(info.value.state.re.cpu().numpy(), ref.re.cpu().numpy())


def _scaled_ints(planes: np.ndarray, scale_bits: int) -> list:
    """Each lane's K-word value times 2^scale_bits as an exact Python int."""
    k, n = planes.shape
    m, e = np.frexp(planes)
    mant = (m * 2.0**53).astype(np.int64)  # exact: |m| < 1, 53-bit significands
    out = [0] * n
    for c in range(k):
        for i in range(n):
            if mant[c, i]:
                sh = scale_bits + int(e[c, i]) - 53
                out[i] += (int(mant[c, i]) << sh) if sh >= 0 else (int(mant[c, i]) >> -sh)
    return out


@pytest.mark.parametrize("k", [2, 3, 4])
def test_tree_reductions_vs_exact_sum(k):
    """The throughput (tree) orders of dot and GEMV against the EXACT
    result (integer arithmetic on a common power-of-two scale -- an
    exact oracle, stronger than a fixed-precision mpmath one): within
    n 2^(-p+4) sum|x||y| (the |A||B|-scale bound of verify.py:369-381), and
    normwise (error / sum|x||y|) no worse than 8x the reference order's
    worst own error over the same samples (or 2^-p)."""
    from paper_2603_14926_b200 import blas, gen

    S = 1400
    p = BITS[k]
    rng = np.random.default_rng(700 + k)
    n = 65536
    x, y = gen.g_k(rng, k, n), gen.g_k(rng, k, n)
    X, Y = LaneBatch(x), LaneBatch(y)
    xi, yi = _scaled_ints(x, S), _scaled_ints(y, S)
    ex = Fraction(sum(a * b for a, b in zip(xi, yi)), 1 << (2 * S))
    mag = Fraction(sum(abs(a * b) for a, b in zip(xi, yi)), 1 << (2 * S))
    tree = exact(np.array(blas.dot(X, Y, Variant.BRANCH_FREE, order="tree")))
    ref = exact(np.array(blas.dot(X, Y, Variant.BRANCH_FREE, order="exact")))
    bound = n * Fraction(2) ** (-p + 4) * mag
    assert abs(tree - ex) <= bound
    assert abs(tree - ex) / mag <= 8 * max(abs(ref - ex) / mag, Fraction(2) ** (-p))
    # GEMV rows (config-2 shape, sampled rows) the same way
    m = 2048
    a, xv = gen.g_k(rng, k, (64, m)), gen.g_k(rng, k, m)
    A, XV = linalg.MWMatrix(a), LaneBatch(xv)
    yt = blas.gemv(A, XV, Variant.BRANCH_FREE, "tree").numpy()
    ye = blas.gemv(A, XV, Variant.BRANCH_FREE, "exact").numpy()
    xs = _scaled_ints(xv, S)
    worst_t = worst_r = Fraction(0)
    for r in range(0, 64, 3):
        ar = _scaled_ints(np.ascontiguousarray(a[:, r]), S)
        e_r = Fraction(sum(u * v for u, v in zip(ar, xs)), 1 << (2 * S))
        g_r = Fraction(sum(abs(u * v) for u, v in zip(ar, xs)), 1 << (2 * S))
        t_err, r_err = abs(exact(yt[:, r]) - e_r), abs(exact(ye[:, r]) - e_r)
        assert t_err <= m * Fraction(2) ** (-p + 4) * g_r
        worst_t, worst_r = max(worst_t, t_err / g_r), max(worst_r, r_err / g_r)
    assert worst_t <= 8 * max(worst_r, Fraction(2) ** (-p))
