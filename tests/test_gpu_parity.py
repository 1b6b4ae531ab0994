"""GPU parity: the CUDA path (through the C-ABI) vs the reference's golden
vectors and the pinned CPU oracle, on identical seeded inputs.

Bar (BASELINE.json north_star): bit-exact wherever the reference's order
and FMA use are replicated (elementwise, axpy, GEMM, Horner, exact-order
dot/GEMV/DK); reordered reductions (tree dot/GEMV/DK) bit-exact with the
oracle's restatement of their documented tree AND within
n * 2^(-p+4) * sum|a||b| of the reference order.
"""

import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_bitwise, rand_mw
from paper_2603_14926_b200 import (
    LaneBatch,
    MatMulPlan,
    MonicPoly,
    MWMatrix,
    MWPolynomial,
    RootState,
    Variant,
    batch_add,
    batch_div,
    batch_mul,
    batch_sub,
    dk_iterate,
    dk_sweeps,
    gen,
    horner_eval,
    horner_eval_batched,
    matmul,
)
from paper_2603_14926_b200 import blas, poly as mwpoly, roots

pytestmark = pytest.mark.gpu

CASES = [(2, "bf"), (3, "bf"), (4, "bf"), (2, "std"), (3, "std"), (4, "std")]
IDS = [f"k{k}_{v}" for k, v in CASES]
P_BITS = {2: 106, 3: 159, 4: 212}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def V(v):
    return Variant.parse(v)


def exact_value(comps):
    return sum(Fraction(float(c)) for c in comps)


# ------------------------------------------------------------ elementwise
@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_ew_golden(golden, k, v):
    g = golden("ew")
    p = f"k{k}_{v}"
    a, b = LaneBatch(g[p + "_a"]), LaneBatch(g[p + "_b"])
    assert_bitwise(batch_add(a, b, V(v)).numpy(), g[p + "_add"])
    assert_bitwise(batch_sub(a, b, V(v)).numpy(), g[p + "_sub"])
    assert_bitwise(batch_mul(a, b, V(v)).numpy(), g[p + "_mul"])
    d = batch_div(a, LaneBatch(g[p + "_bz"]), V(v)).numpy()
    assert_bitwise(d, g[p + "_div"], nan_ok=True)
    assert not np.isfinite(d[0, 5])


@pytest.mark.parametrize("k,v", CASES, ids=IDS)
@pytest.mark.parametrize("w", [1, 2, 7, 1 << 20])
def test_ew_vs_oracle(k, v, w):
    rng = np.random.default_rng(1000 + k + w)
    a, b = rand_mw(rng, k, w), rand_mw(rng, k, w)
    la, lb = LaneBatch(a), LaneBatch(b)
    for op, fn in (("add", batch_add), ("sub", batch_sub), ("mul", batch_mul), ("div", batch_div)):
        assert_bitwise(fn(la, lb, V(v)).numpy(), oracle.ew(op, a, b, v))


def test_ew_unaligned_and_strided_planes():
    """Odd offsets force the 64-bit path; results identical."""
    k = 4
    rng = np.random.default_rng(5)
    a, b = rand_mw(rng, k, 1001), rand_mw(rng, k, 1001)
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b).cuda()
    big = torch.zeros((k, 1003), dtype=torch.float64, device="cuda")
    big[:, 1:1002] = ta
    la = LaneBatch(big[:, 1:1002].contiguous())
    got = batch_add(la, LaneBatch(tb), Variant.BRANCH_FREE).numpy()
    assert_bitwise(got, oracle.ew("add", a, b, "bf"))


def test_ew_kats():
    one = lambda *vals: LaneBatch(np.array(vals + (0.0,) * (4 - len(vals))).reshape(4, 1))
    r = batch_mul(one(2.0**30 + 1), one(2.0**30 + 1), Variant.BRANCH_FREE).lane(0)
    assert r[0] == 2.0**60 + 2.0**31 and r[1] == 1.0
    r = batch_mul(one(2.0), one(3.0), Variant.BRANCH_FREE).lane(0)
    assert r == (6.0, 0.0, 0.0, 0.0)


@pytest.mark.parametrize("k", [3, 4])
def test_ew_standard_renormalising_vs_oracle(k):
    """Standard TD/QD (branchy renormalisation, multiword.py:164-513) on
    wide-exponent inputs, zeros, cancellations and infinities."""
    rng = np.random.default_rng(77 + k)
    a, b = rand_mw(rng, k, 50000), rand_mw(rng, k, 50000)
    a[:, :100] = -b[:, :100]          # exact cancellation
    b[:, 100:200] = 0.0               # zero operand
    a[1:, 200:300] = 0.0              # short expansions
    a[0, 300] = np.inf
    la, lb = LaneBatch(a), LaneBatch(b)
    for op, fn in (("add", batch_add), ("sub", batch_sub), ("mul", batch_mul)):
        assert_bitwise(fn(la, lb, Variant.STANDARD).numpy(), oracle.ew(op, a, b, "std"), nan_ok=True)


def test_ew_mixed_k_raises():
    with pytest.raises(ValueError):
        batch_add(LaneBatch(np.zeros((2, 4))), LaneBatch(np.zeros((3, 4))), Variant.BRANCH_FREE)


# ------------------------------------------------------------ dot / axpy
@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_dot_exact_golden(golden, k, v):
    g = golden("dot")
    p = f"k{k}_{v}"
    got = blas.dot(LaneBatch(g[p + "_x"]), LaneBatch(g[p + "_y"]), V(v), order="exact")
    assert_bitwise(np.array(got), g[p + "_out"])


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("n", [1, 15, 16, 17, 255, 256, 257, 300, 4095, 4096, 4097, 65536, 1 << 20, 1_000_003])
def test_dot_tree_vs_oracle(k, n):
    rng = np.random.default_rng(n + k)
    x, y = gen.g_k(rng, k, n), gen.g_k(rng, k, n)
    got = np.array(blas.dot(LaneBatch(x), LaneBatch(y), Variant.BRANCH_FREE, order="tree"))
    assert_bitwise(got, oracle.dot(x, y, "bf", order=1))
    if n == 1:
        assert_bitwise(got, oracle.dot(x, y, "bf", order=0))
    if n <= 65536:
        ref = oracle.dot(x, y, "bf", order=0)
        diff = abs(exact_value(got) - exact_value(ref))
        scale = float(np.sum(np.abs(x[0] * y[0])))
        assert float(diff) <= n * 2.0 ** (-P_BITS[k] + 4) * scale


def test_dot_config1():
    x, y, alpha = gen.config1_dot()
    got = blas.dot(LaneBatch(x), LaneBatch(y), Variant.BRANCH_FREE)
    assert_bitwise(np.array(got), oracle.dot(x, y, "bf", order=1))
    exact = np.array(blas.dot(LaneBatch(x), LaneBatch(y), Variant.BRANCH_FREE, order="exact"))
    assert_bitwise(exact, oracle.dot(x, y, "bf", order=0))


@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_axpy_golden(golden, k, v):
    g = golden("axpy")
    p = f"k{k}_{v}"
    x, y = LaneBatch(g[p + "_x"]), LaneBatch(g[p + "_y"])
    got = blas.axpy(tuple(g[p + "_alpha"]), x, y, V(v))
    assert_bitwise(got.numpy(), g[p + "_out"])
    assert_bitwise(y.numpy(), g[p + "_y"])  # pure: input untouched


def test_axpy_config1():
    x, y, alpha = gen.config1_dot()
    got = blas.axpy(tuple(alpha), LaneBatch(x), LaneBatch(y), Variant.BRANCH_FREE)
    assert_bitwise(got.numpy(), oracle.axpy(alpha, x, y, "bf"))


# ------------------------------------------------------------------ gemv
@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_gemv_golden(golden, k, v):
    g = golden("gemv")
    p = f"k{k}_{v}"
    A, x = MWMatrix(g[p + "_a"]), LaneBatch(g[p + "_x"])
    assert_bitwise(blas.gemv(A, x, V(v), order="exact").numpy(), g[p + "_out"])
    assert_bitwise(blas.gemv(A, x, V(v), order="tree").numpy(), oracle.gemv(g[p + "_a"], g[p + "_x"], v, order=1))


@pytest.mark.parametrize("k", [3, 4])
def test_gemv_config2(k):
    a, x = gen.config2_gemv(k)
    A, xb = MWMatrix(a), LaneBatch(x)
    got = blas.gemv(A, xb, Variant.BRANCH_FREE, order="tree").numpy()
    assert_bitwise(got, oracle.gemv(a, x, "bf", order=1))
    ex = blas.gemv(A, xb, Variant.BRANCH_FREE, order="exact").numpy()
    ref = oracle.gemv(a, x, "bf", order=0)
    assert_bitwise(ex, ref)
    # tree vs reference order within n 2^-p+4 sum|a||x| per row
    n = a.shape[2]
    scale = np.abs(a[0]) @ np.abs(x[0])
    for i in range(0, a.shape[1], 97):
        diff = abs(exact_value(got[:, i]) - exact_value(ref[:, i]))
        assert float(diff) <= n * 2.0 ** (-P_BITS[k] + 4) * scale[i]


# ------------------------------------------------------------------ gemm
@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_gemm_golden(golden, k, v):
    g = golden("gemm")
    p = f"k{k}_{v}"
    c = matmul(MWMatrix(g[p + "_a"]), MWMatrix(g[p + "_b"]), MatMulPlan(scheme="naive", variant=v))
    assert_bitwise(c.numpy(), g[p + "_out"])


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("shape", [(1, 1, 1), (65, 33, 17), (130, 97, 200), (64, 64, 64), (5, 0, 7)])
def test_gemm_vs_oracle(k, shape):
    m, kd, n = shape
    rng = np.random.default_rng(m * 7 + kd * 3 + n + k)
    a, b = gen.g_k(rng, k, (m, kd)), gen.g_k(rng, k, (kd, n))
    c = matmul(MWMatrix(a), MWMatrix(b), MatMulPlan(scheme="naive", variant="bf"))
    assert_bitwise(c.numpy(), oracle.gemm(a, b, "bf"))


def test_gemm_identity_bitwise():
    rng = np.random.default_rng(9)
    for k in (2, 3, 4):
        a = rand_mw(rng, k, 48 * 48).reshape(k, 48, 48)
        c = matmul(MWMatrix(a), MWMatrix.identity(48, k), MatMulPlan(scheme="naive", variant="bf"))
        assert_bitwise(c.numpy(), a)


@pytest.mark.parametrize("k,n", [(2, 4096), (3, 2048), (4, 2048)])
def test_gemm_config3_sampled_rows(k, n):
    a, b = gen.config3_gemm(k, n)
    c = matmul(MWMatrix(a), MWMatrix(b), MatMulPlan(scheme="naive", variant="bf")).numpy()
    # one full row of C in every 64-row CTA tile band (64 DD rows, 32 TD/QD
    # rows), at a varying offset inside the band, plus the last row: every
    # tile row and, through the full rows, every tile column is checked
    rows = np.unique(np.r_[[band * 64 + (band * 37) % 64 for band in range(n // 64)], n - 1])
    ref = oracle.gemm(np.ascontiguousarray(a[:, rows]), b, "bf")
    assert_bitwise(c[:, rows], ref)


# ---------------------------------------------------------------- horner
@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_horner_golden(golden, k, v):
    g = golden("horner")
    p = f"k{k}_{v}"
    poly = MWPolynomial(g[p + "_coeffs"])
    got = horner_eval_batched(poly, LaneBatch(g[p + "_x"]), V(v)).numpy()
    assert_bitwise(got, g[p + "_out"])
    assert horner_eval(poly, tuple(g[p + "_x"][:, 0]), V(v)) == tuple(g[p + "_out"][:, 0])


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("deg,npts", [(0, 5), (1, 300), (255, 1000), (256, 257), (1024, 4099), (3000, 64)])
def test_horner_vs_oracle(k, deg, npts):
    rng = np.random.default_rng(deg + npts + k)
    coeffs = gen.g_k(rng, k, deg + 1)
    x = gen.g_k(rng, k, npts)
    got = horner_eval_batched(MWPolynomial(coeffs), LaneBatch(x), Variant.BRANCH_FREE).numpy()
    assert_bitwise(got, oracle.horner(coeffs, x, "bf"))


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("case", ["doubles", "zeros", "mixed", "nonfinite", "overflow"])
def test_horner_qd_double_points_fast_path(case, k):
    """TD / QD points that are plain doubles take the shortened product
    (td_/qd_mul_bf_d); the result must be the reference's bit for bit: for
    ordinary points, for exact / negative zeros in coefficients and points,
    for warps that mix double-valued and full QD points (both loop bodies
    in one CTA), and -- through the full-product re-run -- when inf / NaN
    coefficients or an overflow make a result non-finite."""
    rng = np.random.default_rng(77)
    deg, npts = 300, 5000
    coeffs = gen.g_k(rng, k, deg + 1)
    x = np.zeros((k, npts))
    x[0] = rng.uniform(-1.1, 1.1, npts)
    if case == "zeros":
        for c in range(k):
            m = rng.random(deg + 1) < 0.2
            coeffs[c] = np.where(m, np.where(rng.random(deg + 1) < 0.5, 0.0, -0.0), coeffs[c])
        m = rng.random(npts) < 0.2
        x[0] = np.where(m, np.where(rng.random(npts) < 0.5, 0.0, -0.0), x[0])
    if case == "mixed":  # every third point a full QD value, some low words -0.0
        full = gen.g_k(rng, k, npts)
        sel = (np.arange(npts) % 3) == 0
        x[:, sel] = full[:, sel]
        x[1, (np.arange(npts) % 7) == 1] = -0.0
    if case == "nonfinite":
        coeffs[0, 17] = np.inf
        coeffs[2, 120] = np.nan
        x[0, 5] = np.inf
        x[0, 77] = np.nan
    if case == "overflow":  # |x| > 1 with huge coefficients: overflows part of the way down
        coeffs = coeffs * 2.0 ** 1000
        x[0] = rng.uniform(-40, 40, npts)
    got = horner_eval_batched(MWPolynomial(coeffs), LaneBatch(x), Variant.BRANCH_FREE).numpy()
    with np.errstate(all="ignore"):
        want = oracle.horner(coeffs, x, "bf")
    if case in ("nonfinite", "overflow"):
        assert not np.all(np.isfinite(want))
    if case == "overflow":
        assert np.any(np.isfinite(want[0])) and not np.all(np.isfinite(want[0]))
    assert_bitwise(got, want, nan_ok=True)


@pytest.mark.parametrize("k", [3, 4])
def test_horner_qd_special_values_fuzz(k):
    """Randomised special values through the TD / QD Horner kernel (both step
    bodies and the non-finite re-run): coefficients and points drawn from
    ordinary values mixed with +-0, subnormals, huge and tiny magnitudes,
    inf and NaN, in any word; points double-valued or full QD.  Bitwise equal
    to the oracle (NaN positions compared, payloads not)."""
    rng = np.random.default_rng(4242 + k)
    special = np.array([0.0, -0.0, 5e-324, -2.2e-308, 1e-300, -1e300, 1.7e308, np.inf, -np.inf, np.nan,
                        1.0, -1.0, 2.0 ** -53, 2.0 ** 52 + 1])

    def draw(shape, p_special):
        v = gen.g_k(rng, k, shape)
        m = rng.random(v.shape) < p_special
        return np.where(m, rng.choice(special, v.shape), v)

    for case in range(120):
        deg = int(rng.integers(0, 48))
        npts = int(rng.integers(1, 300))
        ps = (0.0, 0.02, 0.3)[case % 3]
        coeffs = draw(deg + 1, ps)
        x = draw(npts, ps)
        mode = case % 4
        if mode in (0, 1):      # all double-valued
            x[1:] = 0.0
        elif mode == 2:         # a mix inside every warp
            dblm = rng.random(npts) < 0.6
            x[1:, dblm] = 0.0
        if mode == 1:           # grow: |x| > 1 with large coefficients overflows part of the way
            with np.errstate(all="ignore"):
                coeffs = coeffs * 2.0 ** 900
                x[0] = np.where(np.isfinite(x[0]), x[0] * 50.0, x[0])
        got = horner_eval_batched(MWPolynomial(coeffs), LaneBatch(x), Variant.BRANCH_FREE).numpy()
        with np.errstate(all="ignore"):
            want = oracle.horner(coeffs, x, "bf")
        assert_bitwise(got, want, nan_ok=True)


def test_horner_config4_full_with_sampled_check():
    coeffs, x = gen.config4_horner()
    y = horner_eval_batched(MWPolynomial(coeffs), LaneBatch(x), Variant.BRANCH_FREE).numpy()
    # 2^20 random points (every CTA's worth of points is sampled) + both ends
    rng = np.random.default_rng(4)
    idx = np.unique(np.r_[rng.choice(1 << 24, 1 << 20, replace=False), 0:256, (1 << 24) - 256:(1 << 24)])
    assert_bitwise(y[:, idx], oracle.horner(coeffs, np.ascontiguousarray(x[:, idx]), "bf"))
    assert np.all(np.isfinite(y[0]))


# -------------------------------------------------------------------- dk
@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_dk_exact_golden_small(golden, k, v):
    g = golden("dk")
    p = f"k{k}_{v}"
    q = MonicPoly(g[p + "_coeffs"])
    st = RootState(re=g[p + "_zre"], im=g[p + "_zim"])
    nxt = dk_iterate(q, st, V(v), exact_order=True)
    assert_bitwise(nxt.re.cpu().numpy(), g[p + "_new_re"])
    assert_bitwise(nxt.im.cpu().numpy(), g[p + "_new_im"])
    assert math.isclose(nxt.last_max_update, float(g[p + "_maxupd"][0]), rel_tol=1e-15)


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("init", ["near", "aberth"])
def test_dk_exact_golden_config5(golden, k, init):
    g = golden("dk")
    p = f"c5_k{k}"
    s = "" if init == "near" else "_ab"
    q = MonicPoly(g[p + "_coeffs"])
    st = RootState(re=g[p + s + "_zre"], im=g[p + s + "_zim"])
    nxt = dk_iterate(q, st, Variant.BRANCH_FREE, exact_order=True)
    assert_bitwise(nxt.re.cpu().numpy(), g[p + s + "_new_re"])
    assert_bitwise(nxt.im.cpu().numpy(), g[p + s + "_new_im"])
    assert math.isclose(nxt.last_max_update, float(g[p + s + "_maxupd"][0]), rel_tol=1e-15)


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("n", [2, 16, 33, 512])
def test_dk_tree_vs_oracle_tree(k, n):
    if n == 512:
        coeffs = gen.config5_poly(k)
        zre, zim = gen.config5_init(k)
    else:
        rng = np.random.default_rng(n + k)
        coeffs = gen.g_k(rng, k, n) * 0.5
        ang = 2 * np.pi * np.arange(n) / n + 0.1
        zre = np.zeros((k, n))
        zim = np.zeros((k, n))
        zre[0] = 1.3 * np.cos(ang)
        zim[0] = 1.3 * np.sin(ang)
    q = MonicPoly(coeffs)
    st = RootState(re=zre, im=zim)
    nxt = dk_iterate(q, st, Variant.BRANCH_FREE, exact_order=False)
    ore, oim, mag, coll = oracle.dk_sweep(coeffs, zre, zim, "bf", exact=False)
    assert coll is None
    assert_bitwise(nxt.re.cpu().numpy(), ore)
    assert_bitwise(nxt.im.cpu().numpy(), oim)


def test_dk_collision_raises():
    q = MonicPoly(np.array([[-1.0, 0.0], [0.0, 0.0]]))
    st = RootState(re=np.array([[0.5, 0.5], [0.0, 0.0]]), im=np.array([[0.1, 0.1], [0.0, 0.0]]))
    for exact in (True, False):
        with pytest.raises(roots.CollisionError):
            dk_iterate(q, st, Variant.BRANCH_FREE, exact_order=exact)


def test_dk_exact_roots_are_fixed_points():
    q = MonicPoly(np.array([[-1.0, 0.0], [0.0, 0.0]]))  # z^2 - 1
    st = RootState(re=np.array([[1.0, -1.0], [0.0, 0.0]]), im=np.zeros((2, 2)))
    new = dk_iterate(q, st, Variant.BRANCH_FREE)
    assert new.last_max_update == 0.0
    assert new.root(0) == st.root(0)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_dk_solve_quadratic(k):
    q = MonicPoly.from_coeffs([(-1.0,) + (0.0,) * (k - 1), (0.0,) * k])
    state, iters = roots.dk_solve(q, Variant.BRANCH_FREE)
    assert iters <= 10
    rs = sorted(r[0][0] for r in state.roots())
    assert abs(rs[0] + 1.0) <= 1e-30 and abs(rs[1] - 1.0) <= 1e-30


@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_aberth_init_on_device_matches_reference(golden, k, v):
    """aberth_init with the device lane ops (centre -c_{n-1}/n by the Newton
    division kernel, rotations by the mul/add kernels) reproduces the
    reference's initial state bit for bit (roots.py:188-221)."""
    g = golden("dk")
    p = f"k{k}_{v}"
    st = roots.aberth_init(MonicPoly(g[p + "_coeffs"]), V(v))
    assert st.re.is_cuda
    assert_bitwise(st.re.cpu().numpy(), g[p + "_zre"])
    assert_bitwise(st.im.cpu().numpy(), g[p + "_zim"])


@pytest.mark.parametrize("k", [3, 4])
def test_aberth_init_config5_circle_on_device(golden, k):
    """The config-5 R0 = 1.5 Aberth circle (reference centre and angles,
    SURVEY §8(d)) built on the device equals the reference's state."""
    g = golden("dk")
    p = f"c5_k{k}"
    st = roots.aberth_init(MonicPoly(g[p + "_coeffs"]), Variant.BRANCH_FREE, radius=1.5)
    assert_bitwise(st.re.cpu().numpy(), g[p + "_ab_zre"])
    assert_bitwise(st.im.cpu().numpy(), g[p + "_ab_zim"])


@pytest.mark.parametrize("exact", [True, False])
def test_dk_sweep_graph_matches_eager(exact):
    k = 3
    coeffs = gen.config5_poly(k)
    zre, zim = gen.config5_init(k)
    q, st = MonicPoly(coeffs), RootState(re=zre, im=zim)
    eager = dk_sweeps(q, st, 5, Variant.BRANCH_FREE, exact_order=exact)
    g = roots.DKSweepGraph(q, st, 5, Variant.BRANCH_FREE, exact_order=exact)
    g.replay()
    g.replay()  # replays are idempotent (state reset inside the graph)
    r = g.result()
    assert_bitwise(r.re.cpu().numpy(), eager.re.cpu().numpy())
    assert_bitwise(r.im.cpu().numpy(), eager.im.cpu().numpy())
    assert r.iteration == 5


# ------------------------------------------------- Estrin / complex eval
POLYX = [(4, "bf", 1024), (3, "bf", 100), (2, "bf", 37), (2, "std", 37), (4, "bf", 0), (3, "bf", 1),
         (3, "std", 20), (4, "std", 20)]


@pytest.mark.parametrize("k,v,deg", POLYX, ids=[f"k{k}_{v}_d{d}" for k, v, d in POLYX])
def test_estrin_complex_golden(golden, k, v, deg):
    g = golden("polyx")
    p = f"k{k}_{v}_d{deg}"
    P = MWPolynomial(g[p + "_coeffs"])
    assert_bitwise(mwpoly.estrin_eval_batched(P, LaneBatch(g[p + "_x"]), V(v)).numpy(), g[p + "_estrin"])
    assert mwpoly.estrin_eval(P, tuple(g[p + "_x"][:, 0]), V(v)) == tuple(g[p + "_estrin"][:, 0])
    for method, tag in (("horner", "ch"), ("estrin", "ce")):
        re, im = mwpoly.eval_complex_batched(P, LaneBatch(g[p + "_zre"]), LaneBatch(g[p + "_zim"]), method, V(v))
        assert_bitwise(re.numpy(), g[f"{p}_{tag}_re"])
        assert_bitwise(im.numpy(), g[f"{p}_{tag}_im"])
    z0 = (tuple(g[p + "_zre"][:, 0]), tuple(g[p + "_zim"][:, 0]))
    r = mwpoly.eval_complex(P, z0, "estrin", V(v))
    assert r == (tuple(g[p + "_ce_re"][:, 0]), tuple(g[p + "_ce_im"][:, 0]))


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("deg,npts", [(2, 100), (255, 1000), (256, 513), (1024, 4096)])
def test_estrin_complex_vs_oracle(k, deg, npts):
    rng = np.random.default_rng(deg * 3 + npts + k)
    coeffs = gen.g_k(rng, k, deg + 1)
    x = gen.g_k(rng, k, npts)
    zi = gen.g_k(rng, k, npts)
    P = MWPolynomial(coeffs)
    assert_bitwise(mwpoly.estrin_eval_batched(P, LaneBatch(x), Variant.BRANCH_FREE).numpy(),
                   oracle.poly_eval(coeffs, x, None, "bf", "estrin"))
    for method in ("horner", "estrin"):
        re, im = mwpoly.eval_complex_batched(P, LaneBatch(x), LaneBatch(zi), method, Variant.BRANCH_FREE)
        ore, oim = oracle.poly_eval(coeffs, x, zi, "bf", method)
        assert_bitwise(re.numpy(), ore)
        assert_bitwise(im.numpy(), oim)


# ------------------------------------------------------- 3M complex GEMM
@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_cmatmul_golden(golden, k, v):
    from paper_2603_14926_b200 import CMWMatrix, cmatmul

    g = golden("cgemm")
    p = f"k{k}_{v}"
    a = CMWMatrix(MWMatrix(g[p + "_a_re"]), MWMatrix(g[p + "_a_im"]))
    b = CMWMatrix(MWMatrix(g[p + "_b_re"]), MWMatrix(g[p + "_b_im"]))
    c = cmatmul(a, b, MatMulPlan(scheme="naive", variant=v))
    assert_bitwise(c.re.numpy(), g[p + "_c_re"])
    assert_bitwise(c.im.numpy(), g[p + "_c_im"])


# --------------------------------------------------------------- Strassen
STRASSEN = [(2, "bf", 37, 8), (3, "bf", 48, 8), (4, "bf", 35, 4), (2, "std", 37, 8), (3, "std", 20, 4),
            (4, "std", 18, 4), (2, "bf", 64, 32)]


@pytest.mark.parametrize("k,v,n,cut", STRASSEN, ids=[f"k{k}_{v}_n{n}_c{c}" for k, v, n, c in STRASSEN])
def test_strassen_golden(golden, k, v, n, cut):
    g = golden("strassen")
    p = f"k{k}_{v}_n{n}_c{cut}"
    c = matmul(MWMatrix(g[p + "_a"]), MWMatrix(g[p + "_b"]),
               MatMulPlan(scheme="strassen", variant=v, strassen_cutoff=cut))
    assert_bitwise(c.numpy(), g[p + "_out"])


@pytest.mark.parametrize("k,n,cut", [(2, 129, 16), (3, 100, 12), (4, 66, 8)])
def test_strassen_vs_oracle_restatement(k, n, cut):
    from test_oracle_golden import _o_strassen

    rng = np.random.default_rng(n + k)
    a, b = gen.g_k(rng, k, (n, n)), gen.g_k(rng, k, (n, n))
    c = matmul(MWMatrix(a), MWMatrix(b), MatMulPlan(scheme="strassen", variant="bf", strassen_cutoff=cut))
    assert_bitwise(c.numpy(), _o_strassen(a, b, "bf", cut))


@pytest.mark.parametrize("k,n", [(2, 33), (2, 128), (3, 33), (3, 64), (4, 33), (4, 64)])
def test_strassen_within_8_ulp_of_naive(k, n):
    """Scheme consistency at the reference's sizes (verify.py:384-424):
    Strassen (cutoff 32, peeled odd sizes) within 8 K-word ulps of naive at
    the |A||B| scale."""
    rng = np.random.default_rng(20240804 + n + k)
    c0 = rng.uniform(-1.0, 1.0, (n, n))
    a = np.stack([c0] + [c0 * 2.0 ** (-53 * j) * 0.3 for j in range(1, k)])
    c0 = rng.uniform(-1.0, 1.0, (n, n))
    b = np.stack([c0] + [c0 * 2.0 ** (-53 * j) * 0.2 for j in range(1, k)])
    A, B = MWMatrix(a), MWMatrix(b)
    cs = matmul(A, B, MatMulPlan(scheme="strassen", variant="bf")).numpy()
    cn = matmul(A, B, MatMulPlan(scheme="naive", variant="bf")).numpy()
    scale = np.abs(a).sum(0) @ np.abs(b).sum(0)
    worst = 0.0
    for i in range(0, n, 3):
        for j in range(0, n, 5):
            d = abs(exact_value(cs[:, i, j]) - exact_value(cn[:, i, j]))
            if d:
                _, e = math.frexp(scale[i, j])
                worst = max(worst, float(d) / math.ldexp(1.0, e - 53 * k))
    assert worst <= 8.0


def test_dot_single_launch_rearms_and_matches_two_stage():
    """Repeated single-launch dots (ticket re-armed in-kernel) agree with the
    two-stage path (mw_dot_partials + mw_tree_fold) bit for bit."""
    from paper_2603_14926_b200 import dist as mwdist

    rng = np.random.default_rng(12)
    for n in (4097, 65536, 1 << 20):
        x, y = gen.g_k(rng, 2, n), gen.g_k(rng, 2, n)
        X, Y = LaneBatch(x), LaneBatch(y)
        first = blas.dot_tensor(X, Y, Variant.BRANCH_FREE).cpu().numpy()
        for _ in range(3):
            assert_bitwise(blas.dot_tensor(X, Y, Variant.BRANCH_FREE).cpu().numpy(), first)
        be = mwdist.gpu_dot_backend(Variant.BRANCH_FREE)
        assert_bitwise(be.fold(be.partials(X.planes, Y.planes)).cpu().numpy(), first)


# ------------------------------------------------------------ edge cases
def test_empty_and_degenerate_shapes():
    """Empty batches, 1x1 products, kd = 0, degree 0 and zero points all go
    through the API without launching garbage (reference semantics)."""
    e = LaneBatch(np.zeros((3, 0)))
    assert batch_add(e, e, Variant.BRANCH_FREE).width == 0
    assert blas.dot(e, e, Variant.BRANCH_FREE) == (0.0, 0.0, 0.0)
    z = matmul(MWMatrix(np.zeros((2, 3, 0))), MWMatrix(np.zeros((2, 0, 4))), MatMulPlan(scheme="naive", variant="bf"))
    assert z.numpy().shape == (2, 3, 4) and not z.numpy().any()
    p0 = MWPolynomial(np.array([[2.5], [1e-20]]))
    ys = horner_eval_batched(p0, LaneBatch(np.ones((2, 5))), Variant.BRANCH_FREE).numpy()
    assert (ys[0] == 2.5).all() and (ys[1] == 1e-20).all()
    assert horner_eval_batched(p0, LaneBatch(np.ones((2, 0))), Variant.BRANCH_FREE).width == 0
    one = matmul(MWMatrix(np.array([[[3.0]], [[0.0]]])), MWMatrix(np.array([[[2.0]], [[0.0]]])),
                 MatMulPlan(scheme="strassen", variant="bf"))
    assert one.numpy()[0, 0, 0] == 6.0


def test_nonfinite_values_propagate():
    """Non-finite values propagate and never trap (multiword.py:18-20)."""
    a = np.zeros((2, 4))
    a[0] = [np.inf, -np.inf, np.nan, 1.0]
    b = np.zeros((2, 4))
    b[0] = [1.0, 1.0, 1.0, 0.0]
    la, lb = LaneBatch(a), LaneBatch(b)
    s = batch_add(la, lb, Variant.BRANCH_FREE).numpy()
    assert not np.isfinite(s[0, :3]).any()
    q = batch_div(la, lb, Variant.BRANCH_FREE).numpy()
    assert not np.isfinite(q[0, 3])


def test_dist_paths_single_rank_nccl():
    """The multi-GPU code paths (dist.py) on a one-rank NCCL group: device
    all-gathers and the MIN all-reduce run, and results equal the 1-GPU
    kernels bit for bit (the gloo tests cover world size 2 on CPU)."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2603_14926_b200 import dist as mwdist

    if dist.is_initialized():
        pytest.skip("process group already initialised")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(8)
        x, y = gen.g_k(rng, 3, 70000), gen.g_k(rng, 3, 70000)
        X, Y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        got = mwdist.dot_allgather(X, Y, mwdist.gpu_dot_backend(Variant.BRANCH_FREE))
        assert_bitwise(got.cpu().numpy(), oracle.dot(x, y, "bf", order=1))
        coeffs = gen.config5_poly(3)
        zre, zim = gen.config5_init(3)
        re, im, first = mwdist.dk_sweeps_sharded(torch.from_numpy(coeffs).cuda(), torch.from_numpy(zre).cuda(),
                                                 torch.from_numpy(zim).cuda(), 2, Variant.BRANCH_FREE)
        assert first is None
        ref = dk_sweeps(MonicPoly(coeffs), RootState(re=zre, im=zim), 2, Variant.BRANCH_FREE)
        assert_bitwise(re.cpu().numpy(), ref.re.cpu().numpy())
        assert_bitwise(im.cpu().numpy(), ref.im.cpu().numpy())
        # the captured form: sweeps + NCCL all-gathers in one CUDA graph
        g = mwdist.DKShardedGraph(torch.from_numpy(coeffs).cuda(), torch.from_numpy(zre).cuda(),
                                  torch.from_numpy(zim).cuda(), 2, Variant.BRANCH_FREE)
        g.replay()
        g.replay()
        gre, gim, first = g.result()
        assert first is None
        assert_bitwise(gre.cpu().numpy(), ref.re.cpu().numpy())
        assert_bitwise(gim.cpu().numpy(), ref.im.cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_multiword_scalar_ops_match_golden(golden):
    """DD/TD/QD value classes (Standard operators) and the scalar mw_*
    functions reproduce the reference's lanes (one-lane device kernels)."""
    from paper_2603_14926_b200 import multiword as mwm

    g = golden("ew")
    for k, v in CASES:
        p = f"k{k}_{v}"
        a, b = g[p + "_a"], g[p + "_b"]
        for lane in (7, 100):
            x, y = tuple(a[:, lane]), tuple(b[:, lane])
            assert mwm.mw_add(x, y, V(v)) == tuple(g[p + "_add"][:, lane])
            assert mwm.mw_mul(x, y, V(v)) == tuple(g[p + "_mul"][:, lane])
            assert mwm.mw_sub(x, y, V(v)) == tuple(g[p + "_sub"][:, lane])
            if v == "std":
                X, Y = mwm.MultiWord.from_components(x), mwm.MultiWord.from_components(y)
                assert (X + Y).comps == tuple(g[p + "_add"][:, lane])
                assert (X * Y).comps == tuple(g[p + "_mul"][:, lane])
                assert (X - Y).comps == tuple(g[p + "_sub"][:, lane])
    q = mwm.DD(1.0) / 3.0
    assert abs(q.to_fraction() - Fraction(1, 3)) < Fraction(1, 2**100)
    z = mwm.cmul(((1.0, 0.0), (2.0, 0.0)), ((3.0, 0.0), (-1.0, 0.0)), Variant.BRANCH_FREE)
    assert z == ((5.0, 0.0), (5.0, 0.0))


def test_eft_kats_on_device():
    """pkg/tests/test_eft.py known answers through the device EFTs."""
    from paper_2603_14926_b200 import eft

    eft.assert_rounding_mode()
    assert eft.quick_two_sum(3.5, 0.0) == (3.5, 0.0)
    assert eft.quick_two_sum(0.0, 1.25) == (1.25, 0.0)
    assert eft.quick_two_sum(1.0, 2.0**-60) == (1.0, 2.0**-60)
    assert eft.quick_two_sum(2.0**53, 1.0) == (2.0**53, 1.0)
    assert eft.two_sum(0.0, 2.5) == (2.5, 0.0)
    assert eft.two_prod(3.7, 1.0) == (3.7, 0.0)
    p, e = eft.two_prod(2.0**30 + 1, 2.0**30 + 1)
    assert p == 2.0**60 + 2.0**31 and e == 1.0
    rng = np.random.default_rng(1)
    a = rng.uniform(-1e10, 1e10, 256)
    b = rng.uniform(-1e-10, 1e10, 256)
    s, err = eft.two_sum(a, b)
    for i in range(256):
        assert Fraction(s[i]) + Fraction(err[i]) == Fraction(a[i]) + Fraction(b[i])
    p, err = eft.two_prod(a, b)
    for i in range(256):
        assert Fraction(p[i]) + Fraction(err[i]) == Fraction(a[i]) * Fraction(b[i])


# ------------------------------------------------- property-based (hypothesis)
from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

_finite = st.floats(min_value=-1e250, max_value=1e250, allow_nan=False, allow_infinity=False).filter(
    lambda x: x == 0.0 or abs(x) > 1e-250)


@st.composite
def _kword_batches(draw):
    k = draw(st.sampled_from([2, 3, 4]))
    w = draw(st.integers(min_value=1, max_value=9))
    lead = draw(st.lists(_finite, min_size=2 * w, max_size=2 * w))
    frac = draw(st.lists(st.floats(min_value=-0.49, max_value=0.49), min_size=2 * w * (k - 1),
                         max_size=2 * w * (k - 1)))
    a = np.zeros((k, w))
    b = np.zeros((k, w))
    a[0], b[0] = lead[:w], lead[w:]
    it = iter(frac)
    for c in range(1, k):
        for i in range(w):
            a[c, i] = a[c - 1, i] * 2.0**-53 * next(it)
            b[c, i] = b[c - 1, i] * 2.0**-53 * next(it)
    v = draw(st.sampled_from(["bf", "std"]))
    return k, v, a, b


@given(_kword_batches())
@settings(max_examples=150, deadline=None)
def test_property_lane_ops_match_oracle(case):
    """Random K-word lanes over the whole binary64 range (the reference's
    hypothesis strategies, test_eft.py:14-23): add / sub / mul equal the
    oracle bit for bit (overflow-free range)."""
    k, v, a, b = case
    la, lb = LaneBatch(a), LaneBatch(b)
    with np.errstate(all="ignore"):
        for op, fn in (("add", batch_add), ("sub", batch_sub), ("mul", batch_mul)):
            want = oracle.ew(op, a, b, v)
            got = fn(la, lb, V(v)).numpy()
            assert_bitwise(got, want, nan_ok=True)


# ----------------------------------------------------- out-of-bounds canaries
_CANARY = np.frombuffer(np.uint64(0x7FF4DEADBEEFCAFE).tobytes(), dtype=np.float64)[0]  # a NaN payload


def _guarded(shape, guard=4096):
    """Device buffer of `shape` (K, ...) flattened per plane inside a
    canary-filled allocation; returns (full_tensor, inner_view, plane_stride)."""
    k = shape[0]
    inner = int(np.prod(shape[1:]))
    full = torch.full((k, inner + 2 * guard), float("nan"), dtype=torch.float64, device="cuda")
    full.view(torch.int64).fill_(int(np.uint64(0x7FF4DEADBEEFCAFE).astype(np.int64)))
    return full, guard, inner + 2 * guard


def _guards_intact(full, guard, inner):
    bits = full.view(torch.int64).cpu().numpy()
    pat = np.int64(np.uint64(0x7FF4DEADBEEFCAFE).astype(np.int64))
    return bool((bits[:, :guard] == pat).all() and (bits[:, guard + inner:] == pat).all())


@pytest.mark.parametrize("k", [2, 3, 4])
def test_no_out_of_bounds_writes(k):
    """Outputs written through the C-ABI into canary-guarded buffers at
    ragged sizes: every kernel stays inside its output (compute-sanitizer
    is closed on this pool)."""
    from paper_2603_14926_b200 import _lib

    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(k)
    m, kd, n = 67, 45, 93
    A = torch.from_numpy(gen.g_k(rng, k, (m, kd))).cuda()
    B = torch.from_numpy(gen.g_k(rng, k, (kd, n))).cuda()
    full, g, ps = _guarded((k, m, n))
    assert lib.mw_gemm(k, 1, A.data_ptr(), kd, m * kd, B.data_ptr(), n, kd * n,
                       full.data_ptr() + g * 8, n, ps, m, n, kd, st) == 0
    torch.cuda.synchronize()
    assert _guards_intact(full, g, m * n)
    # lane ops, Horner, Estrin, GEMV, DK on 1001 lanes / roots
    w = 1001
    x = torch.from_numpy(gen.g_k(rng, k, w)).cuda()
    full, g, ps = _guarded((k, w))
    for fn in ("mw_ew_add", "mw_ew_mul", "mw_ew_div"):
        assert getattr(lib, fn)(k, 1, x.data_ptr(), w, x.data_ptr(), w, full.data_ptr() + g * 8, ps, w, st) == 0
    cf = torch.from_numpy(gen.g_k(rng, k, 77)).cuda()
    assert lib.mw_horner(k, 1, cf.data_ptr(), 77, 76, x.data_ptr(), w, full.data_ptr() + g * 8, ps, w, st) == 0
    assert lib.mw_poly_eval(k, 1, cf.data_ptr(), 77, 76, x.data_ptr(), None, w, full.data_ptr() + g * 8, None,
                            ps, w, 1, st) == 0
    Ag = torch.from_numpy(gen.g_k(rng, k, (w, 33))).cuda()
    xg = torch.from_numpy(gen.g_k(rng, k, 33)).cuda()
    for order in (0, 1):
        assert lib.mw_gemv(k, 1, Ag.data_ptr(), 33, w * 33, xg.data_ptr(), 33, full.data_ptr() + g * 8, ps,
                           w, 33, order, st) == 0
    torch.cuda.synchronize()
    assert _guards_intact(full, g, w)
    nr = 40
    coeffs = torch.from_numpy(gen.g_k(rng, k, nr) * 0.5).cuda()
    ang = 2 * np.pi * np.arange(nr) / nr + 0.1
    zr = np.zeros((k, nr))
    zi = np.zeros((k, nr))
    zr[0], zi[0] = 1.3 * np.cos(ang), 1.3 * np.sin(ang)
    zr_t, zi_t = torch.from_numpy(zr).cuda(), torch.from_numpy(zi).cuda()
    fre, g2, ps2 = _guarded((k, nr))
    fim, _, _ = _guarded((k, nr))
    mag, gm, _ = _guarded((1, nr))
    flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
    for exact in (1, 0):
        assert lib.mw_dk_sweep(k, 1, coeffs.data_ptr(), nr, nr, zr_t.data_ptr(), zi_t.data_ptr(), nr, 3, 37,
                               fre.data_ptr() + g2 * 8, fim.data_ptr() + g2 * 8, ps2, mag.data_ptr() + gm * 8,
                               flag.data_ptr(), exact, st) == 0
    torch.cuda.synchronize()
    assert _guards_intact(fre, g2, nr) and _guards_intact(fim, g2, nr) and _guards_intact(mag, gm, nr)
    # tree sweeps with a workspace: every roots-per-CTA form, ragged last CTA
    i0, i1 = 3, 37  # 34 roots: 4 per CTA leaves 2 in the last
    for roots in (0, 1, 2, 4):
        tune = _lib.tuning(dk_tree_roots=roots)
        wsn = lib.mw_dk_sweep_workspace(k, i0, i1)
        wsf, gw, _ = _guarded((1, wsn))
        assert lib.mw_dk_sweep_ex(k, 1, coeffs.data_ptr(), nr, nr, zr_t.data_ptr(), zi_t.data_ptr(), nr, i0,
                                  i1, fre.data_ptr() + g2 * 8, fim.data_ptr() + g2 * 8, ps2,
                                  mag.data_ptr() + gm * 8, flag.data_ptr(), 0, wsf.data_ptr() + gw * 8,
                                  None, _lib.tuning_ptr(tune), st) == 0
        torch.cuda.synchronize()
        assert _guards_intact(fre, g2, nr) and _guards_intact(fim, g2, nr) and _guards_intact(mag, gm, nr)
        assert _guards_intact(wsf, gw, wsn)
    # kernels outside the dispatch tables, renormalisation, fma
    full, g, ps = _guarded((k, w))
    if k in (2, 3):
        xs = torch.from_numpy(gen.g_k(rng, k, w)).cuda()
        assert lib.mw_named_op(k - 2, xs.data_ptr(), w, xs.data_ptr(), w, full.data_ptr() + g * 8, ps, w, st) == 0
    raw = torch.from_numpy(gen.g_k(rng, {2: 2, 3: 4, 4: 5}[k], w)).cuda()
    assert lib.mw_renormalize(k, raw.data_ptr(), w, full.data_ptr() + g * 8, ps, w, st) == 0
    assert lib.mw_fma(x.data_ptr(), x.data_ptr(), x.data_ptr(), full.data_ptr() + g * 8, w, st) == 0
    torch.cuda.synchronize()
    assert _guards_intact(full, g, w)


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("v", ["bf", "std"])
def test_dk_peer_graph_matches_sweeps(k, exact, v):
    """The fused-exchange sweep (mw_dk_sweep_peer through DKPeerGraph, one
    rank: stores, ticket, slot publication and wait all run) equals the
    plain sweeps bit for bit, for odd and even sweep counts and across
    replays (monotonic slots, alternating start parity)."""
    from paper_2603_14926_b200 import dist as mwdist

    rng = np.random.default_rng(40 + k)
    n = 96
    coeffs = gen.g_k(rng, k, n) * 0.5
    ang = 2 * np.pi * np.arange(n) / n + 0.1
    zre = np.zeros((k, n)); zim = np.zeros((k, n))
    zre[0] = 1.3 * np.cos(ang); zim[0] = 1.3 * np.sin(ang)
    C, R, I = (torch.from_numpy(a).cuda() for a in (coeffs, zre, zim))
    for sweeps in (3, 4):
        ref = dk_sweeps(MonicPoly(coeffs), RootState(re=zre, im=zim), sweeps, V(v),
                        exact_order=exact)
        g = mwdist.DKPeerGraph(C, R, I, sweeps, V(v), exact_order=exact)
        try:
            for _ in range(3):
                g.replay()
                gre, gim, first = g.result()
                assert first is None
                assert_bitwise(gre.cpu().numpy(), ref.re.cpu().numpy())
                assert_bitwise(gim.cpu().numpy(), ref.im.cpu().numpy())
        finally:
            g.close()


def test_dk_peer_wait_times_out_instead_of_hanging():
    """A peer that never publishes (world 2, rank 1 absent: both table
    entries point at this rank's own buffer) makes the last CTA's wait
    expire after spin_limit polls; the kernel returns and sets *timeout."""
    import ctypes

    from paper_2603_14926_b200 import _lib
    from paper_2603_14926_b200 import dist as mwdist

    lib = _lib.load()
    k, n = 2, 64
    lay = mwdist.PeerLayout(k, n, 2)
    buf = ctypes.c_void_p()
    _lib.check(lib.mw_peer_alloc(lay.total_bytes, ctypes.byref(buf)), "alloc")
    try:
        base = buf.value
        outs, slots = mwdist.peer_tables([base, base], lay)
        dev = torch.device("cuda", 0)
        o = torch.tensor(outs[0], dtype=torch.int64, device=dev)
        sl = torch.tensor(slots, dtype=torch.int64, device=dev)
        rng = np.random.default_rng(3)
        coeffs = torch.from_numpy(gen.g_k(rng, k, n) * 0.5).cuda()
        done = torch.zeros(1, dtype=torch.int32, device=dev)
        epoch = torch.zeros(1, dtype=torch.int64, device=dev)
        tout = torch.zeros(1, dtype=torch.int32, device=dev)
        mag = torch.empty(n, dtype=torch.float64, device=dev)
        flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device=dev)
        rc = lib.mw_dk_sweep_peer(k, 1, coeffs.data_ptr(), n, n, base, 0, n // 2, o.data_ptr(), sl.data_ptr(),
                                  base + lay.state_off(1), base + lay.slot_off, done.data_ptr(), epoch.data_ptr(),
                                  tout.data_ptr(), 2, 0, 0, 2, 2000, mag.data_ptr(), flag.data_ptr(), 0,
                                  None, _lib.stream_handle(dev))
        _lib.check(rc, "mw_dk_sweep_peer")
        torch.cuda.synchronize()
        assert int(tout.item()) == 1
        assert int(done.item()) == 0  # ticket reset by the last CTA
        # own slot from rank 0 was published (value epoch*sweeps + 0 + 1)
        sv = torch.as_tensor(mwdist._DevView(base + lay.slot_off, (2,)), device=dev).view(torch.int64)
        assert sv.cpu().tolist() == [1, 0]
    finally:
        lib.mw_peer_free(buf)


def _ipc_worker(rank, port, outdir):
    import ctypes
    import os

    import torch.distributed as dist

    from paper_2603_14926_b200 import _lib
    from paper_2603_14926_b200 import dist as mwdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    lib = _lib.load()
    buf = ctypes.c_void_p()
    _lib.check(lib.mw_peer_alloc(4096, ctypes.byref(buf)), "alloc")
    own = torch.as_tensor(mwdist._DevView(buf.value, (512,)), device="cuda:0")
    own[:256].fill_(rank + 1.0)
    torch.cuda.synchronize()
    h = (ctypes.c_char * 64)()
    _lib.check(lib.mw_ipc_get_handle(buf, h), "handle")
    hs = mwdist.exchange_handles(bytes(h))
    peer = ctypes.c_void_p()
    _lib.check(lib.mw_ipc_open_handle(hs[1 - rank], ctypes.byref(peer)), "open")
    pv = torch.as_tensor(mwdist._DevView(peer.value, (512,)), device="cuda:0")
    seen = float(pv[:256].sum().item())
    pv[256 + rank].fill_(10.0 + rank)  # a store into the peer's buffer
    torch.cuda.synchronize()
    dist.barrier()
    got = own[256:258].cpu().tolist()
    with open(os.path.join(outdir, f"r{rank}.txt"), "w") as fh:
        fh.write(f"{seen} {got[0]} {got[1]}")
    dist.barrier()
    lib.mw_ipc_close_handle(peer)
    dist.barrier()
    lib.mw_peer_free(buf)
    dist.destroy_process_group()


def test_ipc_peer_mapping_two_processes():
    """mw_peer_alloc / mw_ipc_* between two processes on one GPU: each
    reads the other's buffer and stores into it through the mapping (no
    kernel waits on another process)."""
    import tempfile

    import torch.multiprocessing as mp

    from test_dist_gloo import _free_port

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_ipc_worker, args=(_free_port(), d), nprocs=2, join=True)
        r0 = open(f"{d}/r0.txt").read().split()
        r1 = open(f"{d}/r1.txt").read().split()
    assert float(r0[0]) == 256 * 2.0 and float(r1[0]) == 256 * 1.0
    # rank p stored 10 + p at index 256 + p of the other rank's buffer
    assert float(r0[2]) == 11.0 and float(r1[1]) == 10.0


@pytest.mark.parametrize("k", [2, 3, 4])
def test_dot_peer_matches_tree_dot(k):
    """DotPeer (mw_dot_peer: roots stored to every rank's buffer, ticket,
    slot publication, wait, in-kernel fold) on one rank equals the 1-GPU
    tree dot and its oracle restatement bit for bit: ragged n, n below one
    block, n needing the two-level fold (> 256 block roots), and repeated
    calls (alternating root-buffer parity)."""
    from paper_2603_14926_b200 import blas
    from paper_2603_14926_b200 import dist as mwdist

    for n in (1, 100, 4096, 70001, (1 << 20) + 4097):
        rng = np.random.default_rng(n + k)
        x, y = gen.g_k(rng, k, n), gen.g_k(rng, k, n)
        X, Y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        want = blas.dot_tensor(LaneBatch(X), LaneBatch(Y), Variant.BRANCH_FREE).cpu().numpy()
        if n <= 70001:
            assert_bitwise(want, oracle.dot(x, y, "bf", order=1))
        dp = mwdist.DotPeer(k, n, Variant.BRANCH_FREE)
        try:
            for _ in range(3):
                got = dp(X, Y)
                assert_bitwise(got.cpu().numpy(), want)
            dp.check()
        finally:
            dp.close()


def test_dot_peer_wait_times_out_instead_of_hanging():
    """World 2 with the absent peer's table entries pointing at this rank:
    the last block's wait expires and the kernel returns with *timeout set."""
    import ctypes

    from paper_2603_14926_b200 import _lib

    lib = _lib.load()
    k, n = 2, 8192
    nbt = 2
    nbytes = 2 * k * nbt * 8 + 2 * 8
    buf = ctypes.c_void_p()
    _lib.check(lib.mw_peer_alloc(nbytes, ctypes.byref(buf)), "alloc")
    try:
        base = buf.value
        dev = torch.device("cuda", 0)
        roots = torch.tensor([base, base], dtype=torch.int64, device=dev)
        slot_off = 2 * k * nbt * 8
        slots = torch.tensor([base + slot_off] * 2, dtype=torch.int64, device=dev)
        rng = np.random.default_rng(2)
        X = torch.from_numpy(gen.g_k(rng, k, n)).cuda()
        done = torch.zeros(1, dtype=torch.int32, device=dev)
        epoch = torch.zeros(1, dtype=torch.int64, device=dev)
        tout = torch.zeros(1, dtype=torch.int32, device=dev)
        out = torch.empty(k, dtype=torch.float64, device=dev)
        rc = lib.mw_dot_peer(k, 1, X.data_ptr(), n, X.data_ptr(), n, 4096, 0, nbt, roots.data_ptr(),
                             slots.data_ptr(), base + slot_off, done.data_ptr(), epoch.data_ptr(),
                             tout.data_ptr(), 2, 0, 2000, out.data_ptr(), _lib.stream_handle(dev))
        _lib.check(rc, "mw_dot_peer")
        torch.cuda.synchronize()
        assert int(tout.item()) == 1 and int(done.item()) == 0 and int(epoch.item()) == 1
    finally:
        lib.mw_peer_free(buf)


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("v", ["bf", "std"])
def test_dk_exact_split_and_single_warp_forms_agree(k, v):
    """The split-pair exact kernel (QD default) and the single-warp one give
    the same bits, and both equal the oracle's reference-order sweep."""
    from paper_2603_14926_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(70 + k)
    n = 80
    coeffs = gen.g_k(rng, k, n) * 0.5
    ang = 2 * np.pi * np.arange(n) / n + 0.1
    zre = np.zeros((k, n)); zim = np.zeros((k, n))
    zre[0] = 1.3 * np.cos(ang); zim[0] = 1.3 * np.sin(ang)
    want_re, want_im, _, _ = oracle.dk_sweep(coeffs, zre, zim, v, exact=True)
    for split in (0, 1):
        out = dk_sweeps(MonicPoly(coeffs), RootState(re=zre, im=zim), 1, V(v), exact_order=True,
                        tuning=_lib.tuning(dk_exact_split=split))
        assert_bitwise(out.re.cpu().numpy(), want_re)
        assert_bitwise(out.im.cpu().numpy(), want_im)


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("v", ["bf", "std"])
def test_dk_tree_powers_kernel_path_matches_in_warp_path(k, v):
    """Tree sweep with the lane-per-root powers kernel + programmatic
    dependent launch (mw_dk_sweep_ws) equals the in-warp powers path
    (mw_dk_sweep) and the oracle bit for bit, on a sub-range of roots
    (134 roots: ragged last CTA for 4 roots per CTA), for the 3-warp
    single-root kernel and the 2- and 4-roots-per-CTA kernels."""
    from paper_2603_14926_b200 import _lib
    from paper_2603_14926_b200.multiword import variant_code

    lib = _lib.load()
    rng = np.random.default_rng(90 + k)
    n = 150
    coeffs = gen.g_k(rng, k, n) * 0.5
    ang = 2 * np.pi * np.arange(n) / n + 0.1
    zre = np.zeros((k, n)); zim = np.zeros((k, n))
    zre[0] = 1.3 * np.cos(ang); zim[0] = 1.3 * np.sin(ang)
    C, R, I = (torch.from_numpy(a).cuda() for a in (coeffs, zre, zim))
    i0, i1 = 7, 141
    outs = []
    for use_ws, roots in ((False, 2), (True, 0), (True, 1), (True, 2), (True, 4)):
        tune = _lib.tuning(dk_tree_roots=roots)
        ore, oim = torch.zeros_like(R), torch.zeros_like(I)
        mag = torch.zeros(n, dtype=torch.float64, device="cuda")
        flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
        args = [k, variant_code(V(v)), C.data_ptr(), n, n, R.data_ptr(), I.data_ptr(), n, i0, i1, ore.data_ptr(),
                oim.data_ptr(), n, mag.data_ptr(), flag.data_ptr(), 0]
        if use_ws:
            ws = torch.empty(lib.mw_dk_sweep_workspace(k, i0, i1), dtype=torch.float64, device="cuda")
            rc = lib.mw_dk_sweep_ex(*args, ws.data_ptr(), None, _lib.tuning_ptr(tune), _lib.stream_handle(R.device))
        else:
            rc = lib.mw_dk_sweep(*args, _lib.stream_handle(R.device))
        _lib.check(rc, "sweep")
        outs.append((ore.cpu().numpy(), oim.cpu().numpy(), mag.cpu().numpy()))
    for o in outs[1:]:  # in-warp powers == powers kernel, for every roots-per-CTA form
        assert_bitwise(outs[0][0], o[0])
        assert_bitwise(outs[0][1], o[1])
        assert_bitwise(outs[0][2], o[2])
    want_re, want_im, _, _ = oracle.dk_sweep(coeffs, zre, zim, v, exact=False, rows=(i0, i1))
    assert_bitwise(outs[1][0][:, i0:i1], want_re[:, i0:i1])
    assert_bitwise(outs[1][1][:, i0:i1], want_im[:, i0:i1])


# ------------------------------------ Standard variant at benchmark sizes
@pytest.mark.parametrize("k,n", [(2, 1024), (3, 1024), (4, 512)])
def test_standard_gemm_sampled_rows_at_scale(k, n):
    """The Standard (renormalising) GEMM at sizes where every warp sees
    divergent renormalisation paths, sampled rows vs the oracle."""
    a, b = gen.config3_gemm(k, n)
    c = matmul(MWMatrix(a), MWMatrix(b), MatMulPlan(scheme="naive", variant="std")).numpy()
    for r0 in (0, n // 2 + 1, n - 1):
        assert_bitwise(c[:, r0], oracle.gemm(a, b, "std", rows=(r0, r0 + 1))[:, r0])


def test_standard_horner_sampled_points_at_scale():
    coeffs, x = gen.config4_horner(npts=1 << 20)
    y = horner_eval_batched(MWPolynomial(coeffs), LaneBatch(x), Variant.STANDARD).numpy()
    idx = np.r_[0:1024, (1 << 19):(1 << 19) + 1024, (1 << 20) - 1024:(1 << 20)]
    assert_bitwise(y[:, idx], oracle.horner(coeffs, x[:, idx], "std"))


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("exact", [True, False])
def test_standard_dk_sweep_config5(k, exact):
    """One Standard-variant sweep of the degree-512 config-5 problem, both
    orders, vs the oracle (exact: reference order; tree: its restatement)."""
    coeffs = gen.config5_poly(k)
    zre, zim = gen.config5_init(k)
    nxt = dk_iterate(MonicPoly(coeffs), RootState(re=zre, im=zim), Variant.STANDARD, exact_order=exact)
    ore, oim, _, coll = oracle.dk_sweep(coeffs, zre, zim, "std", exact=exact)
    assert coll is None
    assert_bitwise(nxt.re.cpu().numpy(), ore)
    assert_bitwise(nxt.im.cpu().numpy(), oim)


@pytest.mark.parametrize("k,m,n", [(2, 512, 4096), (3, 256, 2048), (4, 512, 2048), (3, 67, 93)])
def test_gemm_tile_slots_bit_identical(k, m, n):
    """Every GEMM tile slot (and the per-shape choice) gives the same bits
    on row-block shard shapes; a sampled row equals the oracle."""
    from paper_2603_14926_b200 import _lib
    from paper_2603_14926_b200.linalg import gemm_into

    lib = _lib.load()
    rng = np.random.default_rng(m + n + k)
    a, b = gen.g_k(rng, k, (m, n)), gen.g_k(rng, k, (n, n))
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    outs = []
    for policy in (0, 1, 2, 3):
        C = torch.empty((k, m, n), dtype=torch.float64, device="cuda")
        gemm_into(A, B, C, Variant.BRANCH_FREE, tuning=_lib.tuning(gemm_tile=policy))
        outs.append(C.cpu().numpy())
    for o in outs[1:]:
        assert_bitwise(o, outs[0])
    r = m // 3
    assert_bitwise(outs[0][:, r], oracle.gemm(a, b, "bf", rows=(r, r + 1))[:, r])


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("n", [4097, 8192, 40000, 65535, 65536, 65537])
def test_dot_cluster_form_matches_ticket_form(k, n):
    """Dots of 2..16 blocks as one thread-block cluster (block roots through
    distributed shared memory) equal the single-launch ticket form and the
    oracle's tree restatement bit for bit (65537 takes the ticket form)."""
    from paper_2603_14926_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(3 * n + k)
    x, y = gen.g_k(rng, k, n), gen.g_k(rng, k, n)
    X, Y = LaneBatch(x), LaneBatch(y)
    outs = []
    for on in (1, 0, 1):  # cluster, ticket, cluster again (repeat calls)
        outs.append(np.array(blas.dot(X, Y, Variant.BRANCH_FREE, order="tree", tuning=_lib.tuning(dot_cluster=on))))
    for o in outs[1:]:
        assert_bitwise(o, outs[0])
    assert_bitwise(outs[0], oracle.dot(x, y, "bf", order=1))


# ------------------------------------------- the extension's host boundary
def test_extension_validates_operands():
    """Wrong dtype, overlapping / strided lanes, mixed K, wrong out shapes
    -> ValueError before any launch (no silent out-of-bounds access)."""
    from paper_2603_14926_b200 import _lib

    e = _lib.ext()
    a = torch.zeros(3, 64, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        e.ew(0, 1, a.float(), a.float())
    with pytest.raises(ValueError):
        e.ew(0, 1, a, torch.zeros(2, 64, dtype=torch.float64, device="cuda"))  # mixed K
    with pytest.raises(ValueError):
        e.ew(0, 1, a[:, ::2], a[:, ::2])  # strided lanes
    with pytest.raises(ValueError):
        e.ew(0, 1, a, a, torch.zeros(3, 63, dtype=torch.float64, device="cuda"))
    A = torch.zeros(3, 8, 8, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        e.gemm(1, A, A.transpose(1, 2), A)  # non-contiguous B
    with pytest.raises(ValueError):
        e.gemm(1, A, A, A, 0, 9)  # rows outside C
    with pytest.raises(ValueError):
        e.horner(1, torch.zeros(3, 5, dtype=torch.float64, device="cuda"), a, a, 10, 5)
    # column slices of a wider batch are fine (plane stride = full width)
    w = torch.from_numpy(gen.g_k(np.random.default_rng(1), 3, 256)).cuda()
    out = e.ew(2, 1, w[:, 10:74], w[:, 100:164])
    assert_bitwise(out.cpu().numpy(), oracle.ew("mul", w[:, 10:74].cpu().numpy(), w[:, 100:164].cpu().numpy(), "bf"))


def test_dot_graphs_on_two_streams_keep_private_workspaces():
    """Two CUDA graphs of the ticket-form tree dot (n = 2^20: 256 blocks,
    workspace ticket + partials) replayed concurrently on two streams give
    the eager result: graph captures get their own workspace."""
    k, n = 3, 1 << 20
    rng = np.random.default_rng(11)
    X, Y = LaneBatch(gen.g_k(rng, k, n)), LaneBatch(gen.g_k(rng, k, n))
    X2, Y2 = LaneBatch(gen.g_k(rng, k, n)), LaneBatch(gen.g_k(rng, k, n))
    want1 = blas.dot_tensor(X, Y, Variant.BRANCH_FREE).cpu().numpy()
    want2 = blas.dot_tensor(X2, Y2, Variant.BRANCH_FREE).cpu().numpy()
    o1 = torch.empty(k, dtype=torch.float64, device="cuda")
    o2 = torch.empty(k, dtype=torch.float64, device="cuda")
    g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1):
        blas.dot_tensor(X, Y, Variant.BRANCH_FREE, out=o1)
    with torch.cuda.graph(g2):
        blas.dot_tensor(X2, Y2, Variant.BRANCH_FREE, out=o2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(20):
        with torch.cuda.stream(s1):
            g1.replay()
        with torch.cuda.stream(s2):
            g2.replay()
    torch.cuda.synchronize()
    assert_bitwise(o1.cpu().numpy(), want1)
    assert_bitwise(o2.cpu().numpy(), want2)


DKSOLVE = [(2, "bf", 16), (3, "bf", 16), (4, "bf", 16), (2, "std", 16), (3, "std", 16), (4, "std", 16),
           (3, "bf", 64), (4, "bf", 64)]


@pytest.mark.parametrize("k,v,n", DKSOLVE, ids=[f"k{k}_{v}_n{n}" for k, v, n in DKSOLVE])
def test_dk_solve_matches_reference_solve(golden, k, v, n):
    """roots.dk_solve on the device (Aberth start on the device, chunked
    sweeps, on-device convergence test) against the reference's dk_solve
    (roots.py:318-340) on chebyshev_coeffs(n): same sweep count, same
    roots bit for bit -- including the paper's n = 64 TD/QD problem."""
    g = golden("dksolve")
    p = f"k{k}_{v}_n{n}"
    state, iters = roots.dk_solve(MonicPoly(g[p + "_coeffs"]), V(v))
    assert iters == int(g[p + "_iters"][0])
    assert_bitwise(state.re.cpu().numpy(), g[p + "_re"])
    assert_bitwise(state.im.cpu().numpy(), g[p + "_im"])
    assert math.isclose(state.last_max_update, float(g[p + "_maxupd"][0]), rel_tol=1e-15)


def test_extension_edge_cases_and_column_slices():
    """Empty operands launch nothing and return exact zeros / untouched
    outputs; column slices of wider batches (plane stride > width) go
    through dot, axpy and Horner without a copy and match the oracle."""
    from paper_2603_14926_b200 import _lib
    from paper_2603_14926_b200.poly import horner_into

    e = _lib.ext()
    rng = np.random.default_rng(21)
    for k in (2, 3, 4):
        z = torch.zeros((k, 0), dtype=torch.float64, device="cuda")
        assert e.ew(2, 1, z, z).shape == (k, 0)
        d = e.dot(1, z, z, 1)
        torch.cuda.synchronize()
        assert_bitwise(d.cpu().numpy(), np.zeros(k))  # fold from an exact zero
        e.axpy_(1, [1.0] + [0.0] * (k - 1), z, z)
        wide_x, wide_y = gen.g_k(rng, k, 10000), gen.g_k(rng, k, 10000)
        X, Y = torch.from_numpy(wide_x).cuda(), torch.from_numpy(wide_y).cuda()
        lo, hi = 1234, 1234 + 5000
        got = e.dot(1, X[:, lo:hi], Y[:, lo:hi], 1).cpu().numpy()
        assert_bitwise(got, oracle.dot(wide_x[:, lo:hi], wide_y[:, lo:hi], "bf", order=1))
        got = e.dot(1, X[:, lo:hi], Y[:, lo:hi], 0).cpu().numpy()
        assert_bitwise(got, oracle.dot(wide_x[:, lo:hi], wide_y[:, lo:hi], "bf", order=0))
        alpha = tuple(gen.g_k(rng, k, 1)[:, 0])
        Yc = Y.clone()
        e.axpy_(1, list(alpha), X[:, lo:hi], Yc[:, lo:hi])
        want = oracle.ew("add", oracle.ew("mul", np.tile(np.array(alpha)[:, None], (1, hi - lo)),
                                          wide_x[:, lo:hi], "bf"), wide_y[:, lo:hi], "bf")
        out = Yc.cpu().numpy()
        assert_bitwise(out[:, lo:hi], want)
        assert_bitwise(out[:, :lo], wide_y[:, :lo])  # outside the slice: untouched
        assert_bitwise(out[:, hi:], wide_y[:, hi:])
        coeffs = gen.g_k(rng, k, 17)
        C = torch.from_numpy(coeffs).cuda()
        yv = torch.full_like(X, 7.0)
        horner_into(C, X, yv, Variant.BRANCH_FREE, 300, 300)  # empty range: nothing written
        assert torch.all(yv == 7.0)
        horner_into(C, X, yv, Variant.BRANCH_FREE, 300, 1300)
        hv = yv.cpu().numpy()
        assert_bitwise(hv[:, 300:1300], oracle.horner(coeffs, np.ascontiguousarray(wide_x[:, 300:1300]), "bf"))
        assert np.all(hv[:, :300] == 7.0) and np.all(hv[:, 1300:] == 7.0)


def test_concurrent_callers_with_different_tuning():
    """The C-ABI is stateless: two host threads on their own streams, one
    forcing GEMM tile slot 0 and the tree dot's ticket form, the other
    slot 2 and the cluster form, issue interleaved calls; every result is
    bitwise the default one (no shared tuning state to race on)."""
    import threading

    from paper_2603_14926_b200 import _lib
    from paper_2603_14926_b200.linalg import gemm_into

    rng = np.random.default_rng(33)
    k, m, n = 3, 160, 96
    A = torch.from_numpy(gen.g_k(rng, k, (m, n))).cuda()
    B = torch.from_numpy(gen.g_k(rng, k, (n, n))).cuda()
    X, Y = LaneBatch(gen.g_k(rng, k, 40000)), LaneBatch(gen.g_k(rng, k, 40000))
    C0 = torch.empty((k, m, n), dtype=torch.float64, device="cuda")
    gemm_into(A, B, C0, Variant.BRANCH_FREE)
    d0 = blas.dot_tensor(X, Y, Variant.BRANCH_FREE).clone()
    torch.cuda.synchronize()
    errors = []

    def worker(tile, cluster):
        try:
            s = torch.cuda.Stream()
            tune = _lib.tuning(gemm_tile=tile, dot_cluster=cluster)
            with torch.cuda.stream(s):
                for _ in range(30):
                    C = torch.empty_like(C0)
                    gemm_into(A, B, C, Variant.BRANCH_FREE, tuning=tune)
                    d = blas.dot_tensor(X, Y, Variant.BRANCH_FREE, tuning=tune)
                    s.synchronize()
                    if not (torch.equal(C.view(torch.int64), C0.view(torch.int64))
                            and torch.equal(d.view(torch.int64), d0.view(torch.int64))):
                        errors.append((tile, cluster))
                        return
        except Exception as e:  # surfaced below
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(1, 0)), threading.Thread(target=worker, args=(3, 1))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("k,v", CASES, ids=IDS)
def test_lane_ops_special_values_vs_oracle(k, v):
    """Signed zeros, subnormal and near-overflow components, infinities and
    NaNs in every lane op, both variants: bitwise equal to the oracle
    (NaN positions compared, payloads not -- CUDA and x86 canonical NaNs
    differ).  Non-finite values propagate, never trap
    (multiword.py:18-20)."""
    rng = np.random.default_rng(500 + k)
    specials = [0.0, -0.0, 5e-324, -5e-324, 2.2250738585072014e-308, 1e-300, 1.0, -1.0, 1e300,
                1.7976931348623157e308, -1.7976931348623157e308, np.inf, -np.inf, np.nan]
    s = np.array(specials)
    w = len(s) ** 2
    a = np.zeros((k, w))
    b = np.zeros((k, w))
    a[0] = np.repeat(s, len(s))
    b[0] = np.tile(s, len(s))
    with np.errstate(all="ignore"):
        for c in range(1, k):  # small trailing components where the leading one is finite
            a[c] = np.where(np.isfinite(a[0]), a[c - 1] * 2.0**-53 * rng.uniform(-0.49, 0.49, w), 0.0)
            b[c] = np.where(np.isfinite(b[0]), b[c - 1] * 2.0**-53 * rng.uniform(-0.49, 0.49, w), 0.0)
    la, lb = LaneBatch(a), LaneBatch(b)
    with np.errstate(all="ignore"):
        for op, fn in (("add", batch_add), ("sub", batch_sub), ("mul", batch_mul), ("div", batch_div)):
            assert_bitwise(fn(la, lb, V(v)).numpy(), oracle.ew(op, a, b, v), nan_ok=True)
