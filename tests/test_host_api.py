"""Host-side API behaviour that needs no GPU: containers, validation and
error mapping mirror the reference (batch.py:61-119, 197-201;
linalg.py:75-158, 553-556; poly.py:40-86; roots.py:73-164), and the
product path fails loudly instead of falling back to the CPU."""

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_bitwise
from paper_2603_14926_b200 import (
    LaneBatch,
    MatMulPlan,
    MonicPoly,
    MWMatrix,
    MWPolynomial,
    RootState,
    Variant,
    batch_add,
    batch_mul,
    default_tolerance,
    matmul,
    pack,
    unpack,
)
from paper_2603_14926_b200 import blas, gen, roots
from paper_2603_14926_b200.multiword import from_fraction, ulp_k

NO_CUDA = not torch.cuda.is_available()


def test_variant_parse():
    assert Variant.parse("bf") is Variant.BRANCH_FREE
    assert Variant.parse("STANDARD") is Variant.STANDARD
    assert Variant.parse(Variant.STANDARD) is Variant.STANDARD
    with pytest.raises(ValueError):
        Variant.parse("fast")


def test_lanebatch_validation():
    with pytest.raises(ValueError):
        LaneBatch((np.zeros(4),) * 5)
    with pytest.raises(ValueError):
        LaneBatch((np.zeros(4), np.zeros(3)))
    lb = LaneBatch((np.arange(4.0), np.zeros(4)))
    assert lb.k == 2 and lb.width == 4 and lb.count == 4
    assert lb.lane(3) == (3.0, 0.0)


def test_pack_unpack_round_trip():
    vals = [(1.5, 2.0**-60), (-2.25, 0.0), (0.1, 0.0)]
    assert [v.comps for v in unpack(pack(vals))] == vals
    lb = pack([(1.0, 0.0)], width=8)
    assert lb.width == 8 and lb.count == 1
    assert all(lb.lane(i) == (0.0, 0.0) for i in range(1, 8))
    with pytest.raises(ValueError):
        pack([])
    with pytest.raises(ValueError):
        pack([(1.0, 0.0), (2.0, 0.0)], width=1)
    with pytest.raises(ValueError):
        pack([(1.0, 0.0), (1.0, 0.0, 0.0)])


def test_mixed_k_and_width_raise_before_any_launch():
    a = LaneBatch(np.zeros((2, 4)))
    with pytest.raises(ValueError):
        batch_add(a, LaneBatch(np.zeros((3, 4))))
    with pytest.raises(ValueError):
        batch_mul(a, LaneBatch(np.zeros((2, 8))))
    with pytest.raises(ValueError):
        blas.dot(a, LaneBatch(np.zeros((3, 4))))


@pytest.mark.skipif(not NO_CUDA, reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    a = LaneBatch(np.ones((2, 4)))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        batch_add(a, a, Variant.BRANCH_FREE)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        matmul(MWMatrix(np.ones((2, 3, 3))), MWMatrix(np.ones((2, 3, 3))), MatMulPlan(scheme="naive", variant="bf"))


def test_matmul_plan_and_shape_checks():
    with pytest.raises(ValueError):
        MatMulPlan(strassen_cutoff=1)
    with pytest.raises(ValueError):
        MatMulPlan(threads=0)
    with pytest.raises(ValueError):
        MatMulPlan(scheme="winograd")
    a = MWMatrix(np.zeros((2, 3, 4)))
    with pytest.raises(ValueError):
        matmul(a, MWMatrix(np.zeros((2, 3, 4))), MatMulPlan(scheme="naive"))
    with pytest.raises(ValueError):
        matmul(a, MWMatrix(np.zeros((3, 4, 4))), MatMulPlan(scheme="naive"))
    with pytest.raises(ValueError):
        matmul(a, MWMatrix(np.zeros((2, 4, 4))), MatMulPlan(scheme="strassen"))
    assert MWMatrix.identity(3, 4).k == 4
    with pytest.raises(ValueError):
        MWMatrix(np.zeros((2, 3)))


def test_polynomial_and_monic_containers():
    p = MWPolynomial.from_coeffs([7.5, 1.0], k=2)
    assert p.degree == 1 and p.coeff(0) == (7.5, 0.0)
    with pytest.raises(ValueError):
        MWPolynomial.from_coeffs([1.0])
    with pytest.raises(ValueError):
        MWPolynomial(np.zeros((2, 0)))
    q = MonicPoly.from_coeffs([(-1.0, 0.0), (0.0, 0.0)])
    assert q.n == 2 and q.k == 2
    with pytest.raises(ValueError):
        MonicPoly(np.zeros((2, 0)))


def test_default_tolerance_values():
    assert default_tolerance(2) == 2.0**-96
    assert default_tolerance(3) == 2.0**-149
    assert default_tolerance(4) == 2.0**-202


def test_ulp_and_rounding_helpers():
    assert ulp_k(1.0, 2) == 2.0**-105
    from fractions import Fraction

    v = from_fraction(Fraction(1, 3), 4)
    total = sum(Fraction(c) for c in v)
    assert abs(total - Fraction(1, 3)) < Fraction(1, 2**210)


def test_dk_solve_rejects_bad_tol():
    q = MonicPoly.from_coeffs([(-1.0, 0.0), (0.0, 0.0)])
    with pytest.raises(ValueError):
        roots.dk_solve(q, tol=0.0)


def _oracle_batch(monkeypatch):
    """Stand the oracle in for the device batch kernels (host-logic test)."""

    def mk(op):
        def f(a, b, v=Variant.STANDARD):
            return LaneBatch(oracle.ew(op, a.numpy(), b.numpy(), Variant.parse(v).value), device="cpu")

        return f

    monkeypatch.setattr(roots, "batch_add", mk("add"))
    monkeypatch.setattr(roots, "batch_mul", mk("mul"))
    monkeypatch.setattr(roots, "batch_div", mk("div"))


@pytest.mark.parametrize("k,v", [(2, "bf"), (3, "bf"), (4, "bf"), (2, "std"), (3, "std"), (4, "std")])
def test_aberth_init_host_logic_matches_reference(golden, monkeypatch, k, v):
    """radius_estimate (mpmath) + angles + lane ops reproduce the
    reference's aberth_init state bit for bit (roots.py:188-221)."""
    _oracle_batch(monkeypatch)
    g = golden("dk")
    p = f"k{k}_{v}"
    q = MonicPoly(g[p + "_coeffs"], device="cpu")
    st = roots.aberth_init(q, Variant.parse(v))
    assert_bitwise(st.re.numpy(), g[p + "_zre"])
    assert_bitwise(st.im.numpy(), g[p + "_zim"])


@pytest.mark.parametrize("k", [3, 4])
def test_aberth_init_config5_circle_host_logic(golden, monkeypatch, k):
    """The R0 = 1.5 circle of config 5 (radius override) with the oracle for
    the lane ops equals the reference's state (roots.py:199-217)."""
    _oracle_batch(monkeypatch)
    g = golden("dk")
    p = f"c5_k{k}"
    st = roots.aberth_init(MonicPoly(g[p + "_coeffs"], device="cpu"), Variant.BRANCH_FREE, radius=1.5)
    assert_bitwise(st.re.numpy(), g[p + "_ab_zre"])
    assert_bitwise(st.im.numpy(), g[p + "_ab_zim"])


def test_aberth_init_collision_check(monkeypatch):
    _oracle_batch(monkeypatch)
    st = RootState(re=np.array([[0.5, 0.5], [0.0, 0.0]]), im=np.array([[0.1, 0.1], [0.0, 0.0]]))
    with pytest.raises(roots.CollisionError):
        roots._check_distinct(st)


def test_generators_are_seeded_and_normalised():
    rng1, rng2 = np.random.default_rng(0), np.random.default_rng(0)
    a, b = gen.g_k(rng1, 4, 1000), gen.g_k(rng2, 4, 1000)
    assert_bitwise(a, b)
    # bottom-up quick_two_sum pass: c0 = fl(c0 + c1)
    assert np.array_equal(a[0] + a[1], a[0])
    x, y, alpha = gen.config1_dot(n=1024)
    assert x.shape == (2, 1024) and alpha.shape == (2,)
    coeffs, pts = gen.config4_horner(npts=100, degree=8)
    assert coeffs.shape == (4, 9) and not pts[1:].any()


@pytest.mark.parametrize("k,n", [(2, 24), (3, 17), (4, 16)])
def test_gen_complex_test_matrices_match_reference(golden, k, n):
    from paper_2603_14926_b200.linalg import gen_complex_test_matrices

    g = golden("cgemm")
    a, b = gen_complex_test_matrices(n, 20240806 + k, k, device="cpu")
    p = f"k{k}_bf"
    assert_bitwise(a.re.numpy(), g[p + "_a_re"])
    assert_bitwise(a.im.numpy(), g[p + "_a_im"])
    assert_bitwise(b.re.numpy(), g[p + "_b_re"])
    assert_bitwise(b.im.numpy(), g[p + "_b_im"])


def test_multiword_value_class_host_parts():
    from paper_2603_14926_b200 import DD, QD, MultiWord, TD
    from paper_2603_14926_b200.multiword import is_normalized

    assert DD(1.5).comps == (1.5, 0.0)
    assert MultiWord.from_components((1.0, 2.0**-60, 0.0)).__class__ is TD
    with pytest.raises(AttributeError):
        DD(1.0).comps = (2.0, 0.0)
    with pytest.raises(ValueError):
        DD(1.0, 2.0, 3.0)
    assert DD(1.0) == 1.0 and QD(2.0) == QD(2.0)
    assert abs(DD(-3.0)) == DD(3.0)  # negation needs no arithmetic kernel
    assert is_normalized((1.0, 2.0**-60)) and not is_normalized((1.0, 0.5))


DKSOLVE = [(2, "bf", 16), (3, "bf", 16), (4, "bf", 16), (2, "std", 16), (3, "std", 16), (4, "std", 16),
           (3, "bf", 64), (4, "bf", 64)]


@pytest.mark.parametrize("k,v,n", DKSOLVE, ids=[f"k{k}_{v}_n{n}" for k, v, n in DKSOLVE])
def test_dk_solve_oracle_loop_matches_reference(golden, monkeypatch, k, v, n):
    """The oracle's reference-order sweep, looped with the reference's
    convergence test (roots.py:334-339, np.hypot), from the Aberth start,
    reproduces the reference's dk_solve: same sweep count, same roots bit
    for bit (dksolve.npz, chebyshev_coeffs(n))."""
    _oracle_batch(monkeypatch)
    g = golden("dksolve")
    p = f"k{k}_{v}_n{n}"
    coeffs = g[p + "_coeffs"]
    st = roots.aberth_init(MonicPoly(coeffs, device="cpu"), Variant.parse(v))
    zre, zim = st.re.numpy(), st.im.numpy()
    tol = roots.default_tolerance(k)
    for it in range(1, 201):
        zre, zim, mag, coll = oracle.dk_sweep(coeffs, zre, zim, v, exact=True)
        assert coll is None
        zmag = float(np.max(np.hypot(zre[0], zim[0])))
        if float(mag.max()) <= tol * max(zmag, 1e-300):
            break
    assert it == int(g[p + "_iters"][0])
    assert_bitwise(zre, g[p + "_re"])
    assert_bitwise(zim, g[p + "_im"])
