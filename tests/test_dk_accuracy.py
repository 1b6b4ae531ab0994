"""Accuracy contract of the tree-order DK sweep against the reference
(roots.py:240-315) and against an mpmath step, at config 5 (n = 512, TD and
QD, the near-root start and the R0 = 1.5 Aberth circle).

The contract (tests/dk_accuracy.py): per root,

    |z_tree - z_ref| <= C_TREE * B_i + 2^(1-p) |z_i|,
    B_i = n 2^-p sum_j |c_j| |z_i|^j / |prod_{j != i}(z_i - z_j)|,

C_TREE = 2 (measured worst 0.39, TD Aberth circle; the tree order's complex
products are the four-multiplication form, oracle c_mul4).  Against the mpmath
step on the worst roots (largest B_i and largest tree-vs-reference
difference) the tree's largest error is within 10x the reference's largest
error (measured <= 3.5x).  SURVEY's size-only bound n 2^(-p+4)|step| +
2^-p|z| is missed by the reference's own step on the ill-conditioned roots
-- recorded by a test below -- which is why the contract is
condition-aware.

CPU tests use the oracle's restatement of the tree order (pinned bit for
bit to the GPU kernel by the -m gpu tests here and in test_gpu_parity.py);
the -m gpu tests run the CUDA kernel itself.
"""

import math

import numpy as np
import pytest

import dk_accuracy as acc
import oracle

CASES = [(3, ""), (3, "_ab"), (4, ""), (4, "_ab")]
IDS = ["td_near", "td_aberth", "qd_near", "qd_aberth"]


def _case(golden, k, s):
    g = golden("dk")
    p = f"c5_k{k}"
    return (g[p + "_coeffs"], g[p + s + "_zre"], g[p + s + "_zim"], g[p + s + "_new_re"], g[p + s + "_new_im"])


def _worst(ratio, b, m=8):
    return np.unique(np.r_[np.argsort(-b)[:m], np.argsort(-ratio)[:m]])


def _check_contract(coeffs, zre, zim, tre, tim, rre, rim):
    ratio, b = acc.contract_ratio(coeffs, zre, zim, tre, tim, rre, rim)
    assert np.all(np.isfinite(ratio))
    assert ratio.max() <= acc.C_TREE, f"worst |tree - ref| / bound = {ratio.max():.3g} (root {ratio.argmax()})"
    idx = _worst(ratio, b)
    ee = np.array(acc.exact_errors(coeffs, zre, zim, tre, tim, rre, rim, idx))
    k = np.asarray(coeffs).shape[0]
    floor = math.ldexp(1.0, -acc.P_BITS[k]) * ee[:, 2]
    err_tree, err_ref = ee[:, 0], ee[:, 1]
    # tree vs the exact step: within the contract on every sampled root ...
    assert np.all(err_tree <= acc.C_TREE * b[idx] + 2 * floor), (err_tree, b[idx])
    # ... and its worst error within 10x the reference's worst error there
    assert err_tree.max() <= acc.EXACT_FACTOR * max(err_ref.max(), floor.max()), (err_tree.max(), err_ref.max())
    return ratio, err_tree, err_ref


@pytest.mark.parametrize("k,s", CASES, ids=IDS)
def test_tree_restatement_meets_contract(golden, k, s):
    coeffs, zre, zim, rre, rim = _case(golden, k, s)
    tre, tim, _, coll = oracle.dk_sweep(coeffs, zre, zim, "bf", exact=False)
    assert coll is None
    _check_contract(coeffs, zre, zim, tre, tim, rre, rim)


@pytest.mark.parametrize("k,s", [(3, ""), (4, "")], ids=["td_near", "qd_near"])
def test_reference_misses_the_size_only_bound(golden, k, s):
    """SURVEY §8(d)(i)'s |dz| <= n 2^(-p+4) |step| + 2^-p |z| does not hold
    for the reference's own step against the exact step on the worst
    conditioned roots: a tree-order kernel cannot be held to it."""
    coeffs, zre, zim, rre, rim = _case(golden, k, s)
    b = acc.cond_bound(coeffs, zre, zim)
    idx = np.argsort(-b)[:4]
    n, p = zre.shape[1], acc.P_BITS[k]
    missed = 0
    for i in idx:
        ex, ctx = acc.exact_step(coeffs, zre, zim, int(i))
        z0 = ctx.mpc(ctx.fsum(ctx.mpf(float(c)) for c in zre[:, i]), ctx.fsum(ctx.mpf(float(c)) for c in zim[:, i]))
        ref = ctx.mpc(ctx.fsum(ctx.mpf(float(c)) for c in rre[:, i]), ctx.fsum(ctx.mpf(float(c)) for c in rim[:, i]))
        step = abs(ex - z0)
        size_bound = n * ctx.mpf(2) ** (-p + 4) * step + ctx.mpf(2) ** (-p) * abs(ex)
        missed += abs(ref - ex) > size_bound
    assert missed >= 1


def test_contract_bound_is_finite_and_positive(golden):
    coeffs, zre, zim, _, _ = _case(golden, 3, "_ab")
    b = acc.cond_bound(coeffs, zre, zim)
    assert b.shape == (512,) and np.all(np.isfinite(b)) and np.all(b > 0)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("k,s", CASES, ids=IDS)
def test_gpu_tree_sweep_meets_contract(golden, k, s):
    from paper_2603_14926_b200 import MonicPoly, RootState, Variant, dk_iterate

    coeffs, zre, zim, rre, rim = _case(golden, k, s)
    nxt = dk_iterate(MonicPoly(coeffs), RootState(re=zre, im=zim), Variant.BRANCH_FREE, exact_order=False)
    tre, tim = nxt.re.cpu().numpy(), nxt.im.cpu().numpy()
    ore, oim, _, _ = oracle.dk_sweep(coeffs, zre, zim, "bf", exact=False)
    assert np.array_equal(tre.view(np.int64), ore.view(np.int64))
    assert np.array_equal(tim.view(np.int64), oim.view(np.int64))
    _check_contract(coeffs, zre, zim, tre, tim, rre, rim)


PLATEAU = {3: (5, 1e-12, 1e-11), 4: (20, 5e-29, 1e-27)}  # from sweep s on: lo <= max update <= hi


@pytest.mark.gpu
@pytest.mark.parametrize("k", [3, 4])
def test_dk_config5_200_sweeps_exact_bitwise_and_plateau(k):
    """The full config-5 run: 200 exact-order sweeps from the near-root
    start, every sweep's state bitwise equal to the oracle trajectory (the
    reference order, roots.py:240-315), and the max update plateau SURVEY
    §8(d) measured with the reference: TD 1e-12..1e-11 from sweep 5, QD
    5e-29..1e-27 from sweep 20."""
    from paper_2603_14926_b200 import MonicPoly, RootState, Variant, dk_iterate, gen

    coeffs = gen.config5_poly(k)
    zre, zim = gen.config5_init(k)
    q = MonicPoly(coeffs)
    st = RootState(re=zre, im=zim)
    ore, oim = zre, zim
    mags = []
    for s in range(200):
        st = dk_iterate(q, st, Variant.BRANCH_FREE, exact_order=True)
        ore, oim, omag, coll = oracle.dk_sweep(coeffs, ore, oim, "bf", exact=True)
        assert coll is None
        gre, gim = st.re.cpu().numpy(), st.im.cpu().numpy()
        assert np.array_equal(gre.view(np.int64), ore.view(np.int64)), f"sweep {s + 1}"
        assert np.array_equal(gim.view(np.int64), oim.view(np.int64)), f"sweep {s + 1}"
        assert math.isclose(st.last_max_update, float(omag.max()), rel_tol=1e-15)
        mags.append(st.last_max_update)
    first, lo, hi = PLATEAU[k]
    tail = np.array(mags[first - 1:])
    assert np.all(np.isfinite(tail)) and tail.min() >= lo and tail.max() <= hi, (tail.min(), tail.max())
