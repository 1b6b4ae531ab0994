"""GPU parity of multiword's named kernels (multiword.py:104-588) and
helpers through the C-ABI: the twelve dispatched kernels (dw_add_bf ...
qw_mul_bf) against the reference's batch goldens, the kernels outside the
dispatch tables (dw_add_sloppy, tw_mul_cleaned), the renormalisers,
normalize and eft.fma against named.npz, each for float / numpy / torch
component forms, and against the oracle on larger seeded inputs."""

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_bitwise, rand_mw
from paper_2603_14926_b200 import eft, multiword as mwm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


NAMED = {
    (2, "std", "add"): "dw_add_accurate", (2, "bf", "add"): "dw_add_bf",
    (2, "std", "mul"): "dw_mul", (2, "bf", "mul"): "dw_mul_bf",
    (3, "std", "add"): "tw_add", (3, "bf", "add"): "tw_add_bf",
    (3, "std", "mul"): "tw_mul", (3, "bf", "mul"): "tw_mul_bf",
    (4, "std", "add"): "qw_add", (4, "bf", "add"): "qw_add_bf",
    (4, "std", "mul"): "qw_mul", (4, "bf", "mul"): "qw_mul_bf",
}


@pytest.mark.parametrize("key", sorted(NAMED), ids=[NAMED[k] for k in sorted(NAMED)])
def test_dispatched_named_kernels_vs_reference_batches(golden, key):
    k, v, op = key
    g = golden("ew")
    p = f"k{k}_{v}"
    fn = getattr(mwm, NAMED[key])
    a, b = g[p + "_a"], g[p + "_b"]
    got = fn(tuple(a), tuple(b))  # numpy components in, numpy out
    assert isinstance(got[0], np.ndarray)
    assert_bitwise(np.stack(got), g[p + "_" + op])
    # scalar components: floats out, same bits per lane
    for lane in (0, 3, 100):
        s = fn(tuple(float(c) for c in a[:, lane]), tuple(float(c) for c in b[:, lane]))
        assert all(isinstance(c, float) for c in s)
        assert_bitwise(np.array(s), g[p + "_" + op][:, lane])
    # torch components stay on the device
    t = fn(tuple(torch.from_numpy(c).cuda() for c in a), tuple(torch.from_numpy(c).cuda() for c in b))
    assert t[0].is_cuda
    assert_bitwise(torch.stack(t).cpu().numpy(), g[p + "_" + op])


def test_sloppy_and_cleaned_vs_reference(golden):
    g = golden("named")
    assert_bitwise(np.stack(mwm.dw_add_sloppy(tuple(g["sloppy_a"]), tuple(g["sloppy_b"]))), g["sloppy_out"])
    assert_bitwise(np.stack(mwm.tw_mul_cleaned(tuple(g["cleaned_a"]), tuple(g["cleaned_b"]))), g["cleaned_out"])
    lane = tuple(float(c) for c in g["cleaned_a"][:, 5]), tuple(float(c) for c in g["cleaned_b"][:, 5])
    assert_bitwise(np.array(mwm.tw_mul_cleaned(*lane)), g["cleaned_out"][:, 5])


def test_sloppy_and_cleaned_vs_oracle_large():
    rng = np.random.default_rng(11)
    for name, k in (("dw_add_sloppy", 2), ("tw_mul_cleaned", 3)):
        a, b = rand_mw(rng, k, 100_003), rand_mw(rng, k, 100_003)
        got = np.stack(getattr(mwm, name)(tuple(a), tuple(b)))
        assert_bitwise(got, oracle.named(name, a, b))


@pytest.mark.parametrize("k", [3, 4])
def test_renormalize_vs_reference(golden, k):
    g = golden("named")
    raw = g[f"renorm{k}_in"]
    fn = mwm.tw_renormalize if k == 3 else mwm.qw_renormalize
    assert_bitwise(np.stack(fn(*raw)), g[f"renorm{k}_out"], nan_ok=True)
    for lane in (1, 2, 7, 50):
        assert_bitwise(np.array(fn(*(float(c) for c in raw[:, lane]))), g[f"renorm{k}_out"][:, lane])


@pytest.mark.parametrize("k", [2, 3, 4])
def test_normalize_vs_reference(golden, k):
    g = golden("named")
    got = mwm.normalize(tuple(g[f"normalize{k}_in"]))
    assert_bitwise(np.stack(got), g[f"normalize{k}_out"])


def test_fma_vs_reference(golden):
    g = golden("named")
    assert_bitwise(eft.fma(g["fma_a"], g["fma_b"], g["fma_c"]), g["fma_out"])
    assert eft.fma(2.0**30 + 1, 2.0**30 + 1, -(2.0**60 + 2.0**31)) == 1.0  # exact residue
    t = eft.fma(torch.tensor([3.0], device="cuda"), 5.0, 1.0)
    assert t.is_cuda and float(t[0]) == 16.0


def test_oracle_conversions_round_trip():
    from fractions import Fraction

    x = Fraction(1, 3)
    for k in (2, 3, 4):
        w = mwm.from_oracle(x, k)
        assert abs(mwm.to_oracle(w) - x) <= abs(x) * Fraction(2) ** -(53 * k - 2)
        assert mwm.from_oracle(mwm.to_oracle(w), k) == w


def test_named_word_count_errors():
    with pytest.raises(ValueError):
        mwm.dw_add_bf((1.0, 0.0, 0.0), (1.0, 0.0, 0.0))
    with pytest.raises(ValueError):
        mwm.normalize((1.0,) * 5)


# --------------------------------------------- property tests (hypothesis)
from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@st.composite
def _raw_expansions(draw):
    """Decreasing raw expansions with random exponents, signs and zero
    terms (every renormalisation branch), 1..64 lanes."""
    k = draw(st.sampled_from([2, 3, 4]))
    w = draw(st.integers(1, 64))
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    m = {2: 2, 3: 4, 4: 5}[k]
    raw = np.zeros((m, w))
    raw[0] = rng.uniform(-1, 1, w) * np.exp2(rng.integers(-900, 900, w))
    for j in range(1, m):
        raw[j] = raw[j - 1] * np.exp2(-rng.integers(40, 60, w)) * rng.uniform(-1, 1, w)
    raw[rng.random((m, w)) < 0.25] = 0.0
    if k == 2:
        raw[1] = np.where(np.abs(raw[1]) > np.abs(raw[0]), 0.0, raw[1])  # quick_two_sum contract
    return k, raw


@given(_raw_expansions())
@settings(max_examples=120, deadline=None)
def test_property_renormalize_matches_oracle(case):
    k, raw = case
    got = np.stack(mwm._renorm(k, tuple(raw)))
    assert_bitwise(got, oracle.renormalize(k, raw))


@given(st.integers(0, 2**31 - 1), st.integers(1, 300))
@settings(max_examples=60, deadline=None)
def test_property_sloppy_cleaned_fma_match_oracle(seed, w):
    rng = np.random.default_rng(seed)
    a2, b2 = rand_mw(rng, 2, w, -500, 500), rand_mw(rng, 2, w, -500, 500)
    assert_bitwise(np.stack(mwm.dw_add_sloppy(tuple(a2), tuple(b2))), oracle.named("dw_add_sloppy", a2, b2))
    a3, b3 = rand_mw(rng, 3, w, -300, 300), rand_mw(rng, 3, w, -300, 300)
    assert_bitwise(np.stack(mwm.tw_mul_cleaned(tuple(a3), tuple(b3))), oracle.named("tw_mul_cleaned", a3, b3))
    x, y, z = (rng.uniform(-1, 1, w) * np.exp2(rng.integers(-300, 300, w)) for _ in range(3))
    assert_bitwise(eft.fma(x, y, z), oracle.fma(x, y, z))
