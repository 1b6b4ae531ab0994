import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def bits(a):
    """float64 array -> int64 view for bitwise comparison (signed zeros
    distinguished, NaNs compared by payload -- keep parity inputs finite)."""
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.int64)


def assert_bitwise(got, want, nan_ok=False):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    if nan_ok:
        gn, wn = np.isnan(got), np.isnan(want)
        assert np.array_equal(gn, wn), "NaN positions differ"
        got = np.where(gn, 0.0, got)
        want = np.where(wn, 0.0, want)
    g, w = bits(got), bits(want)
    if not np.array_equal(g, w):
        idx = np.argwhere(g != w)
        first = tuple(idx[0])
        raise AssertionError(
            f"{len(idx)} of {g.size} components differ bitwise; first at {first}: "
            f"got {got[first]!r} want {want[first]!r}"
        )


@pytest.fixture(scope="session")
def golden():
    return load_golden


def rand_mw(rng, k, w, e_lo=-100, e_hi=100):
    """Normalized wide-exponent K-word values: the reference tests'
    generator (pkg/tests/conftest.py:127-133), component-planar."""
    c0 = rng.uniform(1.0, 2.0, w) * np.exp2(rng.integers(e_lo, e_hi + 1, w))
    c0 *= np.where(rng.random(w) < 0.5, -1.0, 1.0)
    comps = [c0]
    for _ in range(1, k):
        comps.append(comps[-1] * 2.0**-53 * rng.uniform(-0.49, 0.49, w))
    return np.stack(comps)
