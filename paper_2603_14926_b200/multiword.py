"""Word counts, the Variant selector and small host-side helpers.

Mirrors the parts of mwfloat.multiword (pkg/src/mwfloat/multiword.py) the
array-level API needs: ``Variant`` (82-96), ``BITS`` (76), ``ulp_k``
(722-730), ``from_basefloat`` (749-752) and the greedy ``from_oracle``
rounding (760-775, here for exact Fractions).  The arithmetic itself lives
only in the CUDA kernels.
"""

from __future__ import annotations

import enum
import math
from fractions import Fraction

__all__ = ["Variant", "BITS", "DEFAULT_DIGITS", "ulp_k", "from_basefloat", "from_fraction", "variant_code"]

BITS = {2: 106, 3: 159, 4: 212}
DEFAULT_DIGITS = {2: 34, 3: 49, 4: 64}


class Variant(enum.Enum):
    """Selects conventional (Standard) or branch-free kernels."""

    STANDARD = "std"
    BRANCH_FREE = "bf"

    @classmethod
    def parse(cls, name) -> "Variant":
        if isinstance(name, cls):
            return name
        # accept the reference's own enum (same values) and strings
        key = str(getattr(name, "value", name)).lower()
        for v in cls:
            if v.value == key or v.name.lower() == key:
                return v
        raise ValueError(f"unknown variant {name!r}")


def variant_code(v) -> int:
    """C-ABI code: MW_VARIANT_STANDARD = 0, MW_VARIANT_BRANCH_FREE = 1."""
    return 1 if Variant.parse(v) is Variant.BRANCH_FREE else 0


def ulp_k(scale: float, k: int) -> float:
    """Spacing of the K-word grid at |scale|: scale in [2^(e-1), 2^e) -> 2^(e-53K)."""
    if scale == 0.0 or not math.isfinite(scale):
        raise ValueError("ulp needs a finite nonzero scale")
    _, e = math.frexp(abs(scale))
    return math.ldexp(1.0, e - 53 * k)


def from_basefloat(x: float, k: int) -> tuple:
    if k not in BITS:
        raise ValueError(f"unsupported word count {k}")
    return (float(x),) + (0.0,) * (k - 1)


def from_fraction(value, k: int) -> tuple:
    """Round an exact rational to K words by greedy nearest-double
    extraction (multiword.from_oracle)."""
    if k not in BITS:
        raise ValueError(f"unsupported word count {k}")
    fr = Fraction(value)
    out = []
    for _ in range(k):
        c = float(fr)
        out.append(c)
        fr -= Fraction(c)
    return tuple(out)
