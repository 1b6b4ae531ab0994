"""Word counts, the Variant selector, scalar K-word operations and the
DD / TD / QD value classes.

Mirrors mwfloat.multiword (pkg/src/mwfloat/multiword.py): ``Variant``
(82-96), ``BITS`` (76), ``ulp_k`` (722-730), ``from_basefloat`` (749-752),
the greedy ``from_oracle`` rounding (760-775, here for exact Fractions),
the scalar ``mw_*`` / complex ``c*``
operations (617-702) and the immutable ``MultiWord``/``DD``/``TD``/``QD``
classes (850-1004).  All arithmetic runs in the CUDA kernels; scalar
operations are one-lane launches.
"""

from __future__ import annotations

import enum
import math
from fractions import Fraction

__all__ = [
    "Variant", "BITS", "ulp_k", "from_basefloat", "from_fraction", "variant_code",
    "mw_add", "mw_sub", "mw_mul", "mw_div", "mw_neg", "cadd", "csub", "cmul", "cdiv",
    "is_normalized", "MultiWord", "DD", "TD", "QD",
    # the reference's named per-variant kernels (multiword.py:104-588) and helpers
    "dw_add_sloppy", "dw_add_accurate", "dw_add_bf", "dw_mul", "dw_mul_bf",
    "tw_add", "tw_mul", "tw_mul_cleaned", "tw_add_bf", "tw_mul_bf",
    "qw_add", "qw_mul", "qw_add_bf", "qw_mul_bf",
    "tw_renormalize", "qw_renormalize", "normalize", "to_oracle", "from_oracle",
]

BITS = {2: 106, 3: 159, 4: 212}


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
    if v is Variant.BRANCH_FREE:  # fast path: on every call's host path
        return 1
    if v is Variant.STANDARD:
        return 0
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


# --------------------------------------------------------------------------
# scalar K-word operations and the immutable value classes
# (multiword.py:617-702, 850-1004).  Each scalar operation is a one-lane
# launch of the same device kernels the batches use (no CPU arithmetic):
# correct and bit-identical, but latency-bound -- batch work through
# LaneBatch / MWMatrix instead.
# --------------------------------------------------------------------------


def _scalar_op(name: str, a, b, variant) -> tuple:
    import numpy as np

    from .batch import LaneBatch, batch_add, batch_div, batch_mul, batch_sub

    a = tuple(float(c) for c in a)
    b = tuple(float(c) for c in b)
    if len(a) != len(b):
        raise ValueError("mixed word counts")
    if len(a) not in BITS:
        raise ValueError(f"unsupported word count {len(a)}")
    fn = {"add": batch_add, "sub": batch_sub, "mul": batch_mul, "div": batch_div}[name]
    la = LaneBatch(np.array(a).reshape(-1, 1))
    lb = LaneBatch(np.array(b).reshape(-1, 1))
    return fn(la, lb, variant).lane(0)


def mw_add(a, b, variant: Variant = Variant.STANDARD) -> tuple:
    return _scalar_op("add", a, b, variant)


def mw_sub(a, b, variant: Variant = Variant.STANDARD) -> tuple:
    """add(a, -b) (multiword.py:629-630), one fused lane kernel."""
    return _scalar_op("sub", a, b, variant)


def mw_mul(a, b, variant: Variant = Variant.STANDARD) -> tuple:
    return _scalar_op("mul", a, b, variant)


def mw_div(a, b, variant: Variant = Variant.STANDARD) -> tuple:
    """Newton reciprocal division (multiword.py:661-668)."""
    return _scalar_op("div", a, b, variant)


def mw_neg(a) -> tuple:
    return tuple(-float(c) for c in a)


def cadd(a, b, variant: Variant = Variant.STANDARD):
    return mw_add(a[0], b[0], variant), mw_add(a[1], b[1], variant)


def csub(a, b, variant: Variant = Variant.STANDARD):
    return mw_sub(a[0], b[0], variant), mw_sub(a[1], b[1], variant)


def cmul(a, b, variant: Variant = Variant.STANDARD):
    """Three-multiplication complex product (multiword.py:683-692)."""
    ar, ai = a
    br, bi = b
    p1 = mw_mul(ar, br, variant)
    p2 = mw_mul(ai, bi, variant)
    p3 = mw_mul(mw_add(ar, ai, variant), mw_add(br, bi, variant), variant)
    return mw_sub(p1, p2, variant), mw_sub(mw_sub(p3, p1, variant), p2, variant)


def cdiv(a, b, variant: Variant = Variant.STANDARD):
    """(a conj(b)) / |b|^2 (multiword.py:695-702)."""
    ar, ai = a
    br, bi = b
    den = mw_add(mw_mul(br, br, variant), mw_mul(bi, bi, variant), variant)
    num_re = mw_add(mw_mul(ar, br, variant), mw_mul(ai, bi, variant), variant)
    num_im = mw_sub(mw_mul(ai, br, variant), mw_mul(ar, bi, variant), variant)
    return mw_div(num_re, den, variant), mw_div(num_im, den, variant)


# --------------------------------------------------------------------------
# The reference's named kernels (multiword.py:104-588), each taking and
# returning a tuple of K components.  As in the reference, a component may
# be a float or an array (numpy or torch, any shape; all of one shape):
# floats give floats, numpy arrays give numpy arrays, torch tensors give
# CUDA tensors.  All arithmetic runs on the device: the dispatched
# (K, Variant) lane kernels, or mw_named_op / mw_renormalize for the
# kernels no dispatch table selects.
# --------------------------------------------------------------------------


def _to_planes(*tuples):
    """Stack component tuples into (m, W) CUDA planes; returns (planes,
    kind, shape) with kind "float" / "numpy" / "torch"."""
    import numpy as np
    import torch

    from . import _lib

    comps = [c for t in tuples for c in t]
    if any(isinstance(c, torch.Tensor) for c in comps):
        kind = "torch"
    elif any(isinstance(c, np.ndarray) and c.ndim > 0 for c in comps):
        kind = "numpy"
    else:
        kind = "float"
    dev = next((c.device for c in comps if isinstance(c, torch.Tensor) and c.is_cuda), torch.device("cuda"))
    if kind != "torch":
        # host operands: broadcast and stack on the host, one copy up (no
        # device-side stack kernel on this path)
        arrs = np.broadcast_arrays(*[np.asarray(c, dtype=np.float64) for c in comps])
        shape = arrs[0].shape
        host = np.ascontiguousarray(np.stack([a.reshape(-1) for a in arrs]))
        planes = torch.from_numpy(host).to(dev)
        _lib.require_cuda(planes)
        return planes, kind, tuple(shape)
    ts = [torch.as_tensor(c, dtype=torch.float64).to(dev) if isinstance(c, torch.Tensor)
          else torch.as_tensor(np.asarray(c, dtype=np.float64), device=dev) for c in comps]
    shape = torch.broadcast_shapes(*(t.shape for t in ts))
    planes = torch.stack([t.expand(shape).reshape(-1) for t in ts]).contiguous()
    _lib.require_cuda(planes)
    return planes, kind, tuple(shape)


def _from_planes(planes, kind, shape) -> tuple:
    if kind == "float":
        return tuple(float(v) for v in planes[:, 0].cpu())
    if kind == "numpy":
        host = planes.cpu().numpy()
        return tuple(host[c].reshape(shape) for c in range(planes.shape[0]))
    return tuple(planes[c].reshape(shape) for c in range(planes.shape[0]))


def _need_k(t, k):
    if len(t) != k:
        raise ValueError(f"expected {k} components, got {len(t)}")


def _dispatched(k, variant, op):
    """The (K, Variant) kernel of the dispatch tables (multiword.py:595-611)."""

    def fn(a, b):
        from . import _lib

        _need_k(a, k)
        _need_k(b, k)
        planes, kind, shape = _to_planes(a, b)
        n = planes.shape[1]
        out = planes.new_empty((k, n))
        lib = _lib.load()
        call = lib.mw_ew_add if op == "add" else lib.mw_ew_mul
        rc = call(k, variant_code(variant), planes.data_ptr(), n, planes[k:].data_ptr(), n,
                  out.data_ptr(), n, n, _lib.stream_handle(planes.device))
        _lib.check(rc, f"mw_ew_{op}")
        return _from_planes(out, kind, shape)

    return fn


dw_add_accurate = _dispatched(2, Variant.STANDARD, "add")  # multiword.py:118-126
dw_add_bf = _dispatched(2, Variant.BRANCH_FREE, "add")  # 129-137
dw_mul = _dispatched(2, Variant.STANDARD, "mul")  # 140-145
dw_mul_bf = _dispatched(2, Variant.BRANCH_FREE, "mul")  # 148-156
tw_add = _dispatched(3, Variant.STANDARD, "add")  # 279-280
tw_mul = _dispatched(3, Variant.STANDARD, "mul")  # 321-322
tw_add_bf = _dispatched(3, Variant.BRANCH_FREE, "add")  # 361-378
tw_mul_bf = _dispatched(3, Variant.BRANCH_FREE, "mul")  # 381-402
qw_add = _dispatched(4, Variant.STANDARD, "add")  # 442-487
qw_mul = _dispatched(4, Variant.STANDARD, "mul")  # 512-513
qw_add_bf = _dispatched(4, Variant.BRANCH_FREE, "add")  # 516-545
qw_mul_bf = _dispatched(4, Variant.BRANCH_FREE, "mul")  # 548-588
for _f, _n in ((dw_add_accurate, "dw_add_accurate"), (dw_add_bf, "dw_add_bf"), (dw_mul, "dw_mul"),
               (dw_mul_bf, "dw_mul_bf"), (tw_add, "tw_add"), (tw_mul, "tw_mul"), (tw_add_bf, "tw_add_bf"),
               (tw_mul_bf, "tw_mul_bf"), (qw_add, "qw_add"), (qw_mul, "qw_mul"), (qw_add_bf, "qw_add_bf"),
               (qw_mul_bf, "qw_mul_bf")):
    _f.__name__ = _f.__qualname__ = _n
del _f, _n


def _named(code, k, a, b):
    from . import _lib

    _need_k(a, k)
    _need_k(b, k)
    planes, kind, shape = _to_planes(a, b)
    n = planes.shape[1]
    out = planes.new_empty((k, n))
    rc = _lib.load().mw_named_op(code, planes.data_ptr(), n, planes[k:].data_ptr(), n, out.data_ptr(), n, n,
                                 _lib.stream_handle(planes.device))
    _lib.check(rc, "mw_named_op")
    return _from_planes(out, kind, shape)


def dw_add_sloppy(a, b):
    """Fast DD addition without the low-part error term (multiword.py:104-115)."""
    return _named(0, 2, a, b)


def tw_mul_cleaned(a, b):
    """tw_mul with the dangling error chain folded into the tail (multiword.py:325-358)."""
    return _named(1, 3, a, b)


def _renorm(k, raw):
    from . import _lib

    planes, kind, shape = _to_planes(raw)
    n = planes.shape[1]
    out = planes.new_empty((k, n))
    rc = _lib.load().mw_renormalize(k, planes.data_ptr(), n, out.data_ptr(), n, n,
                                    _lib.stream_handle(planes.device))
    _lib.check(rc, "mw_renormalize")
    return _from_planes(out, kind, shape)


def tw_renormalize(s0, s1, s2, t0):
    """Decreasing four-term expansion -> triple word (multiword.py:191-194)."""
    return _renorm(3, (s0, s1, s2, t0))


def qw_renormalize(x0, x1, x2, x3, x4):
    """Decreasing five-term expansion -> quadruple word (multiword.py:197-241)."""
    return _renorm(4, (x0, x1, x2, x3, x4))


def normalize(comps):
    """Raw components -> non-overlapping form (multiword.py:710-719)."""
    k = len(comps)
    if k == 2:
        return _renorm(2, tuple(comps))
    if k == 3:
        return _renorm(3, tuple(comps) + (0.0,))
    if k == 4:
        return _renorm(4, tuple(comps) + (0.0,))
    raise ValueError(f"unsupported word count {k}")


def to_oracle(comps) -> Fraction:
    """Exact value of a K-word tuple (multiword.py:755-757); the reference
    returns its OracleValue, here the exact dyadic ``Fraction``."""
    return sum((Fraction(float(c)) for c in comps), Fraction(0))


def from_oracle(value, k: int) -> tuple:
    """Greedy nearest-double extraction to K words (multiword.py:760-775);
    accepts anything ``Fraction`` accepts or an object with
    ``as_fraction()`` / ``to_fraction()``."""
    for attr in ("as_fraction", "to_fraction"):
        if hasattr(value, attr):
            value = getattr(value, attr)()
            break
    return from_fraction(value, k)


def is_normalized(comps) -> bool:
    """Non-overlap invariant (733-741): every component is at most half an
    ulp of the one before it, and nothing follows a zero component."""
    prev = None
    for c in comps:
        if prev is not None:
            if prev == 0.0 and c != 0.0:
                return False
            if prev != 0.0 and abs(c) > math.ulp(abs(prev)) / 2:
                return False
        prev = c
    return True


# The value classes (multiword.py:850-1004): an immutable tuple of K
# floats with the Standard-variant operators.  The operator methods are
# generated from one table; every arithmetic operator is a one-lane device
# kernel (mw_add / mw_sub / mw_mul / mw_div above).
_BINOPS = {"add": mw_add, "sub": mw_sub, "mul": mw_mul, "truediv": mw_div}


def _operator(op: str, reflected: bool):
    fn = _BINOPS[op]

    def method(self, other):
        rhs = self._as_comps(other)
        if rhs is NotImplemented:
            return NotImplemented
        return self._of(fn(rhs, self.comps) if reflected else fn(self.comps, rhs))

    method.__name__ = f"__{'r' if reflected else ''}{op}__"
    return method


class MultiWord:
    """Immutable K-word value: ``comps`` is a tuple of K floats, leading
    component first.  ``DD``, ``TD`` and ``QD`` fix K; the base class takes
    K from the number of components.  Operators use the Standard variant,
    as the reference's do."""

    __slots__ = ("comps",)

    K: int | None = None

    def __init__(self, *parts):
        seq = parts[0] if len(parts) == 1 and isinstance(parts[0], (tuple, list)) else parts
        k = len(seq) if self.K is None else self.K
        if k not in BITS:
            raise ValueError(f"unsupported word count {k}")
        if len(seq) > k:
            raise ValueError(f"{len(seq)} components for a {k}-word value")
        padded = [float(v) for v in seq] + [0.0] * (k - len(seq))
        object.__setattr__(self, "comps", tuple(padded))

    def __setattr__(self, name, value):
        raise AttributeError("MultiWord values are immutable")

    # -- construction / conversion
    @property
    def k(self) -> int:
        return len(self.comps)

    @staticmethod
    def _of(comps) -> "MultiWord":
        return _CLASS_BY_K[len(comps)](*comps)

    @classmethod
    def from_components(cls, comps) -> "MultiWord":
        return MultiWord._of(tuple(comps))

    @classmethod
    def from_float(cls, x: float, k: int | None = None) -> "MultiWord":
        width = cls.K or k or 2
        return MultiWord._of(from_basefloat(x, width))

    def to_float(self) -> float:
        """Components summed smallest first in binary64."""
        total = 0.0
        for c in self.comps[::-1]:
            total += c
        return total

    def to_fraction(self) -> Fraction:
        return sum(map(Fraction, self.comps), Fraction(0))

    def _as_comps(self, other):
        if isinstance(other, MultiWord):
            if other.k != self.k:
                raise ValueError("mixed word counts")
            return other.comps
        if isinstance(other, (int, float)):
            return from_basefloat(float(other), self.k)
        return NotImplemented

    # -- arithmetic (one-lane device kernels, Standard variant)
    # x + y and y + x both compute mw_add(x, y) (and likewise *), exactly
    # as the reference aliases __radd__ / __rmul__ (the Standard kernels
    # are not all bitwise commutative); - and / really reflect
    __add__ = __radd__ = _operator("add", False)
    __sub__ = _operator("sub", False)
    __rsub__ = _operator("sub", True)
    __mul__ = __rmul__ = _operator("mul", False)
    __truediv__ = _operator("truediv", False)
    __rtruediv__ = _operator("truediv", True)

    def __neg__(self):
        return MultiWord._of(mw_neg(self.comps))

    def __abs__(self):
        return self if self.comps[0] >= 0.0 else -self

    # -- comparison by exact value
    def __eq__(self, other):
        if isinstance(other, (int, float)):
            return self.to_fraction() == Fraction(float(other))
        if isinstance(other, MultiWord):
            return self.k == other.k and self.to_fraction() == other.to_fraction()
        return NotImplemented

    def __hash__(self):
        return hash(self.to_fraction())

    def __repr__(self):
        label = f"MultiWord{self.k}" if self.K is None else type(self).__name__
        return label + "(" + ", ".join(map(repr, self.comps)) + ")"

    __str__ = __repr__


DD = type("DD", (MultiWord,), {"K": 2, "__slots__": (), "__doc__": "Double-word (double-double) value."})
TD = type("TD", (MultiWord,), {"K": 3, "__slots__": (), "__doc__": "Triple-word value."})
QD = type("QD", (MultiWord,), {"K": 4, "__slots__": (), "__doc__": "Quadruple-word (quad-double) value."})
DD.__module__ = TD.__module__ = QD.__module__ = __name__

_CLASS_BY_K = {2: DD, 3: TD, 4: QD}
