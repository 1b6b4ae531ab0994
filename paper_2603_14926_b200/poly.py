"""Real-coefficient polynomial evaluation on the GPU (Horner, Estrin,
complex points).

Drop-in for the Horner path of mwfloat.poly (pkg/src/mwfloat/poly.py):
``MWPolynomial`` (40-86) keeps coefficients a[0..n] (a[i] multiplies x^i)
as a (K, n+1) float64 CUDA tensor; ``horner_eval(p, x, variant)`` (89-96)
keeps its signature and returns the K-word tuple; the batched form
``horner_eval_batched(p, xs: LaneBatch, variant)`` (the name pattern of
estrin_eval_batched, 125-153) evaluates every lane with the same op
sequence in one mw_horner launch -- bit-exact per point.  ``estrin_eval``
/ ``estrin_eval_batched`` (106-153) and ``eval_complex`` (156-178, Horner
or Estrin with the 3M complex product) run through mw_poly_eval, also
bit-exact per point; ``eval_complex_batched`` is the lane-batched form.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .batch import LaneBatch, as_planes, coefficient_planes
from .multiword import BITS, Variant, from_basefloat, variant_code

__all__ = [
    "MWPolynomial",
    "horner_eval",
    "horner_eval_batched",
    "horner_into",
    "estrin_eval",
    "estrin_eval_batched",
    "eval_complex",
    "eval_complex_batched",
    "random_polynomial",
]

_METHODS = {"horner": 0, "estrin": 1}


class MWPolynomial:
    """Coefficients a[0..n] (a[i] multiplies x^i), component-planar."""

    __slots__ = ("planes",)

    def __init__(self, comps, device=None):
        self.planes = as_planes(comps, 1, device)
        if self.planes.shape[1] == 0:
            raise ValueError("a polynomial needs at least one coefficient")

    @property
    def comps(self) -> tuple:
        return tuple(self.planes[c] for c in range(self.k))

    @property
    def k(self) -> int:
        return self.planes.shape[0]

    @property
    def degree(self) -> int:
        return self.planes.shape[1] - 1

    @property
    def device(self) -> torch.device:
        return self.planes.device

    @classmethod
    def from_coeffs(cls, coeffs, k: int | None = None, device=None) -> "MWPolynomial":
        """coeffs: K-word tuples / objects with .comps / floats, low to high."""
        return cls(coefficient_planes(coeffs, k), device=device)

    def coeff(self, i: int) -> tuple:
        return tuple(float(v) for v in self.planes[:, i].cpu())

    def coeffs(self) -> list:
        arr = self.planes.cpu().numpy()
        return [tuple(float(v) for v in arr[:, i]) for i in range(self.degree + 1)]

    def __repr__(self):
        return f"MWPolynomial(k={self.k}, degree={self.degree}, device={self.device})"


def horner_into(coeffs: torch.Tensor, x: torch.Tensor, y: torch.Tensor, variant, p0: int = 0,
                p1: int | None = None) -> None:
    """y[:, p0:p1] = Horner(coeffs, x[:, p0:p1]) on planes tensors -- the
    point-shard form the multi-GPU path uses."""
    _lib.ext().horner(variant_code(variant), coeffs, x, y, p0, -1 if p1 is None else p1)


def horner_eval_batched(p: MWPolynomial, xs: LaneBatch, variant: Variant = Variant.STANDARD) -> LaneBatch:
    """Per-lane bitwise equal to horner_eval at each lane's point."""
    if xs.k != p.k:
        raise ValueError("mixed word counts")
    _lib.require_cuda(p.planes, xs.planes)
    y = torch.empty_like(xs.planes)
    horner_into(p.planes, xs.planes, y, variant)
    return LaneBatch._wrap(y, xs.count)


def horner_eval(p: MWPolynomial, x, variant: Variant = Variant.STANDARD) -> tuple:
    """b := a[n]; b := b*x + a[i] downward at one K-word point x."""
    x = tuple(float(c) for c in getattr(x, "comps", x))
    if len(x) != p.k:
        raise ValueError("mixed word counts")
    xs = LaneBatch(np.array(x, dtype=np.float64).reshape(p.k, 1), device=p.device)
    return horner_eval_batched(p, xs, variant).lane(0)


def _poly_eval(p: MWPolynomial, xre: torch.Tensor, xim, variant, method: str):
    if method not in _METHODS:
        raise ValueError(f"unknown method {method!r}")
    _lib.require_cuda(p.planes, xre)
    k, npts = xre.shape
    yre = torch.empty_like(xre)
    yim = torch.empty_like(xim) if xim is not None else None
    rc = _lib.load().mw_poly_eval(
        k, variant_code(variant), p.planes.data_ptr(), p.planes.shape[1], p.degree,
        xre.data_ptr(), None if xim is None else xim.data_ptr(), npts,
        yre.data_ptr(), None if yim is None else yim.data_ptr(), npts, npts, _METHODS[method],
        _lib.stream_handle(xre.device),
    )
    _lib.check(rc, "mw_poly_eval")
    return yre, yim


def estrin_eval_batched(p: MWPolynomial, xs: LaneBatch, variant: Variant = Variant.STANDARD) -> LaneBatch:
    """Per-lane bitwise equal to estrin_eval at each lane's point
    (poly.py:125-153)."""
    if xs.k != p.k:
        raise ValueError("mixed word counts")
    y, _ = _poly_eval(p, xs.planes, None, variant, "estrin")
    return LaneBatch(y, count=xs.count)


def estrin_eval(p: MWPolynomial, x, variant: Variant = Variant.STANDARD) -> tuple:
    """Pairwise combine a[2i] + a[2i+1] * x, square x, repeat (poly.py:106-122)."""
    x = tuple(float(c) for c in getattr(x, "comps", x))
    if len(x) != p.k:
        raise ValueError("mixed word counts")
    xs = LaneBatch(np.array(x, dtype=np.float64).reshape(p.k, 1), device=p.device)
    return estrin_eval_batched(p, xs, variant).lane(0)


def eval_complex_batched(p: MWPolynomial, zre: LaneBatch, zim: LaneBatch, method: str = "horner",
                         variant: Variant = Variant.STANDARD):
    """Evaluate at complex points (zre + i zim) lane-wise with the 3M
    complex product; returns (re, im) batches (poly.py:156-178 per lane)."""
    if zre.k != p.k or zim.k != p.k:
        raise ValueError("mixed word counts")
    if zre.width != zim.width:
        raise ValueError("mixed lane widths")
    yre, yim = _poly_eval(p, zre.planes, zim.planes, variant, method)
    return LaneBatch(yre, count=zre.count), LaneBatch(yim, count=zre.count)


def eval_complex(p: MWPolynomial, z, method: str = "horner", variant: Variant = Variant.STANDARD):
    """Evaluate at one complex point z = (re, im) of K-word tuples."""
    re = tuple(float(c) for c in z[0])
    im = tuple(float(c) for c in z[1])
    if len(re) != p.k or len(im) != p.k:
        raise ValueError("mixed word counts")
    a = LaneBatch(np.array(re).reshape(p.k, 1), device=p.device)
    b = LaneBatch(np.array(im).reshape(p.k, 1), device=p.device)
    yr, yi = eval_complex_batched(p, a, b, method, variant)
    return yr.lane(0), yi.lane(0)


def random_polynomial(n: int, seed: int, k: int, device=None) -> MWPolynomial:
    """poly.random_polynomial (181-192): degree-n, U[-1, 1] base-float
    coefficients promoted exactly to K words, leading one nonzero."""
    if n < 0:
        raise ValueError("degree must be >= 0")
    rng = np.random.Generator(np.random.PCG64(seed))
    c0 = rng.uniform(-1.0, 1.0, n + 1)
    while c0[n] == 0.0:
        c0[n] = rng.uniform(-1.0, 1.0)
    arr = np.zeros((k, n + 1))
    arr[0] = c0
    if k not in BITS:
        raise ValueError(f"unsupported word count {k}")
    return MWPolynomial(arr, device=device)
