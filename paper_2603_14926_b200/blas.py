"""dot, axpy and GEMV over K-word arrays on the GPU.

The reference has no functions by these names; SURVEY §8(a) defines them
from its primitives, and these definitions are what the kernels compute:

* ``dot(x, y)``  = fold_t add(acc, mul(x_t, y_t)) from an exact zero, t
  ascending -- the naive matmul fold for 1xn . nx1 (linalg.py:300-314).
  ``order="exact"`` replays that fold bit for bit (one GPU thread);
  ``order="tree"`` (default, the throughput path) folds 16-element leaf
  chunks in that order and combines the chunk partials by a fixed pairwise
  tree -- a function of n only, so the result is deterministic and
  independent of launch shape and GPU count; within n 2^-p+4 sum|x||y|.
* ``axpy(alpha, x, y)`` = batch_add(batch_mul(alpha, x), y)
  (batch.py:204-213), bit-exact.  Pure (returns a new batch) like the
  reference; ``axpy_`` updates y in place.
* ``gemv(A, x)`` = y_i folded like dot over row i; bit-exact with
  matmul(A, x as n x 1, naive) for ``order="exact"``; ``order="tree"``
  splits each row over 128 partials (four warps; partial u folds
  t = u, u+128, ...) combined by the pairwise tree.
"""

from __future__ import annotations

import torch

from . import _lib
from .batch import LaneBatch
from .linalg import MWMatrix
from .multiword import Variant, variant_code

__all__ = ["dot", "dot_tensor", "axpy", "axpy_", "gemv", "ORDERS"]

ORDERS = {"exact": _lib.ORDER_EXACT, "tree": _lib.ORDER_TREE}


def _order(order) -> int:
    if order not in ORDERS:
        raise ValueError(f"unknown order {order!r} (expected 'exact' or 'tree')")
    return ORDERS[order]


def _check_pair(x: LaneBatch, y: LaneBatch):
    if x.k != y.k:
        raise ValueError("mixed word counts")
    if x.width != y.width:
        raise ValueError("mixed lane widths")


def dot_tensor(x: LaneBatch, y: LaneBatch, variant: Variant = Variant.BRANCH_FREE, order: str = "tree",
               out: torch.Tensor | None = None, tuning=None) -> torch.Tensor:
    """dot(x, y) as a (K,) device tensor (no host synchronisation).  The
    tree order's workspace lives in the extension: one zeroed buffer per
    (device, stream) for eager calls, a private one per call captured into
    a CUDA graph (csrc/ext/mwext.cpp)."""
    return _lib.ext().dot(variant_code(variant), x.planes, y.planes, _order(order), out,
                          **_lib.tune_kw(tuning, "dot_cluster"))


def dot(x: LaneBatch, y: LaneBatch, variant: Variant = Variant.BRANCH_FREE, order: str = "tree",
        tuning=None) -> tuple:
    """dot(x, y) as a K-word tuple."""
    return tuple(float(c) for c in dot_tensor(x, y, variant, order, tuning=tuning).cpu())


def axpy_(alpha, x: LaneBatch, y: LaneBatch, variant: Variant = Variant.BRANCH_FREE) -> LaneBatch:
    """y <- alpha x + y in place; alpha is a K-word tuple.  (K, widths and
    devices are checked by the extension: ValueError on a mismatch.)"""
    words = getattr(alpha, "comps", alpha)
    if not isinstance(words, (tuple, list)):  # numpy / torch vectors of K words
        words = [float(v) for v in words]
    _lib.ext().axpy_(variant_code(variant), words, x.planes, y.planes)
    y.count = max(x.count, y.count)
    return y


def axpy(alpha, x: LaneBatch, y: LaneBatch, variant: Variant = Variant.BRANCH_FREE) -> LaneBatch:
    """alpha x + y as a new batch (inputs untouched)."""
    _check_pair(x, y)
    out = LaneBatch(y.planes.clone(), count=y.count)
    return axpy_(alpha, x, out, variant)


def gemv(a: MWMatrix, x: LaneBatch, variant: Variant = Variant.BRANCH_FREE, order: str = "tree",
         row0: int = 0, row1: int | None = None, out: torch.Tensor | None = None) -> LaneBatch:
    """y = A x for rows [row0, row1) (all rows by default)."""
    if a.k != x.k:
        raise ValueError("mixed word counts")
    if a.cols != x.width:
        raise ValueError(f"shape mismatch: {a.rows}x{a.cols} @ {x.width}")
    out = _lib.ext().gemv(variant_code(variant), a.planes, x.planes, row0, a.rows if row1 is None else row1,
                          _order(order), out)
    return LaneBatch(out)
