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


_WS: dict = {}


def _workspace(device, n: int, stream: int | None = None) -> torch.Tensor:
    """Zero-initialised dot workspace, cached per (device, stream) and grown
    on demand (the single-launch dot re-arms its ticket itself).  Calls on
    one stream are serialised, so reuse is safe."""
    key = (str(device), _lib.stream_handle(device) if stream is None else stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < max(n, 1):
        ws = torch.zeros(max(n, 1), dtype=torch.float64, device=device)
        _WS[key] = ws
    return ws


def dot_tensor(x: LaneBatch, y: LaneBatch, variant: Variant = Variant.BRANCH_FREE, order: str = "tree",
               out: torch.Tensor | None = None, tuning=None) -> torch.Tensor:
    """dot(x, y) as a (K,) device tensor (no host synchronisation)."""
    _check_pair(x, y)
    o = _order(order)
    v = variant_code(variant)
    _lib.require_cuda(x.planes, y.planes)
    k, n = x.k, x.width
    lib = _lib.load()
    if out is None:
        out = torch.empty(k, dtype=torch.float64, device=x.device)
    wsn = lib.mw_dot_workspace(k, n) if o == _lib.ORDER_TREE else 0
    st = _lib.stream_handle(x.device)
    ws = _workspace(x.device, wsn, st)
    rc = lib.mw_dot_ex(k, v, x.planes.data_ptr(), n, y.planes.data_ptr(), n, n, ws.data_ptr(), out.data_ptr(), o,
                       _lib.tuning_ptr(tuning), st)
    _lib.check(rc, "mw_dot")
    return out


def dot(x: LaneBatch, y: LaneBatch, variant: Variant = Variant.BRANCH_FREE, order: str = "tree",
        tuning=None) -> tuple:
    """dot(x, y) as a K-word tuple."""
    return tuple(float(c) for c in dot_tensor(x, y, variant, order, tuning=tuning).cpu())


def axpy_(alpha, x: LaneBatch, y: LaneBatch, variant: Variant = Variant.BRANCH_FREE) -> LaneBatch:
    """y <- alpha x + y in place; alpha is a K-word tuple."""
    _check_pair(x, y)
    alpha = tuple(float(a) for a in getattr(alpha, "comps", alpha))
    if len(alpha) != x.k:
        raise ValueError("mixed word counts")
    _lib.require_cuda(x.planes, y.planes)
    import ctypes

    al = (ctypes.c_double * x.k)(*alpha)
    n = x.width
    rc = _lib.load().mw_axpy(x.k, variant_code(variant), ctypes.cast(al, ctypes.c_void_p), x.planes.data_ptr(), n,
                             y.planes.data_ptr(), n, n, _lib.stream_handle(x.device))
    _lib.check(rc, "mw_axpy")
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
    o = _order(order)
    _lib.require_cuda(a.planes, x.planes)
    k, m, n = a.k, a.rows, a.cols
    row1 = m if row1 is None else row1
    rows = row1 - row0
    if out is None:
        out = torch.empty((k, rows), dtype=torch.float64, device=a.device)
    es = a.planes.element_size()
    rc = _lib.load().mw_gemv(k, variant_code(variant), a.planes.data_ptr() + row0 * n * es, n, m * n,
                             x.planes.data_ptr(), n, out.data_ptr(), out.shape[1], rows, n, o,
                             _lib.stream_handle(a.device))
    _lib.check(rc, "mw_gemv")
    return LaneBatch(out)
