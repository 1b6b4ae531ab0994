"""Error-free transformations on binary64 (mwfloat.eft, eft.py:33-94).

``quick_two_sum``, ``two_sum`` and ``two_prod`` take floats, numpy arrays
or torch tensors and return the pair (rounded result, exact error); the
work runs in the device kernel mw_eft (explicitly rounded intrinsics, one
FMA in two_prod).  ``assert_rounding_mode`` checks round-to-nearest-even
on the device (the _rn intrinsics fix it per instruction).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

__all__ = ["fma", "quick_two_sum", "two_sum", "two_prod", "assert_rounding_mode"]


def _run(op: int, a, b):
    scalar = isinstance(a, (int, float)) and isinstance(b, (int, float))
    to_np = isinstance(a, np.ndarray) or isinstance(b, np.ndarray) or scalar
    ta = torch.as_tensor(np.asarray(a, dtype=np.float64) if not isinstance(a, torch.Tensor) else a,
                         dtype=torch.float64)
    tb = torch.as_tensor(np.asarray(b, dtype=np.float64) if not isinstance(b, torch.Tensor) else b,
                         dtype=torch.float64)
    ta, tb = torch.broadcast_tensors(ta, tb)
    dev = ta.device if ta.is_cuda else (tb.device if tb.is_cuda else torch.device("cuda"))
    ta = ta.to(dev).contiguous()
    tb = tb.to(dev).contiguous()
    _lib.require_cuda(ta, tb)
    s = torch.empty_like(ta)
    e = torch.empty_like(ta)
    rc = _lib.load().mw_eft(op, ta.data_ptr(), tb.data_ptr(), s.data_ptr(), e.data_ptr(), ta.numel(),
                            _lib.stream_handle(dev))
    _lib.check(rc, "mw_eft")
    if scalar:
        return float(s.item()), float(e.item())
    if to_np:
        return s.cpu().numpy(), e.cpu().numpy()
    return s, e


def fma(a, b, c):
    """Correctly rounded a*b + c, one rounding (eft.py:33-48): floats give a
    float, arrays an array of the broadcast shape; device kernel mw_fma."""
    scalar = all(isinstance(v, (int, float)) for v in (a, b, c))
    to_np = scalar or any(isinstance(v, np.ndarray) for v in (a, b, c))
    ts = [v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v, dtype=np.float64))
          for v in (a, b, c)]
    dev = next((t.device for t in ts if t.is_cuda), torch.device("cuda"))
    ts = [t.to(device=dev, dtype=torch.float64) for t in ts]
    shape = torch.broadcast_shapes(*(t.shape for t in ts))
    ta, tb, tc = (t.expand(shape).contiguous() for t in ts)
    _lib.require_cuda(ta, tb, tc)
    out = torch.empty_like(ta)
    rc = _lib.load().mw_fma(ta.data_ptr(), tb.data_ptr(), tc.data_ptr(), out.data_ptr(), ta.numel(),
                            _lib.stream_handle(dev))
    _lib.check(rc, "mw_fma")
    if scalar:
        return float(out.item())
    if to_np:
        return out.cpu().numpy()
    return out


def quick_two_sum(a, b):
    """(s, e), s = fl(a+b), a + b = s + e exactly; needs |a| >= |b|."""
    return _run(0, a, b)


def two_sum(a, b):
    """(s, e), s = fl(a+b), a + b = s + e exactly, any magnitudes."""
    return _run(1, a, b)


def two_prod(a, b):
    """(p, e), p = fl(a*b), a * b = p + e exactly (no overflow/underflow)."""
    return _run(2, a, b)


def assert_rounding_mode():
    """Round-to-nearest-ties-even on the device (eft.py:86-94)."""
    s, _ = two_sum(np.array([1.0, 1.0]), np.array([2.0**-53, 3.0 * 2.0**-54]))
    if s[0] != 1.0 or s[1] != 1.0 + 2.0**-52:
        raise RuntimeError("device FP arithmetic is not round-to-nearest-ties-even")
