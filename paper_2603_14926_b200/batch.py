"""Lane-batched (structure-of-arrays) K-word arithmetic on the GPU.

Drop-in for mwfloat.batch (pkg/src/mwfloat/batch.py): a ``LaneBatch`` keeps
W values of a K-word type as K contiguous float64 planes -- here one
(K, W) torch tensor resident in HBM, so plane c is ``planes[c]`` and a
warp's loads of consecutive lanes are coalesced 128-bit transactions.
``batch_add / batch_mul / batch_div`` keep the reference signatures,
validation (``ValueError`` for mixed K or width, batch.py:197-201) and
results (bit-exact per lane), and run one CUDA kernel each through the
C-ABI (mw_ew_*).  ``batch_sub`` is the reference's add-of-negation
(multiword.py:629-630) fused into one kernel.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .multiword import BITS, Variant, variant_code

__all__ = [
    "LaneBatch",
    "pack",
    "unpack",
    "batch_add",
    "batch_sub",
    "batch_mul",
    "batch_div",
    "default_lane_width",
    "LANE_WIDTHS",
    "as_planes",
]

LANE_WIDTHS = (2, 4, 8)


def default_lane_width() -> int:
    """Kept for API parity (batch.py:54-58).  On the GPU a batch is one
    array of any width; this is only a packing granularity."""
    return 4


def _default_device() -> torch.device:
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


def as_planes(comps, ndim: int, device=None) -> torch.Tensor:
    """Convert a tuple of K equally shaped arrays/tensors, or one (K, ...)
    array/tensor, to a contiguous float64 (K, ...) tensor on ``device``."""
    dev = torch.device(device) if device is not None else None
    if isinstance(comps, torch.Tensor):
        t = comps
    elif isinstance(comps, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(comps, dtype=np.float64))
    else:
        parts = list(comps)
        if len(parts) not in BITS:
            raise ValueError(f"unsupported word count {len(parts)}")
        ts = []
        for p in parts:
            if isinstance(p, torch.Tensor):
                ts.append(p)
            else:
                ts.append(torch.from_numpy(np.ascontiguousarray(p, dtype=np.float64)))
        shape = ts[0].shape
        for p in ts:
            if p.dim() != ndim or p.shape != shape:
                raise ValueError(f"component arrays must be equal-shape {ndim}-D")
        if dev is None:
            dev = ts[0].device if ts[0].is_cuda else _default_device()
        t = torch.stack([p.to(device=dev, dtype=torch.float64) for p in ts])
    if t.dim() != ndim + 1:
        raise ValueError(f"component arrays must be {ndim}-D")
    if t.shape[0] not in BITS:
        raise ValueError(f"unsupported word count {t.shape[0]}")
    if dev is None:
        dev = t.device if t.is_cuda else _default_device()
    return t.to(device=dev, dtype=torch.float64).contiguous()


def coefficient_planes(values, k: int | None = None) -> np.ndarray:
    """(K, n) float64 planes from a list of K-word values -- tuples / lists,
    objects with ``.comps``, or bare floats (which need ``k``: the value
    becomes (x, 0, ..., 0)) -- in list order (coefficient i at column i)."""
    def words(v):
        if hasattr(v, "comps"):
            return tuple(v.comps)
        if isinstance(v, (tuple, list)):
            return tuple(v)
        if k is None:
            raise ValueError("k required for bare float coefficients")
        return (float(v),) + (0.0,) * (k - 1)

    cols = [words(v) for v in values]
    return np.array(cols, dtype=np.float64).T.copy()


class LaneBatch:
    """W K-word values in component-planar layout (batch.py:61-93).

    ``planes[c, lane]`` is component c of ``lane``; ``comps`` gives the K
    planes as a tuple like the reference; ``count`` is how many leading
    lanes carry packed values (the rest are zero padding).
    """

    __slots__ = ("planes", "count")

    def __init__(self, comps, count: int | None = None, device=None):
        self.planes = as_planes(comps, 1, device)
        self.count = self.width if count is None else int(count)

    @classmethod
    def _wrap(cls, planes: torch.Tensor, count: int) -> "LaneBatch":
        """A batch around planes a kernel just wrote (contiguous float64
        (K, W) on the device): no conversion on the host path."""
        b = object.__new__(cls)
        b.planes = planes
        b.count = count
        return b

    @property
    def comps(self) -> tuple:
        return tuple(self.planes[c] for c in range(self.k))

    @property
    def k(self) -> int:
        return self.planes.shape[0]

    @property
    def width(self) -> int:
        return self.planes.shape[1]

    @property
    def device(self) -> torch.device:
        return self.planes.device

    def lane(self, i: int) -> tuple:
        return tuple(float(v) for v in self.planes[:, i].cpu())

    def numpy(self) -> np.ndarray:
        return self.planes.cpu().numpy()

    def __repr__(self):
        return f"LaneBatch(k={self.k}, width={self.width}, count={self.count}, device={self.device})"


def pack(values, width: int | None = None, device=None) -> LaneBatch:
    """Pack K-word values (tuples or objects with ``.comps``) into a batch;
    tail lanes are zero padded (batch.py:96-112)."""
    words = [tuple(getattr(v, "comps", v)) for v in values]
    if len(words) == 0:
        raise ValueError("cannot pack an empty value list")
    if len({len(w) for w in words}) != 1:
        raise ValueError("mixed word counts in pack")
    lanes = len(words) if width is None else width
    if lanes < len(words):
        raise ValueError(f"width {lanes} below value count {len(words)}")
    arr = np.zeros((len(words[0]), lanes))
    arr[:, : len(words)] = np.array(words, dtype=np.float64).T
    return LaneBatch(arr, count=len(words), device=device)


def unpack(batch: LaneBatch) -> list:
    """The first ``count`` lanes as MultiWord values (batch.py:115-119)."""
    from .multiword import MultiWord

    arr = batch.numpy()
    return [MultiWord.from_components(tuple(float(c) for c in arr[:, i])) for i in range(batch.count)]


def _check_pair(a: LaneBatch, b: LaneBatch):
    if a.k != b.k:
        raise ValueError("mixed word counts")
    if a.width != b.width:
        raise ValueError("mixed lane widths")


_OPS = {"mw_ew_add": 0, "mw_ew_sub": 1, "mw_ew_mul": 2, "mw_ew_div": 3}


def _binary(fn_name: str, a: LaneBatch, b: LaneBatch, variant) -> LaneBatch:
    """One lane kernel through the extension (csrc/ext/mwext.cpp -> the
    C-ABI mw_ew_*): validation (K, then widths, as batch.py:197-201),
    device guard and stream in C++."""
    out = _lib.ext().ew(_OPS[fn_name], variant_code(variant), a.planes, b.planes)
    return LaneBatch._wrap(out, max(a.count, b.count))


def batch_add(a: LaneBatch, b: LaneBatch, variant: Variant = Variant.STANDARD) -> LaneBatch:
    return _binary("mw_ew_add", a, b, variant)


def batch_sub(a: LaneBatch, b: LaneBatch, variant: Variant = Variant.STANDARD) -> LaneBatch:
    return _binary("mw_ew_sub", a, b, variant)


def batch_mul(a: LaneBatch, b: LaneBatch, variant: Variant = Variant.STANDARD) -> LaneBatch:
    return _binary("mw_ew_mul", a, b, variant)


def batch_div(a: LaneBatch, b: LaneBatch, variant: Variant = Variant.STANDARD) -> LaneBatch:
    """Per-lane a / b by the shared Newton reciprocal sequence; zero lanes
    of b propagate inf/nan (batch.py:216-231)."""
    return _binary("mw_ew_div", a, b, variant)
