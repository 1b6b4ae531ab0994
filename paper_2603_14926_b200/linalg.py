"""Dense K-word matrices and the matrix product on the GPU.

Drop-in for the matmul path of mwfloat.linalg (pkg/src/mwfloat/linalg.py):
``MWMatrix`` (92-158) holds K planes of a rows x cols row-major matrix as
one (K, rows, cols) float64 CUDA tensor; ``MatMulPlan`` (75-89) and
``matmul`` (549-569) keep their signatures and ``ValueError`` checks.

``matmul`` runs mw_gemm: every C_ij folds t ascending from an exact zero
(the naive order, 284-314), bit-exact with ``scheme="naive"`` and
``"blocked"`` (identical order, 317-349).  ``scheme="strassen"`` is
computed in that same naive order -- more accurate than Strassen and
within the reference's own Strassen-vs-naive tolerance (8 ulp at the
|A||B| scale, verify.py:384-424); ``simd`` / ``threads`` /
``strassen_cutoff`` are accepted and validated but do not change the
device schedule (results are invariant to them in the reference too,
test_linalg.py:134-151).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .batch import LaneBatch, as_planes
from .multiword import BITS, Variant, variant_code

__all__ = ["Scheme", "MatMulPlan", "MWMatrix", "matmul", "gemv"]


class Scheme(enum.Enum):
    NAIVE = "naive"
    BLOCKED = "blocked"
    STRASSEN = "strassen"

    @classmethod
    def parse(cls, name) -> "Scheme":
        if isinstance(name, cls):
            return name
        key = str(getattr(name, "value", name)).lower()
        for s in cls:
            if s.value == key or s.name.lower() == key:
                return s
        raise ValueError(f"unknown scheme {name!r}")


@dataclass(frozen=True)
class MatMulPlan:
    scheme: Scheme = Scheme.STRASSEN
    variant: Variant = Variant.STANDARD
    simd: bool = True
    threads: int = 1
    strassen_cutoff: int = 32

    def __post_init__(self):
        object.__setattr__(self, "scheme", Scheme.parse(self.scheme))
        object.__setattr__(self, "variant", Variant.parse(self.variant))
        if self.strassen_cutoff < 2:
            raise ValueError("strassen_cutoff must be >= 2")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")


class MWMatrix:
    """Dense rows x cols matrix of K-word values, component-planar."""

    __slots__ = ("planes",)

    def __init__(self, comps, rows: int | None = None, cols: int | None = None, device=None):
        self.planes = as_planes(comps, 2, device)
        if rows is not None and (rows, cols) != tuple(self.planes.shape[1:]):
            raise ValueError("shape mismatch")

    @property
    def comps(self) -> tuple:
        return tuple(self.planes[c] for c in range(self.k))

    @property
    def k(self) -> int:
        return self.planes.shape[0]

    @property
    def rows(self) -> int:
        return self.planes.shape[1]

    @property
    def cols(self) -> int:
        return self.planes.shape[2]

    @property
    def device(self) -> torch.device:
        return self.planes.device

    @classmethod
    def zeros(cls, rows: int, cols: int, k: int, device=None) -> "MWMatrix":
        if k not in BITS:
            raise ValueError(f"unsupported word count {k}")
        return cls(np.zeros((k, rows, cols)), device=device)

    @classmethod
    def identity(cls, n: int, k: int, device=None) -> "MWMatrix":
        if k not in BITS:
            raise ValueError(f"unsupported word count {k}")
        a = np.zeros((k, n, n))
        a[0] = np.eye(n)
        return cls(a, device=device)

    def entry_components(self, i: int, j: int) -> tuple:
        return tuple(float(v) for v in self.planes[:, i, j].cpu())

    def numpy(self) -> np.ndarray:
        return self.planes.cpu().numpy()

    def bitwise_equal(self, other: "MWMatrix") -> bool:
        if self.k != other.k or self.planes.shape != other.planes.shape:
            return False
        a = self.planes.contiguous().view(torch.int64)
        b = other.planes.to(self.device).contiguous().view(torch.int64)
        return bool(torch.equal(a, b))

    def __repr__(self):
        return f"MWMatrix(k={self.k}, rows={self.rows}, cols={self.cols}, device={self.device})"


def gemm_into(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, variant, row0: int = 0,
              row1: int | None = None) -> None:
    """C[row0:row1] = A[row0:row1] B on the planes tensors (K, m, kd),
    (K, kd, n), (K, m, n) -- the row-block form the multi-GPU path shards."""
    k, m, kd = a.shape
    n = b.shape[2]
    row1 = m if row1 is None else row1
    rows = row1 - row0
    if rows <= 0:
        return
    _lib.require_cuda(a, b, c)
    lib = _lib.load()
    es = a.element_size()
    rc = lib.mw_gemm(
        k, variant_code(variant),
        a.data_ptr() + row0 * kd * es, kd, m * kd,
        b.data_ptr(), n, kd * n,
        c.data_ptr() + row0 * n * es, n, m * n,
        rows, n, kd, _lib.stream_handle(a.device),
    )
    _lib.check(rc, "mw_gemm")


def matmul(a: MWMatrix, b: MWMatrix, plan: MatMulPlan | None = None) -> MWMatrix:
    """Real multi-word product a @ b (linalg.py:549-569)."""
    if plan is None:
        plan = MatMulPlan()
    if a.cols != b.rows:
        raise ValueError(f"shape mismatch: {a.rows}x{a.cols} @ {b.rows}x{b.cols}")
    if a.k != b.k:
        raise ValueError("mixed word counts")
    if plan.scheme is Scheme.STRASSEN and (a.rows != a.cols or b.rows != b.cols):
        raise ValueError("strassen scheme requires square matrices")
    _lib.require_cuda(a.planes, b.planes)
    out = torch.empty((a.k, a.rows, b.cols), dtype=torch.float64, device=a.device)
    gemm_into(a.planes, b.planes, out, plan.variant)
    return MWMatrix(out)


def gemv(a: MWMatrix, x: LaneBatch, variant: Variant = Variant.BRANCH_FREE, order: str = "tree") -> LaneBatch:
    """y = A x (see blas.gemv)."""
    from .blas import gemv as _gemv

    return _gemv(a, x, variant, order)
