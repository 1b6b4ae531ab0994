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

__all__ = ["Scheme", "MatMulPlan", "MWMatrix", "CMWMatrix", "matmul", "cmatmul", "gemv",
           "gen_complex_test_matrices"]


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


class CMWMatrix:
    """Complex matrix as a (re, im) pair of equally shaped MWMatrix
    (linalg.py:161-193)."""

    __slots__ = ("re", "im")

    def __init__(self, re: MWMatrix, im: MWMatrix):
        if (re.rows, re.cols, re.k) != (im.rows, im.cols, im.k):
            raise ValueError("re/im shape mismatch")
        self.re = re
        self.im = im

    @property
    def rows(self):
        return self.re.rows

    @property
    def cols(self):
        return self.re.cols

    @property
    def k(self):
        return self.re.k

    def bitwise_equal(self, other: "CMWMatrix") -> bool:
        return self.re.bitwise_equal(other.re) and self.im.bitwise_equal(other.im)

    def __repr__(self):
        return f"CMWMatrix(k={self.k}, rows={self.rows}, cols={self.cols})"


def gen_complex_test_matrices(n: int, seed: int, k: int, device=None):
    """The reference's random complex pair (linalg.py:247-276): per matrix
    u1, u2 ~ U[0,1) (n^2 each) for Box-Muller normals r = sqrt(-2 ln(1-u1))
    (cos, sin)(2 pi u2), then U[0,1) factors for re and im; entries
    exp(r) (u - 1/2) promoted exactly to K words.  Host numpy, seeded
    PCG64, identical draws to the reference."""
    if n < 1:
        raise ValueError("n must be >= 1")
    rng = np.random.Generator(np.random.PCG64(seed))

    def one_matrix():
        u1 = rng.random((n, n))
        u2 = rng.random((n, n))
        radial = np.sqrt(-2.0 * np.log1p(-u1))
        rn_re = radial * np.cos(2.0 * np.pi * u2)
        rn_im = radial * np.sin(2.0 * np.pi * u2)
        ure = rng.random((n, n))
        uim = rng.random((n, n))
        re0 = np.exp(rn_re) * (ure - 0.5)
        im0 = np.exp(rn_im) * (uim - 0.5)
        re = np.zeros((k, n, n))
        im = np.zeros((k, n, n))
        re[0] = re0
        im[0] = im0
        return CMWMatrix(MWMatrix(re, device=device), MWMatrix(im, device=device))

    return one_matrix(), one_matrix()


def _ew(name: str, a: torch.Tensor, b: torch.Tensor, variant) -> torch.Tensor:
    """Lane-wise K-word op over two equally shaped planes tensors."""
    k = a.shape[0]
    n = a[0].numel()
    out = torch.empty_like(a)
    rc = getattr(_lib.load(), name)(k, variant_code(variant), a.data_ptr(), n, b.data_ptr(), n, out.data_ptr(), n, n,
                                    _lib.stream_handle(a.device))
    _lib.check(rc, name)
    return out


def cmatmul(a: CMWMatrix, b: CMWMatrix, plan: MatMulPlan | None = None) -> CMWMatrix:
    """Complex product via three real multiplications (linalg.py:572-590):
    P1 = Re(a) Re(b), P2 = Im(a) Im(b), P3 = (Re+Im)(a) (Re+Im)(b);
    Re = P1 - P2, Im = (P3 - P1) - P2 -- the same kernels and order as the
    reference, so bit-exact with cmatmul(..., naive)."""
    if plan is None:
        plan = MatMulPlan()
    if a.cols != b.rows:
        raise ValueError("shape mismatch")
    if a.k != b.k:
        raise ValueError("mixed word counts")
    v = plan.variant
    _lib.require_cuda(a.re.planes, b.re.planes)
    sum_a = MWMatrix(_ew("mw_ew_add", a.re.planes, a.im.planes, v))
    sum_b = MWMatrix(_ew("mw_ew_add", b.re.planes, b.im.planes, v))
    p1 = matmul(a.re, b.re, plan).planes
    p2 = matmul(a.im, b.im, plan).planes
    p3 = matmul(sum_a, sum_b, plan).planes
    re = _ew("mw_ew_sub", p1, p2, v)
    im = _ew("mw_ew_sub", _ew("mw_ew_sub", p3, p1, v), p2, v)
    return CMWMatrix(MWMatrix(re), MWMatrix(im))


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
