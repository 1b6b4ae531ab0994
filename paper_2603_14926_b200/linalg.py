"""Dense K-word matrices and the matrix product on the GPU.

Drop-in for the matmul path of mwfloat.linalg (pkg/src/mwfloat/linalg.py):
``MWMatrix`` (92-158) holds K planes of a rows x cols row-major matrix as
one (K, rows, cols) float64 CUDA tensor; ``MatMulPlan`` (75-89) and
``matmul`` (549-569) keep their signatures and ``ValueError`` checks.

``matmul`` runs mw_gemm: every C_ij folds t ascending from an exact zero
(the naive order, 284-314), bit-exact with ``scheme="naive"`` and
``"blocked"`` (identical order, 317-349).  ``scheme="strassen"`` runs the
reference's Strassen recursion (390-546: seven products per even split,
odd sizes peeled, blocked products at or below ``strassen_cutoff``)
breadth-first: each recursion level is a handful of lane-wise kernels over
all 7^L sub-problems at once and the leaves are ONE batched GEMM launch
(mw_gemm_batched) -- bit-exact with the reference's Strassen.  ``simd``
and ``threads`` are accepted and validated but do not change the device
schedule (results are invariant to them in the reference too,
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

__all__ = ["Scheme", "MatMulPlan", "MWMatrix", "CMWMatrix", "matmul", "cmatmul", "gemv", "strassen_pad_policy",
           "gen_complex_test_matrices", "gen_test_matrices", "sqrt_constant"]


class Scheme(enum.Enum):
    """Product scheme (linalg.py:59-72): the naive t-ascending fold, the
    blocked form of the same fold, or Strassen's recursion."""

    NAIVE = "naive"
    BLOCKED = "blocked"
    STRASSEN = "strassen"

    @classmethod
    def parse(cls, name) -> "Scheme":
        """A Scheme, its value or name (any case), or the reference's own
        enum member."""
        if isinstance(name, cls):
            return name
        wanted = str(getattr(name, "value", name)).lower()
        found = {m.value: m for m in cls} | {m.name.lower(): m for m in cls}
        if wanted not in found:
            raise ValueError(f"unknown scheme {name!r}")
        return found[wanted]


@dataclass(frozen=True)
class MatMulPlan:
    """How ``matmul`` multiplies (linalg.py:75-89): scheme, kernel variant,
    and the reference's ``simd`` / ``threads`` / ``strassen_cutoff`` knobs
    (accepted and validated; the device kernels need no threads, and
    results never depend on them)."""

    scheme: Scheme = Scheme.STRASSEN
    variant: Variant = Variant.STANDARD
    simd: bool = True
    threads: int = 1
    strassen_cutoff: int = 32

    def __post_init__(self):
        for field, parse in (("scheme", Scheme.parse), ("variant", Variant.parse)):
            object.__setattr__(self, field, parse(getattr(self, field)))
        checks = (("strassen_cutoff", 2), ("threads", 1))
        for field, least in checks:
            if getattr(self, field) < least:
                raise ValueError(f"{field} must be >= {least}")


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
    """Complex matrix: real and imaginary parts as two MWMatrix of one
    shape and word count (linalg.py:161-193)."""

    __slots__ = ("re", "im")

    def __init__(self, re: MWMatrix, im: MWMatrix):
        same = re.rows == im.rows and re.cols == im.cols and re.k == im.k
        if not same:
            raise ValueError("re/im shape mismatch")
        self.re, self.im = re, im

    rows = property(lambda self: self.re.rows)
    cols = property(lambda self: self.re.cols)
    k = property(lambda self: self.re.k)

    def bitwise_equal(self, other: "CMWMatrix") -> bool:
        return self.re.bitwise_equal(other.re) and self.im.bitwise_equal(other.im)

    def __repr__(self):
        return f"CMWMatrix(k={self.k}, rows={self.rows}, cols={self.cols})"


def sqrt_constant(value: int, k: int) -> tuple:
    """K-word rounding of sqrt(value) (linalg.sqrt_constant, 217-221): the
    reference rounds its 300-bit oracle root; here mpmath at 400 bits, both
    by greedy nearest-double extraction."""
    import mpmath
    from fractions import Fraction

    from .multiword import from_fraction

    mpmath.mp.prec = 400
    sign, man, exp, _ = mpmath.sqrt(mpmath.mpf(value))._mpf_
    fr = Fraction(int(man)) * (Fraction(2) ** int(exp))
    return from_fraction(-fr if sign else fr, k)


def gen_test_matrices(n: int, k: int, device=None):
    """The paper's accuracy-benchmark pair (linalg.py:224-244):
    a_ij = sqrt(5) (i+j-1), b_ij = sqrt(3) (n-i+1), 1-based; each entry the
    K-word Standard product of the rounded constant with the exact integer
    factor, computed on the device (batch_mul STANDARD)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    from .batch import LaneBatch, batch_mul

    i_idx = np.arange(1, n + 1).reshape(n, 1)
    j_idx = np.arange(1, n + 1).reshape(1, n)
    fac_a = (i_idx + j_idx - 1).astype(np.float64)
    fac_b = np.broadcast_to((n - i_idx + 1).astype(np.float64), (n, n)).copy()
    out = []
    for const, fac in ((sqrt_constant(5, k), fac_a), (sqrt_constant(3, k), fac_b)):
        cst = np.zeros((k, n * n))
        f = np.zeros((k, n * n))
        for c in range(k):
            cst[c] = const[c]
        f[0] = fac.ravel()
        prod = batch_mul(LaneBatch(cst, device=device), LaneBatch(f, device=device), Variant.STANDARD)
        out.append(MWMatrix(prod.planes.reshape(k, n, n)))
    return out[0], out[1]


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
              row1: int | None = None, tuning=None) -> None:
    """C[row0:row1] = A[row0:row1] B on the planes tensors (K, m, kd),
    (K, kd, n), (K, m, n) -- the row-block form the multi-GPU path shards.
    ``tuning``: an optional _lib.Tuning (launch shape only; same bits)."""
    # validation (shapes, K, float64, contiguity, one device), the device
    # guard and torch's current stream are in the extension
    _lib.ext().gemm(variant_code(variant), a, b, c, row0, -1 if row1 is None else row1,
                    **_lib.tune_kw(tuning, "gemm_tile"))


def _ew_planes(name: str, a: torch.Tensor, b: torch.Tensor, variant) -> torch.Tensor:
    """Lane-wise op over (K, ...) tensors whose non-plane dims are
    contiguous (any plane stride); returns a contiguous result."""
    for t in (a, b):
        inner = t[0]
        if not inner.is_contiguous():
            raise ValueError("operand planes must be contiguous")
    k = a.shape[0]
    n = a[0].numel()
    out = torch.empty(a.shape, dtype=torch.float64, device=a.device)
    rc = getattr(_lib.load(), name)(k, variant_code(variant), a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0),
                                    out.data_ptr(), n, n, _lib.stream_handle(a.device))
    _lib.check(rc, name)
    return out


def _gemm4(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, variant, cin: torch.Tensor | None = None):
    """Batched C = Cin + A B on (K, batch, rows, cols) views (unit column
    stride); strides are passed through, no copies."""
    k, bt, m, kd = a.shape
    n = b.shape[3]
    for t in (a, b, c) + ((cin,) if cin is not None else ()):
        if t.shape[3] > 1 and t.stride(3) != 1:
            raise ValueError("matrix views need unit column stride")
    rc = _lib.load().mw_gemm_batched(
        k, variant_code(variant),
        a.data_ptr(), max(a.stride(2), kd), a.stride(0), a.stride(1),
        b.data_ptr(), max(b.stride(2), n), b.stride(0), b.stride(1),
        c.data_ptr(), max(c.stride(2), n), c.stride(0), c.stride(1),
        None if cin is None else cin.data_ptr(), 0 if cin is None else max(cin.stride(2), n),
        0 if cin is None else cin.stride(0), 0 if cin is None else cin.stride(1),
        m, n, kd, bt, _lib.stream_handle(a.device),
    )
    _lib.check(rc, "mw_gemm_batched")


def strassen_pad_policy(n: int, cutoff: int = 32) -> list:
    """The decomposition Strassen applies to an n x n product, top down
    (linalg.py:390-406): ("split", m) halves an even m, ("peel", m) strips
    the last row/column of an odd m, ("blocked", m) is a leaf at m <= cutoff."""
    out = []
    m = int(n)
    while m > cutoff:
        odd = m & 1
        out.append(("peel" if odd else "split", m))
        m = m - 1 if odd else m >> 1
    out.append(("blocked", m))
    return out


def _strassen_rec(a: torch.Tensor, b: torch.Tensor, variant, cutoff: int) -> torch.Tensor:
    """Batched Strassen on contiguous (K, batch, s, s) operands
    (linalg._strassen_rec, linalg.py:503-511)."""
    k, bt, s, _ = a.shape
    if s <= cutoff:
        c = torch.empty_like(a)
        _gemm4(a, b, c, variant)  # _blocked_mm: the naive per-entry order
        return c
    if s % 2:
        return _strassen_peel(a, b, variant, cutoff)
    h = s // 2

    def q(t, i, j):
        return t[:, :, i * h:(i + 1) * h, j * h:(j + 1) * h].contiguous()

    def add(x, y):
        return _ew_planes("mw_ew_add", x, y, variant)

    def sub(x, y):
        return _ew_planes("mw_ew_sub", x, y, variant)

    a11, a12, a21, a22 = q(a, 0, 0), q(a, 0, 1), q(a, 1, 0), q(a, 1, 1)
    b11, b12, b21, b22 = q(b, 0, 0), q(b, 0, 1), q(b, 1, 0), q(b, 1, 1)
    # _strassen_products (linalg.py:418-436), in its order M1..M7
    x = torch.stack([add(a11, a22), add(a21, a22), a11, a22, add(a11, a12), sub(a21, a11), sub(a12, a22)], dim=1)
    y = torch.stack([add(b11, b22), b11, sub(b12, b22), sub(b21, b11), b22, add(b11, b12), add(b21, b22)], dim=1)
    m = _strassen_rec(x.reshape(k, 7 * bt, h, h), y.reshape(k, 7 * bt, h, h), variant, cutoff)
    m = m.reshape(k, 7, bt, h, h)
    m1, m2, m3, m4, m5, m6, m7 = (m[:, i] for i in range(7))
    # _strassen_combine (linalg.py:439-452)
    out = torch.empty((k, bt, s, s), dtype=torch.float64, device=a.device)
    out[:, :, :h, :h] = add(sub(add(m1, m4), m5), m7)
    out[:, :, :h, h:] = add(m3, m5)
    out[:, :, h:, :h] = add(m2, m4)
    out[:, :, h:, h:] = add(add(sub(m1, m2), m3), m6)
    return out


def _strassen_peel(a: torch.Tensor, b: torch.Tensor, variant, cutoff: int) -> torch.Tensor:
    """Odd size: recurse on the even core, then the border folds
    (linalg._strassen_peel, linalg.py:455-500), each a GEMM whose fold
    starts from the reference's initial term."""
    k, bt, n, _ = a.shape
    e = n - 1
    core = _strassen_rec(a[:, :, :e, :e].contiguous(), b[:, :, :e, :e].contiguous(), variant, cutoff)
    out = torch.empty_like(a)
    a_col, a_row, a_cor = a[:, :, :e, e:e + 1], a[:, :, e:e + 1, :e], a[:, :, e:e + 1, e:e + 1]
    b_col, b_row, b_cor = b[:, :, :e, e:e + 1], b[:, :, e:e + 1, :e], b[:, :, e:e + 1, e:e + 1]

    def mul(x, y):
        return _ew_planes("mw_ew_mul", x.contiguous(), y.contiguous(), variant)

    # C00 = core + a_col (outer) b_row: rows fold add(core, mul(a_col_i, b_row))
    _gemm4(a_col, b_row, out[:, :, :e, :e], variant, cin=core)
    # C01 = mul(a_col, b_cor) + sum_t mul(A[:, t], b_col[t])
    init = mul(a_col, b_cor.expand(k, bt, e, 1))
    _gemm4(a[:, :, :e, :e], b_col, out[:, :, :e, e:e + 1], variant, cin=init)
    # C10 = mul(a_cor, b_row) + sum_t mul(a_row[t], B[t, :])
    init = mul(a_cor.expand(k, bt, 1, e), b_row)
    _gemm4(a_row, b[:, :, :e, :e], out[:, :, e:e + 1, :e], variant, cin=init)
    # C11 = mul(a_cor, b_cor) + sum_t mul(a_row[t], b_col[t])
    init = mul(a_cor, b_cor)
    _gemm4(a_row, b_col, out[:, :, e:e + 1, e:e + 1], variant, cin=init)
    return out


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
    if plan.scheme is Scheme.STRASSEN:
        k, n = a.k, a.rows
        c = _strassen_rec(a.planes.reshape(k, 1, n, n), b.planes.reshape(k, 1, n, n), plan.variant,
                          plan.strassen_cutoff)
        return MWMatrix(c.reshape(k, n, n))
    out = torch.empty((a.k, a.rows, b.cols), dtype=torch.float64, device=a.device)
    gemm_into(a.planes, b.planes, out, plan.variant)
    return MWMatrix(out)


def gemv(a: MWMatrix, x: LaneBatch, variant: Variant = Variant.BRANCH_FREE, order: str = "tree") -> LaneBatch:
    """y = A x (see blas.gemv)."""
    from .blas import gemv as _gemv

    return _gemv(a, x, variant, order)
