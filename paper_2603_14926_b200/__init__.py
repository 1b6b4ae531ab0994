"""mwgpu: branch-free DD/TD/QD arithmetic and its data-parallel kernels on
B200 (sm_100a), behind the array-level API of the reference mwfloat package
(pkg/src/mwfloat: batch, linalg, poly, roots).

Layers: ``csrc/mw_eft.cuh`` (EFTs + BF kernels as inlined device functions)
-> ``csrc/*.cu`` (kernels) -> ``include/mwgpu.h`` C-ABI (``libmwgpu.so``)
-> ctypes (``_lib``) -> this package.  No CPU fallback: operations raise if
the native library or a CUDA device is missing.
"""

from . import _lib
from .eft import assert_rounding_mode, quick_two_sum, two_prod, two_sum
from .batch import LaneBatch, batch_add, batch_div, batch_mul, batch_sub, pack, unpack
from .blas import axpy, axpy_, dot, dot_tensor, gemv
from .linalg import CMWMatrix, MatMulPlan, MWMatrix, Scheme, cmatmul, gen_complex_test_matrices, matmul
from .multiword import BITS, DD, QD, TD, MultiWord, Variant, ulp_k
from .poly import (
    MWPolynomial,
    estrin_eval,
    estrin_eval_batched,
    eval_complex,
    eval_complex_batched,
    horner_eval,
    horner_eval_batched,
    random_polynomial,
)
from .roots import (
    DKSweepGraph,
    CollisionError,
    MonicPoly,
    NoConvergence,
    RootState,
    aberth_init,
    default_tolerance,
    dk_iterate,
    dk_solve,
    dk_sweeps,
    radius_estimate,
    chebyshev_coeffs,
    residual_check,
)

__version__ = "0.1.0"

__all__ = [
    "quick_two_sum", "two_sum", "two_prod", "assert_rounding_mode",
    "LaneBatch", "pack", "unpack", "batch_add", "batch_sub", "batch_mul", "batch_div",
    "dot", "dot_tensor", "axpy", "axpy_", "gemv",
    "MatMulPlan", "MWMatrix", "CMWMatrix", "Scheme", "matmul", "cmatmul", "gen_complex_test_matrices",
    "BITS", "Variant", "ulp_k", "MultiWord", "DD", "TD", "QD",
    "MWPolynomial", "horner_eval", "horner_eval_batched", "estrin_eval", "estrin_eval_batched",
    "eval_complex", "eval_complex_batched", "random_polynomial",
    "MonicPoly", "RootState", "CollisionError", "NoConvergence", "aberth_init", "radius_estimate",
    "default_tolerance", "dk_iterate", "dk_sweeps", "dk_solve", "DKSweepGraph", "chebyshev_coeffs",
    "residual_check",
]
