"""The reference-side binding: ``mwfloat`` (the reference package) calling
``libmwgpu.so`` through its C-ABI (``include/mwgpu.h``) with ctypes.

This is the module a maintainer would add to the reference as
``mwfloat/_gpu.py``.  ``install()`` rebinds the
reference's own dispatch points -- nothing else in the reference changes:

* ``batch._BATCH_ADD`` / ``batch._BATCH_MUL`` (``batch.py:178-194``), all six
  ``(K, Variant)`` entries -> ``mw_ew_add`` / ``mw_ew_mul``.  Every caller of
  the tables goes through them: ``batch_add/mul/div`` (``batch.py:204-231``),
  ``linalg._ew_*`` (``linalg.py:196-205``, hence the blocked and Strassen
  schemes and ``cmatmul``), ``poly.estrin_eval_batched`` (``poly.py:133``),
  ``roots.aberth_init`` / ``dk_iterate`` (``roots.py:196, 249``).
* ``linalg._naive_mm`` (``linalg.py:368-375``) -> ``mw_gemm``.

Operands cross the boundary as numpy component tuples (the reference's own
SoA layout): they are stacked into one (K, n) float64 array, copied to the
device, computed with torch's current stream, and copied back.  Lanes are
bit-exact with the reference kernels, so the reference's own tests pass
unchanged (``tests/test_reference_binding.py`` runs them on the B200).

No CPU fallback for float data: a failing device call raises.  Operands the
device cannot represent (object arrays such as the reference tests'
operation-counting floats) are handed to the original table entry and
counted in ``CALLS['host_passthrough']``.
"""

from __future__ import annotations

import ctypes
import os
from collections import Counter

import numpy as np

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(_REPO, "paper_2603_14926_b200", "libmwgpu.so")

CALLS: Counter = Counter()

_P, _I, _I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
_lib = None


def _load(path=None):
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(path or LIB_PATH)
        for name in ("mw_ew_add", "mw_ew_mul"):
            fn = getattr(lib, name)
            fn.argtypes = [_I, _I, _P, _I64, _P, _I64, _P, _I64, _I64, _P]
            fn.restype = _I
        lib.mw_gemm.argtypes = [_I, _I, _P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _P]
        lib.mw_gemm.restype = _I
        lib.mw_status_string.argtypes = [_I]
        lib.mw_status_string.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def _check(rc, what):
    if rc == 0:
        return
    if rc == -2:
        raise NotImplementedError(f"{what}: no device kernel for this (K, variant)")
    if rc == -1:
        raise ValueError(f"{what}: invalid arguments")
    raise RuntimeError(f"{what}: CUDA error {rc}: {_lib.mw_status_string(rc).decode()}")


def _device_arrays(arrs):
    """Host float64 arrays -> one device (len, n) tensor."""
    import torch

    host = np.ascontiguousarray(np.stack([np.ravel(a) for a in arrs]), dtype=np.float64)
    return torch.from_numpy(host).cuda()


def _stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


def _lanewise(fn_name, k, variant_code, original):
    def op(a_comps, b_comps):
        parts = [np.asarray(c) for c in tuple(a_comps) + tuple(b_comps)]
        if any(p.dtype.kind not in "fiub" for p in parts):
            CALLS["host_passthrough"] += 1
            return original(a_comps, b_comps)
        parts = np.broadcast_arrays(*[p.astype(np.float64, copy=False) for p in parts])
        shape = parts[0].shape
        n = int(np.prod(shape, dtype=np.int64))
        if n == 0:
            return tuple(np.zeros(shape) for _ in range(k))
        import torch

        dev = _device_arrays(parts)  # rows 0..k-1: a, k..2k-1: b
        out = torch.empty((k, n), dtype=torch.float64, device=dev.device)
        es = dev.element_size()
        rc = getattr(_load(), fn_name)(k, variant_code, dev.data_ptr(), n, dev.data_ptr() + k * n * es, n,
                                       out.data_ptr(), n, n, _stream())
        _check(rc, fn_name)
        CALLS[fn_name] += 1
        res = out.cpu().numpy()
        if shape == ():
            return tuple(np.float64(res[c, 0]) for c in range(k))
        return tuple(res[c].reshape(shape) for c in range(k))

    op.__name__ = f"{fn_name}_k{k}_v{variant_code}"
    return op


def _naive_mm_gpu(a, b, variant, simd, threads):
    """linalg._naive_mm(a, b, variant, simd, threads) on mw_gemm: every C_ij
    folded t-ascending from an exact zero (bit-exact; ``simd``/``threads``
    do not change the result in the reference either)."""
    import torch

    from mwfloat.multiword import Variant

    k, m, kd, n = len(a), a[0].shape[0], a[0].shape[1], b[0].shape[1]
    if m == 0 or n == 0:
        return tuple(np.zeros((m, n)) for _ in range(k))
    A = _device_arrays(a)
    B = _device_arrays(b)
    C = torch.empty((k, m * n), dtype=torch.float64, device=A.device)
    v = 1 if variant is Variant.BRANCH_FREE else 0
    rc = _load().mw_gemm(k, v, A.data_ptr(), kd, m * kd, B.data_ptr(), n, kd * n, C.data_ptr(), n, m * n, m, n, kd,
                         _stream())
    _check(rc, "mw_gemm")
    CALLS["mw_gemm"] += 1
    res = C.cpu().numpy()
    return tuple(res[c].reshape(m, n).copy() for c in range(k))


def install(lib_path=None) -> Counter:
    """Rebind the imported reference package's dispatch points to the GPU.
    Returns the call counter (per entry point)."""
    from mwfloat import batch, linalg
    from mwfloat.multiword import Variant

    _load(lib_path)
    for k in (2, 3, 4):
        for var in (Variant.STANDARD, Variant.BRANCH_FREE):
            code = 1 if var is Variant.BRANCH_FREE else 0
            batch._BATCH_ADD[k, var] = _lanewise("mw_ew_add", k, code, batch._BATCH_ADD[k, var])
            batch._BATCH_MUL[k, var] = _lanewise("mw_ew_mul", k, code, batch._BATCH_MUL[k, var])
    linalg._naive_mm = _naive_mm_gpu
    return CALLS
