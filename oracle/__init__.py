"""CPU oracle for the DD/TD/QD hot path — TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``libmworacle.so`` (built from ``mw_oracle.c`` by
``make -C oracle``), a C restatement of the reference mwfloat package's
algorithms (each C function cites the reference file:line it follows).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / reference arm may import this module, and only as the checker
or the CPU comparison -- never as the measured or shipped path.

Pinned against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``); see ``tests/test_oracle_golden.py``.

All arrays are numpy float64 with K planes along axis 0 (component-planar),
the layout of the reference's tuples of K arrays.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmworacle.so")

STANDARD = 0
BRANCH_FREE = 1

_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int
        I64 = ctypes.c_int64
        L.mwo_ew.argtypes = [I, I, I, P, I64, P, I64, P, I64, I64]
        L.mwo_axpy.argtypes = [I, I, P, P, I64, P, I64, I64]
        L.mwo_dot.argtypes = [I, I, P, I64, P, I64, I64, I, P, P]
        L.mwo_tree_fold.argtypes = [I, I, P, I64, I64, P, P]
        L.mwo_gemv.argtypes = [I, I, P, I64, I64, P, I64, P, I64, I64, I64, I]
        L.mwo_gemm_rows.argtypes = [I, I, P, I64, I64, P, I64, I64, P, I64, I64, I64, I64, I64, I64]
        L.mwo_horner.argtypes = [I, I, P, I64, I64, P, I64, P, I64, I64]
        L.mwo_poly_eval.argtypes = [I, I, P, I64, I64, P, P, I64, P, P, I64, I64, I, P, I64]
        L.mwo_dk_sweep.argtypes = [I, I, P, I64, I64, P, P, I64, I64, I64, P, P, I64, P, P, I]
        L.mwo_set_threads.argtypes = [I]
        L.mwo_named.argtypes = [I, P, I64, P, I64, P, I64, I64]
        L.mwo_renormalize.argtypes = [I, P, I64, P, I64, I64]
        L.mwo_fma.argtypes = [P, P, P, P, I64]
        L.mwo_max_threads.restype = I
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _planes(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a


def _variant(v) -> int:
    if isinstance(v, int):
        return v
    s = str(getattr(v, "value", v)).lower()
    return STANDARD if s in ("std", "standard") else BRANCH_FREE


def _check(rc: int):
    if rc == -2:
        raise NotImplementedError("oracle restates STANDARD for K=2 only")
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (rc={rc})")


def set_threads(n: int):
    lib().mwo_set_threads(int(n))


def max_threads() -> int:
    return lib().mwo_max_threads()


_EW = {"add": 0, "sub": 1, "mul": 2, "div": 3}


def ew(op: str, a, b, variant=BRANCH_FREE) -> np.ndarray:
    """Lane-wise add/sub/mul/div over K x n planes."""
    a = _planes(a)
    b = _planes(b)
    k = a.shape[0]
    n = a[0].size
    out = np.empty_like(a)
    with np.errstate(all="ignore"):
        _check(lib().mwo_ew(_EW[op], k, _variant(variant), _ptr(a), n, _ptr(b), n, _ptr(out), n, n))
    return out


def axpy(alpha, x, y, variant=BRANCH_FREE) -> np.ndarray:
    x = _planes(x)
    y = _planes(y).copy()
    al = np.ascontiguousarray(np.asarray(alpha, dtype=np.float64))
    k, n = x.shape
    _check(lib().mwo_axpy(k, _variant(variant), _ptr(al), _ptr(x), n, _ptr(y), n, n))
    return y


def dot(x, y, variant=BRANCH_FREE, order: int = 0) -> np.ndarray:
    x = _planes(x)
    y = _planes(y)
    k, n = x.shape
    out = np.zeros(k)
    scratch = np.zeros(max(1, n) * 4)
    _check(lib().mwo_dot(k, _variant(variant), _ptr(x), n, _ptr(y), n, n, order, _ptr(out), _ptr(scratch)))
    return out


def tree_fold(v, variant=BRANCH_FREE) -> np.ndarray:
    v = _planes(v)
    k, cnt = v.shape
    out = np.zeros(k)
    scratch = np.zeros(max(1, cnt) * 4)
    _check(lib().mwo_tree_fold(k, _variant(variant), _ptr(v), cnt, cnt, _ptr(out), _ptr(scratch)))
    return out


def gemv(a, x, variant=BRANCH_FREE, order: int = 0) -> np.ndarray:
    a = _planes(a)
    x = _planes(x)
    k, m, n = a.shape
    y = np.zeros((k, m))
    _check(lib().mwo_gemv(k, _variant(variant), _ptr(a), n, m * n, _ptr(x), n, _ptr(y), m, m, n, order))
    return y


def gemm(a, b, variant=BRANCH_FREE, rows=None) -> np.ndarray:
    """C = A B (reference naive order).  rows=(r0, r1) computes that row
    block only (the other rows of the result stay zero)."""
    a = _planes(a)
    b = _planes(b)
    k, m, kd = a.shape
    _, kd2, n = b.shape
    if kd != kd2:
        raise ValueError("shape mismatch")
    r0, r1 = rows if rows is not None else (0, m)
    c = np.zeros((k, m, n))
    _check(
        lib().mwo_gemm_rows(k, _variant(variant), _ptr(a), kd, m * kd, _ptr(b), n, kd * n, _ptr(c), n, m * n, r0, r1, n, kd)
    )
    return c


def horner(coeffs, x, variant=BRANCH_FREE) -> np.ndarray:
    coeffs = _planes(coeffs)
    x = _planes(x)
    k, nc = coeffs.shape
    npts = x.shape[1]
    y = np.zeros((k, npts))
    _check(lib().mwo_horner(k, _variant(variant), _ptr(coeffs), nc, nc - 1, _ptr(x), npts, _ptr(y), npts, npts))
    return y


def poly_eval(coeffs, xre, xim=None, variant=BRANCH_FREE, method: str = "estrin"):
    """Batched Horner / Estrin (poly.py:89-178) at real points (xim None)
    or complex points; returns y or (yre, yim)."""
    coeffs = _planes(coeffs)
    xre = _planes(xre)
    k, npts = xre.shape
    deg = coeffs.shape[1] - 1
    length = 1
    while length < deg + 1:
        length *= 2
    nt = max_threads()
    scratch = np.zeros(nt * length * 8 * 2 + 8)
    yre = np.zeros((k, npts))
    yim = None
    xp = None
    if xim is not None:
        xim = _planes(xim)
        yim = np.zeros((k, npts))
        xp = _ptr(xim)
    _check(
        lib().mwo_poly_eval(k, _variant(variant), _ptr(coeffs), coeffs.shape[1], deg, _ptr(xre), xp, npts,
                            _ptr(yre), None if yim is None else _ptr(yim), npts, npts,
                            {"horner": 0, "estrin": 1}[method], _ptr(scratch), length * 2)
    )
    return yre if xim is None else (yre, yim)


def dk_sweep(coeffs, zre, zim, variant=BRANCH_FREE, exact: bool = True, rows=None):
    """One dk_iterate sweep.  Returns (new_re, new_im, step_mag, collision)
    where collision is None or (j, i) of the first vanishing factor."""
    coeffs = _planes(coeffs)
    zre = _planes(zre)
    zim = _planes(zim)
    k, n = zre.shape
    i0, i1 = rows if rows is not None else (0, n)
    ore = zre.copy()
    oim = zim.copy()
    mag = np.zeros(n)
    coll = np.zeros(1, dtype=np.int64)
    with np.errstate(all="ignore"):
        _check(
            lib().mwo_dk_sweep(
                k, _variant(variant), _ptr(coeffs), coeffs.shape[1], n, _ptr(zre), _ptr(zim), n, i0, i1,
                _ptr(ore), _ptr(oim), n, _ptr(mag), _ptr(coll), 1 if exact else 0,
            )
        )
    c = int(coll[0])
    return ore, oim, mag, (None if c < 0 else (c // n, c % n))


def named(op: str, a, b) -> np.ndarray:
    """dw_add_sloppy (op "dw_add_sloppy", DD) or tw_mul_cleaned ("tw_mul_cleaned", TD)."""
    code = {"dw_add_sloppy": 0, "tw_mul_cleaned": 1}[op]
    a, b = _planes(a), _planes(b)
    out = np.empty_like(a)
    n = a.shape[1]
    _check(lib().mwo_named(code, _ptr(a), n, _ptr(b), n, _ptr(out), n, n))
    return out


def renormalize(k: int, raw) -> np.ndarray:
    """k = 2: quick_two_sum of 2 planes; 3: tw_renormalize of 4; 4: qw_renormalize of 5."""
    raw = _planes(raw)
    n = raw.shape[1]
    out = np.empty((k, n))
    _check(lib().mwo_renormalize(k, _ptr(raw), n, _ptr(out), n, n))
    return out


def fma(a, b, c) -> np.ndarray:
    a, b, c = (np.ascontiguousarray(v, dtype=np.float64).ravel() for v in (a, b, c))
    out = np.empty_like(a)
    _check(lib().mwo_fma(_ptr(a), _ptr(b), _ptr(c), _ptr(out), a.size))
    return out
