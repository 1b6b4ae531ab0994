"""Bindings of the C-ABI library ``libmwgpu.so`` (include/mwgpu.h).

The package reaches the GPU only through that library:

* ``ext()`` -- the PyTorch extension ``_mwext.so`` (csrc/ext/mwext.cpp)
  for the hot entry points (lane ops, axpy, dot, GEMV, GEMM, Horner, DK
  sweep): tensors in, validation, device guard and torch's current stream
  in C++;
* ``load()`` -- ctypes for the cold paths (peer memory / IPC, named ops,
  Estrin, partial dots, the microbenchmark), with raw device pointers and
  torch's current stream.

There is no CPU fallback -- if a library or a CUDA device is missing,
calls raise.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmwgpu.so")
CSRC = os.path.join(_HERE, "csrc")

MW_OK = 0
MW_ERR_INVALID = -1
MW_ERR_UNSUPPORTED = -2
ORDER_EXACT = 0
ORDER_TREE = 1

_lib = None

P = ctypes.c_void_p
I = ctypes.c_int
I64 = ctypes.c_int64

_SIGS = {
    "mw_version": ([], ctypes.c_char_p),
    "mw_status_string": ([I], ctypes.c_char_p),
    "mw_eft": ([I, P, P, P, P, I64, P], I),
    "mw_ew_add": ([I, I, P, I64, P, I64, P, I64, I64, P], I),
    "mw_ew_sub": ([I, I, P, I64, P, I64, P, I64, I64, P], I),
    "mw_ew_mul": ([I, I, P, I64, P, I64, P, I64, I64, P], I),
    "mw_named_op": ([I, P, I64, P, I64, P, I64, I64, P], I),
    "mw_renormalize": ([I, P, I64, P, I64, I64, P], I),
    "mw_fma": ([P, P, P, P, I64, P], I),
    "mw_ew_div": ([I, I, P, I64, P, I64, P, I64, I64, P], I),
    "mw_axpy": ([I, I, P, P, I64, P, I64, I64, P], I),
    "mw_dot_workspace": ([I, I64], I64),
    "mw_dot": ([I, I, P, I64, P, I64, I64, P, P, I, P], I),
    "mw_dot_num_partials": ([I64], I64),
    "mw_dot_partials": ([I, I, P, I64, P, I64, I64, P, I64, P], I),
    "mw_tree_fold_workspace": ([I, I64], I64),
    "mw_tree_fold": ([I, I, P, I64, I64, P, P, P], I),
    "mw_gemv": ([I, I, P, I64, I64, P, I64, P, I64, I64, I64, I, P], I),
    "mw_gemm": ([I, I, P, I64, I64, P, I64, I64, P, I64, I64, I64, I64, I64, P], I),
    "mw_gemm_batched": ([I, I, P, I64, I64, I64, P, I64, I64, I64, P, I64, I64, I64, P, I64, I64, I64, I64, I64,
                         I64, I64, P], I),
    "mw_horner": ([I, I, P, I64, I64, P, I64, P, I64, I64, P], I),
    "mw_poly_eval": ([I, I, P, I64, I64, P, P, I64, P, P, I64, I64, I, P], I),
    "mw_dk_sweep": ([I, I, P, I64, I64, P, P, I64, I64, I64, P, P, I64, P, P, I, P], I),
    "mw_tuning_defaults": ([P], I),
    "mw_gemm_ex": ([I, I, P, I64, I64, P, I64, I64, P, I64, I64, I64, I64, I64, P, P], I),
    "mw_dot_ex": ([I, I, P, I64, P, I64, I64, P, P, I, P, P], I),
    "mw_dk_sweep_ex": ([I, I, P, I64, I64, P, P, I64, I64, I64, P, P, I64, P, P, I, P, P, P, P], I),
    "mw_dk_sweep_peer": ([I, I, P, I64, I64, P, I64, I64, P, P, P, P, P, P, P, I, I, I, I, ctypes.c_longlong, P, P,
                          I, P, P], I),
    "mw_dk_sweep_workspace": ([I, I64, I64], I64),
    "mw_dk_sweep_ws": ([I, I, P, I64, I64, P, P, I64, I64, I64, P, P, I64, P, P, I, P, P], I),
    "mw_dot_peer": ([I, I, P, I64, P, I64, I64, I64, I64, P, P, P, P, P, P, I, I, ctypes.c_longlong, P, P], I),
    "mw_peer_alloc": ([I64, ctypes.POINTER(P)], I),
    "mw_peer_free": ([P], I),
    "mw_ipc_get_handle": ([P, P], I),
    "mw_ipc_open_handle": ([P, ctypes.POINTER(P)], I),
    "mw_ipc_close_handle": ([P], I),
    "mw_fp64_peak_kernel": ([I, I, I, I, P, P], I),
    "mw_device_sm_count": ([], I),
}

EXPORTS = tuple(_SIGS)


class Tuning(ctypes.Structure):
    """mw_tuning (include/mwgpu.h): per-call launch-shape choices; results
    never depend on them.  Defaults as in the library."""

    _fields_ = [("gemm_tile", I), ("dot_cluster", I), ("dk_tree_roots", I), ("dk_exact_roots", I),
                ("dk_exact_split", I)]


def tuning(**kw) -> Tuning:
    """A Tuning with the library defaults, overridden by ``kw``."""
    t = Tuning()
    load().mw_tuning_defaults(ctypes.byref(t))
    for key, val in kw.items():
        if not hasattr(t, key):
            raise TypeError(f"unknown tuning field {key!r}")
        setattr(t, key, int(val))
    return t


def tune_kw(t, *fields) -> dict:
    """Keyword arguments for the extension from an optional Tuning."""
    return {} if t is None else {f: int(getattr(t, f)) for f in fields}


def tuning_ptr(t):
    """ctypes argument for an optional Tuning (None -> NULL = defaults)."""
    return None if t is None else ctypes.cast(ctypes.byref(t), ctypes.c_void_p)


def build(verbose: bool = False) -> str:
    """Compile libmwgpu.so in-tree for sm_100a (nvcc, see csrc/Makefile)."""
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(["make", "-s", "-j8", "-C", CSRC], check=True, stdout=out)
    return LIB_PATH


EXT_PATH = os.path.join(_HERE, "_mwext.so")
_ext = None


def ext():
    """The PyTorch extension over the C-ABI (csrc/ext/mwext.cpp): the hot
    entry points take torch tensors directly (validation, device guard and
    torch's current stream in C++).  Raises if it has not been built."""
    global _ext
    if _ext is None:
        if not os.path.exists(EXT_PATH):
            raise RuntimeError(
                f"mwgpu: extension missing at {EXT_PATH}; build it with "
                "`make -C paper_2603_14926_b200/csrc` (no CPU fallback exists)"
            )
        import importlib.machinery
        import importlib.util

        load()  # libmwgpu.so first (the extension links it)
        loader = importlib.machinery.ExtensionFileLoader("_mwext", EXT_PATH)
        spec = importlib.util.spec_from_file_location("_mwext", EXT_PATH, loader=loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        _ext = mod
    return _ext


def load() -> ctypes.CDLL:
    """Load the library (once).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"mwgpu: native library missing at {LIB_PATH}; build it with "
                "`make -C paper_2603_14926_b200/csrc` (no CPU fallback exists)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(device: torch.device | None = None) -> int:
    """cudaStream_t of torch's current stream on ``device`` (as an int).
    The C library launches on the CURRENT device, so an operand on another
    device is an error here (wrap the call in ``torch.cuda.device(...)``;
    the extension's entry points switch devices themselves) -- never a
    launch on the wrong GPU.  Uses torch's
    raw-handle accessor when present (no Stream object: this is on every
    call's host path), else torch.cuda.current_stream."""
    cur = torch.cuda.current_device()
    idx = getattr(device, "index", None)
    if idx is None:
        idx = cur
    elif idx != cur:
        raise ValueError(f"mwgpu: operands on cuda:{idx} but the current device is cuda:{cur}; "
                         "launch under torch.cuda.device(...)")
    if _raw_stream is not None:
        return _raw_stream(idx)
    return torch.cuda.current_stream(device).cuda_stream


def check(rc: int, what: str):
    if rc == MW_OK:
        return
    if rc == MW_ERR_UNSUPPORTED:
        raise NotImplementedError(
            f"{what}: no device kernel for this (k, variant) (no CPU fallback)"
        )
    if rc == MW_ERR_INVALID:
        raise ValueError(f"{what}: invalid arguments")
    msg = load().mw_status_string(rc)
    raise RuntimeError(f"{what}: CUDA error {rc}: {msg.decode() if msg else '?'}")


def require_cuda(*tensors: torch.Tensor):
    for t in tensors:
        if not t.is_cuda:
            raise RuntimeError(
                "mwgpu: operands must live on a CUDA device; the B200 path has no CPU fallback"
            )


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def version() -> str:
    return load().mw_version().decode()
