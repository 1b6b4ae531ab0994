"""ctypes binding of the C-ABI library ``libmwgpu.so`` (include/mwgpu.h).

This is the only way the Python package reaches the GPU: every public
operation calls one of these entry points with raw device pointers taken
from torch CUDA tensors and torch's current CUDA stream.  There is no CPU
fallback -- if the library or a CUDA device is missing, calls raise.
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
    "mw_dk_exact_set_roots_per_cta": ([I], I),
    "mw_dk_exact_set_split": ([I], I),
    "mw_dk_tree_set_roots_per_cta": ([I], I),
    "mw_gemm_set_tile_policy": ([I], I),
    "mw_dot_set_cluster": ([I], I),
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


def build(verbose: bool = False) -> str:
    """Compile libmwgpu.so in-tree for sm_100a (nvcc, see csrc/Makefile)."""
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(["make", "-s", "-j8", "-C", CSRC], check=True, stdout=out)
    return LIB_PATH


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
    Uses torch's raw-handle accessor when present (no Stream object: this
    is on every call's host path), else torch.cuda.current_stream."""
    if _raw_stream is not None:
        idx = getattr(device, "index", None)
        if idx is None:
            idx = torch.cuda.current_device()
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
