"""The C-ABI library: loads without a GPU, exports every symbol the header
declares, and rejects bad arguments before launching anything."""

import ctypes
import os
import re

import pytest

from paper_2603_14926_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "mwgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mw_\w+)\s*\(", text)))


def test_library_loads_on_cpu():
    lib = _lib.load()
    assert _lib.version().startswith("mwgpu")
    assert lib is _lib.load()


def test_every_declared_symbol_is_exported():
    syms = declared_symbols()
    assert len(syms) >= 17
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert missing == []


def test_binding_covers_the_header():
    assert set(declared_symbols()) == set(_lib.EXPORTS)


def test_status_strings():
    lib = _lib.load()
    assert lib.mw_status_string(0) == b"ok"
    assert b"invalid" in lib.mw_status_string(-1)
    assert b"variant" in lib.mw_status_string(-2)


@pytest.mark.parametrize("fn", ["mw_ew_add", "mw_ew_sub", "mw_ew_mul", "mw_ew_div"])
def test_ew_argument_checks(fn):
    f = getattr(_lib.load(), fn)
    p = 0x1000  # never dereferenced: every call below returns before a launch
    assert f(5, 1, p, 8, p, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID  # bad k
    assert f(3, 0, p, 4, p, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID  # TD STANDARD, bad stride
    assert f(2, 7, p, 8, p, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID  # bad variant
    assert f(2, 1, p, 4, p, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID  # stride < n
    assert f(2, 1, None, 8, p, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID  # null
    assert f(2, 1, p, 8, p, 8, p, 8, -1, None) == _lib.MW_ERR_INVALID
    assert f(2, 1, None, 0, None, 0, None, 0, 0, None) == _lib.MW_OK  # empty


def test_gemm_argument_checks():
    f = _lib.load().mw_gemm
    p = 0x1000
    assert f(3, 2, p, 4, 16, p, 4, 16, p, 4, 16, 4, 4, 4, None) == _lib.MW_ERR_INVALID  # variant
    assert f(2, 1, p, 3, 16, p, 4, 16, p, 4, 16, 4, 4, 4, None) == _lib.MW_ERR_INVALID  # lda < kd
    assert f(2, 1, p, 4, 15, p, 4, 16, p, 4, 16, 4, 4, 4, None) == _lib.MW_ERR_INVALID  # plane stride
    assert f(2, 1, p, 4, 16, p, 4, 16, p, 4, 16, 0, 4, 4, None) == _lib.MW_OK  # m = 0


def test_other_entry_checks():
    lib = _lib.load()
    p = 0x1000
    assert lib.mw_horner(2, 1, p, 3, 5, p, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID  # sc < deg+1
    assert lib.mw_horner(4, 5, p, 8, 5, p, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID
    assert lib.mw_gemv(2, 1, p, 8, 64, p, 8, p, 8, 8, 8, 3, None) == _lib.MW_ERR_INVALID  # order
    assert lib.mw_dot(2, 1, p, 8, p, 8, 8, None, p, 9, None) == _lib.MW_ERR_INVALID
    assert lib.mw_dk_sweep(3, 1, p, 8, 8, p, p, 8, 4, 2, p, p, 8, p, p, 1, None) == _lib.MW_ERR_INVALID  # i1 < i0
    assert lib.mw_fp64_peak_kernel(0, 1, 512, 1, p, None) == _lib.MW_ERR_INVALID
    # kernels outside the dispatch tables, renormalisation, fma, the tree-sweep knob
    assert lib.mw_named_op(2, p, 8, p, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID  # unknown op
    assert lib.mw_named_op(0, p, 4, p, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID  # plane stride < n
    assert lib.mw_named_op(1, p, 8, p, 8, p, 8, 0, None) == _lib.MW_OK  # empty: nothing launched
    assert lib.mw_renormalize(5, p, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID
    assert lib.mw_renormalize(3, None, 8, p, 8, 8, None) == _lib.MW_ERR_INVALID
    assert lib.mw_fma(p, p, None, p, 8, None) == _lib.MW_ERR_INVALID
    assert lib.mw_fma(p, p, p, p, -1, None) == _lib.MW_ERR_INVALID
    # per-call tuning (no global knobs): defaults, and out-of-range values
    # rejected before anything is launched
    t = _lib.tuning()
    assert (t.gemm_tile, t.dot_cluster, t.dk_tree_roots, t.dk_exact_roots, t.dk_exact_split) == (0, 1, -1, 32, 1)
    tp = _lib.tuning_ptr
    for bad in (dict(gemm_tile=4), dict(gemm_tile=-1), dict(dot_cluster=2), dict(dk_tree_roots=3),
                dict(dk_tree_roots=-2), dict(dk_exact_roots=0), dict(dk_exact_roots=33), dict(dk_exact_split=2)):
        bt = _lib.tuning(**bad)
        assert lib.mw_gemm_ex(2, 1, p, 8, 64, p, 8, 64, p, 8, 64, 8, 8, 8, tp(bt), None) == _lib.MW_ERR_INVALID, bad
        assert lib.mw_dot_ex(2, 1, p, 8, p, 8, 8, p, p, 1, tp(bt), None) == _lib.MW_ERR_INVALID, bad
        assert lib.mw_dk_sweep_ex(3, 1, p, 8, 8, p, p, 8, 0, 8, p, p, 8, p, p, 0, p, None, tp(bt), None) == \
            _lib.MW_ERR_INVALID, bad
    # the DK collision key j*n + i must fit an int: larger degrees are refused
    assert lib.mw_dk_sweep(3, 1, p, 46341, 46341, p, p, 46341, 0, 1, p, p, 46341, p, p, 1, None) == \
        _lib.MW_ERR_INVALID
    for name in ("mw_dk_tree_set_roots_per_cta", "mw_gemm_set_tile_policy", "mw_dot_set_cluster",
                 "mw_dk_exact_set_split", "mw_dk_exact_set_roots_per_cta"):
        assert not hasattr(lib, name), f"{name}: the C-ABI keeps no global tuning state"


def test_peer_sweep_checks():
    import ctypes

    lib = _lib.load()
    p = 0x1000
    f = lib.mw_dk_sweep_peer
    ok = dict(k=3, variant=1, coeffs=p, sc=8, n=8, state_in=p, i0=0, i1=8, peer_out=p, peer_slot=p, out=p,
              my_slot=p, done=p, epoch=p, timeout=p, world=2, rank=1, sweep=0, sweeps=4, spin=1000,
              mag=p, flag=p, exact=1, ws=None, stream=None)

    def call(**kw):
        a = dict(ok, **kw)
        return f(*a.values())

    assert call(rank=2) == _lib.MW_ERR_INVALID          # rank outside world
    assert call(sweep=4) == _lib.MW_ERR_INVALID         # sweep outside [0, sweeps)
    assert call(i1=0) == _lib.MW_ERR_INVALID            # empty shard
    assert call(i1=9) == _lib.MW_ERR_INVALID            # past n
    assert call(spin=0) == _lib.MW_ERR_INVALID
    assert call(peer_slot=None) == _lib.MW_ERR_INVALID
    assert call(sc=7) == _lib.MW_ERR_INVALID
    d = lib.mw_dot_peer
    #          k  v  x  sx y  sy nl  b0 nbt roots slot my done ep to world rank spin out stream
    assert d(2, 1, p, 8, p, 8, 8, 0, 0, p, p, p, p, p, p, 2, 0, 100, p, None) == _lib.MW_ERR_INVALID  # nbt
    assert d(2, 1, p, 8, p, 8, 8, 1, 1, p, p, p, p, p, p, 2, 0, 100, p, None) == _lib.MW_ERR_INVALID  # past nbt
    assert d(2, 1, p, 8, p, 8, 8, 0, 1, p, p, p, p, p, p, 2, 2, 100, p, None) == _lib.MW_ERR_INVALID  # rank
    assert d(2, 1, p, 8, p, 8, 8, 0, 1, p, p, p, p, p, p, 2, 0, 0, p, None) == _lib.MW_ERR_INVALID  # spin
    assert d(2, 1, p, 8, p, 8, 8, 0, 65537, p, p, p, p, p, p, 2, 0, 9, p, None) == _lib.MW_ERR_INVALID
    assert d(2, 1, p, 4, p, 8, 8, 0, 1, p, p, p, p, p, p, 2, 0, 9, p, None) == _lib.MW_ERR_INVALID  # sx
    out = ctypes.c_void_p()
    assert lib.mw_peer_alloc(0, ctypes.byref(out)) == _lib.MW_ERR_INVALID
    assert lib.mw_peer_free(None) == _lib.MW_ERR_INVALID
    assert lib.mw_ipc_get_handle(None, p) == _lib.MW_ERR_INVALID
    assert lib.mw_ipc_open_handle(None, ctypes.byref(out)) == _lib.MW_ERR_INVALID


def test_workspace_sizes():
    lib = _lib.load()
    assert lib.mw_dot_workspace(2, 4096) == 0
    assert lib.mw_dot_num_partials(4097) == 2
    assert lib.mw_dot_workspace(2, 4097) == 1 + 2 * 2  # ticket + partials
    assert lib.mw_dot_workspace(4, 65536) == 1 + 16 * 4
    # 2^28 elements: ticket, 65536 partials, then 256 level-2 values
    assert lib.mw_dot_workspace(2, 1 << 28) == 1 + 65536 * 2 + 256 * 2
    assert lib.mw_tree_fold_workspace(3, 256) == 0
    assert lib.mw_tree_fold_workspace(3, 257) == 2 * 3


def test_extension_loads_and_refuses_cpu_tensors():
    """The PyTorch extension over the C-ABI (csrc/ext/mwext.cpp) loads on a
    CPU-only host, exposes the hot entry points, and refuses host tensors
    (no CPU fallback) before anything is launched."""
    import torch

    e = _lib.ext()
    for name in ("ew", "axpy_", "dot", "gemv", "gemm", "horner", "dk_sweep", "version"):
        assert hasattr(e, name), name
    assert e.version() == _lib.version()
    x = torch.zeros(2, 8, dtype=torch.float64)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        e.ew(0, 1, x, x)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        e.dot(1, x, x, 1)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        e.gemm(1, x.reshape(2, 2, 4), x.reshape(2, 4, 2), x.reshape(2, 2, 4)[:, :, :2].contiguous())
