"""Host-side cost of the public API per call at config 1 (DD n = 65536):
blas.dot_tensor / blas.axpy_ / batch_add through the PyTorch extension,
against the raw C-ABI call through ctypes with precomputed arguments.

Two numbers per call: the host time per call when calls are issued back to
back (wall clock / calls, GPU work queued asynchronously), and the
event-bracketed time of one eager call (device idle before it)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_14926_b200 as mw  # noqa: E402
from paper_2603_14926_b200 import _lib, blas, gen  # noqa: E402

x, y, alpha = gen.config1_dot()
X, Y = mw.LaneBatch(x), mw.LaneBatch(y)
out = torch.empty(2, dtype=torch.float64, device="cuda")
BF = mw.Variant.BRANCH_FREE
al = tuple(alpha[:, 0]) if getattr(alpha, "ndim", 1) == 2 else tuple(alpha)


def host_us(fn, n=5000):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


def event_us(fn, reps=200):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


lib = _lib.load()
ws = torch.zeros(lib.mw_dot_workspace(2, 65536), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
xp, yp, wp, op = X.planes.data_ptr(), Y.planes.data_ptr(), ws.data_ptr(), out.data_ptr()
rows = [
    ("dot_tensor (public API, extension)", lambda: blas.dot_tensor(X, Y, BF, out=out)),
    ("dot raw ctypes (precomputed args)", lambda: lib.mw_dot(2, 1, xp, 65536, yp, 65536, 65536, wp, op, 1, st)),
    ("axpy_ (public API, extension)", lambda: blas.axpy_(al, X, Y, BF)),
    ("batch_add (public API, extension)", lambda: mw.batch_add(X, Y, BF)),
]
for name, fn in rows:
    print(f"{name:40s} host {host_us(fn):6.2f} us/call   one eager call (events) {event_us(fn):6.2f} us", flush=True)
