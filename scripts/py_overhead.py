"""Host-side cost of the public API per call (config-1 dot / axpy), against a
raw ctypes launch with precomputed arguments (tuning harness)."""
import time, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import blas, gen, _lib
x, y, alpha = gen.config1_dot()
X, Y = mw.LaneBatch(x), mw.LaneBatch(y)
out = torch.empty(2, dtype=torch.float64, device="cuda")
BF = mw.Variant.BRANCH_FREE
for _ in range(100): blas.dot_tensor(X, Y, BF, out=out)
torch.cuda.synchronize()
def t(fn, n=2000):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e6
print("dot_tensor", t(lambda: blas.dot_tensor(X, Y, BF, out=out)))
lib = _lib.load()
ws = blas._workspace(X.device, lib.mw_dot_workspace(2, 65536))
st = torch.cuda.current_stream().cuda_stream
xp, yp, wp, op = X.planes.data_ptr(), Y.planes.data_ptr(), ws.data_ptr(), out.data_ptr()
print("raw ctypes", t(lambda: lib.mw_dot(2, 1, xp, 65536, yp, 65536, 65536, wp, op, 1, st)))
print("current_stream", t(lambda: torch.cuda.current_stream(X.device).cuda_stream))
print("variant_code", t(lambda: mw.multiword.variant_code(BF)))
print("ws size", t(lambda: lib.mw_dot_workspace(2, 65536)))
print("axpy_", t(lambda: blas.axpy_(tuple(alpha), X, Y, BF)))
