import sys, time, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import _lib
e = _lib.ext(); lib = _lib.load()
a = torch.zeros(2, 1024, dtype=torch.float64, device="cuda"); z = torch.zeros(2, 0, dtype=torch.float64, device="cuda")
t1 = torch.zeros(1024, device="cuda"); t2 = torch.zeros(1024, device="cuda"); t3 = torch.zeros(1024, device="cuda")
st = torch.cuda.current_stream().cuda_stream
ap = a.data_ptr()
def host(fn, n=20000):
    for _ in range(500): fn()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e6
print("ext.version (pybind only)      ", host(lambda: e.version()))
print("ext.ew w=0 (validate, no launch)", host(lambda: e.ew(0, 1, z, z, z)))
print("ext.ew w=1024 (launch)          ", host(lambda: e.ew(0, 1, a, a, a)))
print("ctypes mw_ew_add w=1024          ", host(lambda: lib.mw_ew_add(2, 1, ap, 1024, ap, 1024, ap, 1024, 1024, st)))
print("torch.add out= (1 kernel)        ", host(lambda: torch.add(t1, t2, out=t3)))
print("ctypes mw_version (no launch)    ", host(lambda: lib.mw_version()))
