"""Run one GEMV tuning-harness configuration once at config 2 (for ncu)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import gen
lib = ctypes.CDLL(os.path.join(os.path.dirname(mw._lib.LIB_PATH), "csrc", "tune", os.environ.get("TUNELIB", "libmwtune.so")))
lib.mwt_gemv.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                         ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
k, cfg = int(sys.argv[1]), int(sys.argv[2])
a, x = gen.config2_gemv(k)
A, X = torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda()
y = torch.empty((k, a.shape[1]), dtype=torch.float64, device="cuda")
for _ in range(2):
    assert lib.mwt_gemv(cfg, k, A.data_ptr(), X.data_ptr(), y.data_ptr(), a.shape[1], a.shape[2],
                        torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
print("ok", k, cfg)
