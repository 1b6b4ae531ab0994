"""Time alternative GEMM tile configurations (csrc/tune/libmwtune.so) at
the config-3 sizes and check each is bit-identical to the product kernel."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_14926_b200 as mw  # noqa: E402
from paper_2603_14926_b200 import gen  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(mw._lib.LIB_PATH), "csrc", "tune", "libmwtune.so"))
lib.mwt_gemm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                         ctypes.c_int64, ctypes.c_void_p]
lib.mwt_config_name.restype = ctypes.c_char_p
MAC = {2: 29, 3: 96, 4: 209}
only_k = [int(a) for a in sys.argv[1:]] or [2, 3, 4]
for k, n in ((2, 4096), (3, 2048), (4, 2048)):
    if k not in only_k:
        continue
    a, b = gen.config3_gemm(k, n)
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    ref = mw.matmul(mw.MWMatrix(A), mw.MWMatrix(B), mw.MatMulPlan(scheme="naive", variant="bf")).planes
    C = torch.empty_like(A)
    for cfg in range(lib.mwt_num_configs()):
        st = torch.cuda.current_stream().cuda_stream
        rc = lib.mwt_gemm(cfg, k, A.data_ptr(), B.data_ptr(), C.data_ptr(), n, st)
        torch.cuda.synchronize()
        if rc:
            print(k, lib.mwt_config_name(cfg).decode(), "rc", rc)
            continue
        same = torch.equal(C.view(torch.int64), ref.view(torch.int64))
        times = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lib.mwt_gemm(cfg, k, A.data_ptr(), B.data_ptr(), C.data_ptr(), n, st)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = min(times)
        print(f"k={k} n={n} {lib.mwt_config_name(cfg).decode():18s} {ms:9.3f} ms  "
              f"{MAC[k] * n**3 / (ms / 1e3) / 1e12:6.2f} T/s  bitwise={same}", flush=True)
