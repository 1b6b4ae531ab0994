"""GEMM tile configurations on a row-block shard (n/G rows of A and C, full
B) -- what one rank multiplies at G GPUs -- at the config-3 sizes
(csrc/tune/libmwtune.so; timing only)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import gen
lib = ctypes.CDLL(os.path.join(os.path.dirname(mw._lib.LIB_PATH), "csrc", "tune", "libmwtune.so"))
lib.mwt_gemm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                         ctypes.c_int64, ctypes.c_void_p]
lib.mwt_gemm_set_rows.argtypes = [ctypes.c_int64]
lib.mwt_config_name.restype = ctypes.c_char_p
MAC = {2: 29, 3: 96, 4: 209}
cfgs = [int(c) for c in os.environ.get("CFGS", "0,1,2,4,5,6,7,8,9").split(",")]
for k, n in ((2, 4096), (3, 2048), (4, 2048)):
    a, b = gen.config3_gemm(k, n)
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    for G in (1, 4, 8):
        m = n // G
        C = torch.empty((k, m, n), dtype=torch.float64, device="cuda")
        lib.mwt_gemm_set_rows(m)
        out = []
        for cfg in cfgs:
            st = torch.cuda.current_stream().cuda_stream
            if lib.mwt_gemm(cfg, k, A.data_ptr(), B.data_ptr(), C.data_ptr(), n, st):
                continue
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); lib.mwt_gemm(cfg, k, A.data_ptr(), B.data_ptr(), C.data_ptr(), n, st); e1.record()
                torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[1]
            out.append(f"{lib.mwt_config_name(cfg).decode()} {ms:7.2f}ms {MAC[k]*m*n*n/(ms/1e3)/1e12:5.2f}T")
        print(f"k={k} G={G} rows={m}: " + " | ".join(out), flush=True)
    lib.mwt_gemm_set_rows(0)
