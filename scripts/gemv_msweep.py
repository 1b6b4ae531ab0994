"""GEMV kernel timing vs number of rows m (n = 2048), L2 not flushed: separates
per-wave throughput from wave quantisation (tuning harness)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
lib = ctypes.CDLL(os.path.join(os.path.dirname(mw._lib.LIB_PATH), "csrc", "tune", os.environ.get("TUNELIB", "libmwtune.so")))
lib.mwt_gemv.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                         ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
lib.mwt_gemv_config_name.restype = ctypes.c_char_p
MAC = {2: 29, 3: 96, 4: 209}
cfgs = [int(c) for c in os.environ.get("CFGS", "0,26").split(",")]
n = 2048
for k in (3, 4):
    for m in [int(v) for v in os.environ.get("MS", "148,296,592,740,1184,1480,2048,2960,4096,8192").split(",")]:
        A = torch.rand((k, m, n), dtype=torch.float64, device="cuda") * 2 - 1
        X = torch.rand((k, n), dtype=torch.float64, device="cuda") * 2 - 1
        A[1:] *= 1e-17; X[1:] *= 1e-17
        y = torch.empty((k, m), dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        out = []
        for cfg in cfgs:
            lib.mwt_gemv(cfg, k, A.data_ptr(), X.data_ptr(), y.data_ptr(), m, n, st)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    lib.mwt_gemv(cfg, k, A.data_ptr(), X.data_ptr(), y.data_ptr(), m, n,
                                 torch.cuda.current_stream().cuda_stream)
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 20
            out.append(f"{lib.mwt_gemv_config_name(cfg).decode()} {us:7.1f}us {MAC[k]*m*n/(us*1e-6)/1e12:5.2f}T")
        print(f"k={k} m={m:5d} " + " | ".join(out), flush=True)
