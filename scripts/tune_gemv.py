"""Time GEMV tree-kernel shapes (csrc/tune/libmwtune.so) at config 2, L2 flushed."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import gen
lib = ctypes.CDLL(os.path.join(os.path.dirname(mw._lib.LIB_PATH), "csrc", "tune", os.environ.get("TUNELIB", "libmwtune.so")))
lib.mwt_gemv.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                         ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
lib.mwt_gemv_config_name.restype = ctypes.c_char_p
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
NOFLUSH = "--noflush" in sys.argv
MAC = {3: 96, 4: 209}
PAD = int(os.environ.get("PAD", "0"))  # extra elements between A's planes (layout experiment)
lib.mwt_gemv_set_sa.argtypes = [ctypes.c_int64]
lib.mwt_gemv_set_lda.argtypes = [ctypes.c_int64]
lib.mwt_gemv_set_lda(int(os.environ.get("LDA", "0")))  # -1: every row reads row 0 (A L2-resident; timing probe)
for k in (3, 4):
    a, x = gen.config2_gemv(k)
    m, n = a.shape[1], a.shape[2]
    if PAD:
        buf = torch.empty((k, m * n + PAD), dtype=torch.float64, device="cuda")
        buf[:, : m * n] = torch.from_numpy(a.reshape(k, m * n)).cuda()
        A = buf
        lib.mwt_gemv_set_sa(m * n + PAD)
    else:
        A = torch.from_numpy(a).cuda()
        lib.mwt_gemv_set_sa(0)
    X = torch.from_numpy(x).cuda()
    y = torch.empty((k, m), dtype=torch.float64, device="cuda")
    ref = None
    sel = [int(c) for c in os.environ.get("CFGS", "").split(",") if c]
    for cfg in (sel or range(lib.mwt_gemv_num_configs())):
        st = torch.cuda.current_stream().cuda_stream
        y.fill_(float("nan"))
        rc = lib.mwt_gemv(cfg, k, A.data_ptr(), X.data_ptr(), y.data_ptr(), m, n, st)
        torch.cuda.synchronize()
        if rc != 0:
            print(f"k={k} {lib.mwt_gemv_config_name(cfg).decode():10s} rc={rc} (skipped)", flush=True)
            continue
        same = ""
        if cfg == 0:
            ref = y.clone()
        elif (cfg >= 8 or cfg == 6 or os.environ.get("TUNELIB")) and not os.environ.get("LDA"):  # (cfg 61+: persistent shuffle tree)  # staged variants keep the P = 128 order: must be bit-identical
            same = " bits==W4" if torch.equal(y.view(torch.int64), ref.view(torch.int64)) else " BITS DIFFER"
        ts = []
        for _ in range(10):
            if not NOFLUSH:
                flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); lib.mwt_gemv(cfg, k, A.data_ptr(), X.data_ptr(), y.data_ptr(), m, n, st); e1.record()
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        print(f"k={k} pad={PAD} {lib.mwt_gemv_config_name(cfg).decode():10s} {ms*1e3:8.1f} us  {MAC[k]*m*n/(ms/1e3)/1e12:6.2f} T/s{same}", flush=True)
