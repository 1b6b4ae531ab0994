"""Time matmul schemes on one GPU (CUDA events)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import gen

for k, n in ((2, 4096), (3, 2048), (4, 2048)):
    a, b = gen.config3_gemm(k, n)
    A, B = mw.MWMatrix(a), mw.MWMatrix(b)
    for scheme, cut in (("naive", 32), ("strassen", 32), ("strassen", 64), ("strassen", 128), ("strassen", 256)):
        plan = mw.MatMulPlan(scheme=scheme, variant="bf", strassen_cutoff=cut)
        mw.matmul(A, B, plan)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mw.matmul(A, B, plan)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"k={k} n={n} {scheme:8s} cut={cut:4d}: {ms:8.2f} ms  eff {2*n**3/ms/1e6:8.1f} G MP-ops/s", flush=True)
