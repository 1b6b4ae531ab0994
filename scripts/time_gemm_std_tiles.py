"""Standard (renormalising) GEMM per tile slot at config-3 sizes (timing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import _lib, gen
from paper_2603_14926_b200.linalg import gemm_into
lib = _lib.load()
for var in (mw.Variant.STANDARD, mw.Variant.BRANCH_FREE):
    for k, n in ((3, 2048), (4, 2048), (3, 1024), (4, 1024)):
        A, B = (torch.from_numpy(t).cuda() for t in gen.config3_gemm(k, n))
        C = torch.empty_like(A)
        row = []
        for pol in (1, 2, 3, 0):
            tune = _lib.tuning(gemm_tile=pol)
            gemm_into(A, B, C, var, tuning=tune); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); gemm_into(A, B, C, var, tuning=tune); e1.record(); torch.cuda.synchronize()
            row.append(f"{['auto','slot0','slot1','slot2'][pol]} {e0.elapsed_time(e1):7.2f}ms")
        print(f"{var.value} k={k} n={n}: " + " | ".join(row), flush=True)
