"""Config-1 tree dot (DD n = 65536): cluster form vs single-launch ticket
form, 100 calls per CUDA graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import _lib, blas, gen
lib = _lib.load()
BF = mw.Variant.BRANCH_FREE
for k in (2, 3, 4):
    rng = __import__("numpy").random.default_rng(k)
    X, Y = mw.LaneBatch(gen.g_k(rng, k, 65536)), mw.LaneBatch(gen.g_k(rng, k, 65536))
    out = torch.empty(k, dtype=torch.float64, device="cuda")
    for on in (0, 1):
        tune = _lib.tuning(dot_cluster=on)
        blas.dot_tensor(X, Y, BF, out=out, tuning=tune); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(100):
                blas.dot_tensor(X, Y, BF, out=out, tuning=tune)
        g.replay(); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 10)
        print(f"k={k} {'cluster' if on else 'ticket '}: {sorted(ts)[2]:.2f} us per dot", flush=True)
