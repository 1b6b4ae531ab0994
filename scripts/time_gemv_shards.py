"""Per-rank GEMV time for a 1/G row-block shard of config 2 (TD / QD
2048 x 2048), one call after an L2 flush and back to back in a graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import blas, gen
BF = mw.Variant.BRANCH_FREE
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for k in (3, 4):
    a, x = gen.config2_gemv(k)
    A, X = mw.MWMatrix(a), mw.LaneBatch(x)
    for G in (1, 2, 4, 8):
        m = a.shape[1] // G
        y = torch.empty((k, m), dtype=torch.float64, device="cuda")
        fn = lambda: blas.gemv(A, X, BF, "tree", 0, m, out=y)
        fn(); torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                fn()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        print(f"k={k} G={G} rows={m}: flushed {sorted(ts)[5]*1e3:6.1f} us, back-to-back {e0.elapsed_time(e1)/20*1e3:6.1f} us", flush=True)
