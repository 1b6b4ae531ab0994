"""Per-rank DK tree sweep time at config 5 for a 1/G root shard (what one
rank computes at G GPUs, exchange excluded), for each roots-per-CTA form of
the tree kernel: 50 sweeps of roots [0, 512/G) in one CUDA graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import _lib, gen
from paper_2603_14926_b200.roots import sweep_into

lib = _lib.load()
BF = mw.Variant.BRANCH_FREE
for k in (3, 4):
    coeffs = torch.from_numpy(gen.config5_poly(k)).cuda()
    zre, zim = (torch.from_numpy(t).cuda() for t in gen.config5_init(k))
    n = zre.shape[1]
    ore, oim = torch.empty_like(zre), torch.empty_like(zim)
    mag = torch.empty(n, dtype=torch.float64, device="cuda")
    flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
    for G in (1, 2, 4, 8):
        i1 = n // G
        row = []
        for r in (0, 1, 2, 4, -1):
            tune = _lib.tuning(dk_tree_roots=r)
            sweep_into(coeffs, zre, zim, ore, oim, mag, flag, BF, False, 0, i1, tuning=tune)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(50):
                    sweep_into(coeffs, zre, zim, ore, oim, mag, flag, BF, False, 0, i1, tuning=tune)
            g.replay(); torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 50 * 1e3)
            ts.sort()
            row.append(f"R={r:2d} {ts[2]:6.2f}us")
        print(f"k={k} G={G} roots={i1:3d}: " + " | ".join(row), flush=True)
