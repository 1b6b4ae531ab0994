"""Exact-order DK sweep time vs roots per CTA (config 5, 20 sweeps per graph)."""
import os, sys
sys.path.insert(0, '/root/repo')
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import _lib, gen
from paper_2603_14926_b200.roots import DKSweepGraph
lib = _lib.load()
for k in (2, 3, 4):
    q = mw.MonicPoly(torch.from_numpy(gen.config5_poly(k)).cuda())
    zre, zim = (torch.from_numpy(t).cuda() for t in gen.config5_init(k))
    for r in (4, 8, 16, 32):
        g = DKSweepGraph(q, mw.RootState(re=zre, im=zim), 20, mw.Variant.BRANCH_FREE, exact_order=True,
                         tuning=_lib.tuning(dk_exact_roots=r))
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        print(f"k={k} roots/cta={r}: {e0.elapsed_time(e1)/20*1e3:.1f} us/sweep", flush=True)
