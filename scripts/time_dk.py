"""Time config-5 DK sweeps (200 per CUDA graph) for both orders, TD and QD."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import gen
from paper_2603_14926_b200.roots import DKSweepGraph
orders = sys.argv[1:] or ["tree", "exact"]
from paper_2603_14926_b200 import _lib
tune = _lib.tuning(dk_tree_roots=int(os.environ["DK_TREE_ROOTS"])) if os.environ.get("DK_TREE_ROOTS") else None
for k in (3, 4):
    q = mw.MonicPoly(torch.from_numpy(gen.config5_poly(k)).cuda())
    zre, zim = (torch.from_numpy(t).cuda() for t in gen.config5_init(k))
    for order in orders:
        g = DKSweepGraph(q, mw.RootState(re=zre, im=zim), 200, mw.Variant.BRANCH_FREE, exact_order=order == "exact", tuning=tune)
        g.replay(); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(f"k={k} {order}: {ts[2] / 200 * 1e3:.2f} us/sweep", flush=True)
