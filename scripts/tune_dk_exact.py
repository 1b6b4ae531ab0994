"""Time the exact-order DK sweep: single-warp chains vs split warp pairs,
for several roots-per-CTA settings (config 5, n = 512).  Every setting must
give bit-identical roots.  (The split form is used for QD only; for DD/TD
split=1 runs the single-warp kernel.)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import gen, _lib
lib = _lib.load()
for k in (2, 3, 4):
    q = mw.MonicPoly(gen.config5_poly(k))
    st = mw.RootState(*[torch.from_numpy(t).cuda() for t in gen.config5_init(k)])
    ref = None
    for split in (0, 1):
        for r in (32, 16, 8):
            tune = _lib.tuning(dk_exact_split=split, dk_exact_roots=r)
            out = mw.dk_sweeps(q, st, 2, mw.Variant.BRANCH_FREE, exact_order=True, tuning=tune)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = mw.dk_sweeps(q, st, 10, mw.Variant.BRANCH_FREE, exact_order=True, tuning=tune)
            e1.record(); torch.cuda.synchronize()
            bits = np.stack([out.re.cpu().numpy(), out.im.cpu().numpy()]).view(np.int64)
            same = ref is None or np.array_equal(bits, ref)
            ref = bits if ref is None else ref
            print(f"k={k} split={split} roots/CTA={r:2d}: {e0.elapsed_time(e1)/10*1e3:8.1f} us/sweep  "
                  f"bitwise_same={same}", flush=True)
