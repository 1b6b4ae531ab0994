"""Time the exact-order DK sweep for several roots-per-CTA settings."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import gen, _lib
lib = _lib.load()
lib.mw_dk_exact_set_roots_per_cta.argtypes = [ctypes.c_int]
for k in (3, 4):
    q = mw.MonicPoly(gen.config5_poly(k))
    st = mw.RootState(*[torch.from_numpy(t).cuda() for t in gen.config5_init(k)])
    ref = None
    for r in (32, 16, 8, 4, 2, 1):
        lib.mw_dk_exact_set_roots_per_cta(r)
        out = mw.dk_sweeps(q, st, 2, mw.Variant.BRANCH_FREE, exact_order=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = mw.dk_sweeps(q, st, 10, mw.Variant.BRANCH_FREE, exact_order=True)
        e1.record(); torch.cuda.synchronize()
        bits = out.re.cpu().numpy().view(np.int64)
        same = ref is None or np.array_equal(bits, ref)
        ref = bits if ref is None else ref
        print(f"k={k} roots/CTA={r:2d}: {e0.elapsed_time(e1)/10*1e3:8.1f} us/sweep  bitwise_same={same}", flush=True)
