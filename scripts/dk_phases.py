"""Phase timeline of the tree DK sweep (dk_treem_kernel built with
MW_DK_PROFILE in csrc/tune/libdkphase.so): per CTA, %globaltimer at each
phase boundary; prints medians over CTAs relative to the CTA's start, and
the span from the first CTA start to the last CTA end."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import gen

lib = ctypes.CDLL(os.path.join(os.path.dirname(mw._lib.LIB_PATH), "csrc", "tune", "libdkphase.so"))
P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
lib.dkp_sweep.argtypes = [I, P, I64, P, P, I64, I64, P, P, P, P, P, I, P]
lib.dkp_read.argtypes = [P, I]
NAMES = ["start", "den chains", "num chains", "pow wait", "scan done", "sync1", "sync2(tA)", "trees", "tail"]
for k in (3, 4):
    coeffs = torch.from_numpy(gen.config5_poly(k)).cuda()
    zre, zim = (torch.from_numpy(t).cuda() for t in gen.config5_init(k))
    n = zre.shape[1]
    ore, oim = torch.empty_like(zre), torch.empty_like(zim)
    mag = torch.empty(n, dtype=torch.float64, device="cuda")
    flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
    ws = torch.empty(4 * k * n, dtype=torch.float64, device="cuda")
    for i1, roots in ((512, 4), (256, 2), (64, 1)):
        for rep in range(4):
            rc = lib.dkp_sweep(k, coeffs.data_ptr(), n, zre.data_ptr(), zim.data_ptr(), 0, i1, ore.data_ptr(),
                               oim.data_ptr(), mag.data_ptr(), flag.data_ptr(), ws.data_ptr(), roots,
                               torch.cuda.current_stream().cuda_stream)
            assert rc == 0, rc
        torch.cuda.synchronize()
        ctas = (i1 + roots - 1) // roots
        buf = (ctypes.c_ulonglong * (12 * ctas))()
        assert lib.dkp_read(buf, ctas) == 0
        t = np.frombuffer(buf, dtype=np.uint64).reshape(ctas, 12).astype(np.int64)
        rel = (t[:, :9] - t[:, :1]) / 1e3
        med = np.median(rel, axis=0)
        span = (t[:, 8].max() - t[:, 0].min()) / 1e3
        print(f"k={k} roots={i1} R={roots} CTAs={ctas}: span {span:.2f} us; start spread {(t[:,0].max()-t[:,0].min())/1e3:.2f} us")
        print("   " + "  ".join(f"{nm}={v:.2f}" for nm, v in zip(NAMES, med)), flush=True)
        if os.environ.get("DKP_DUMP"):
            np.save(os.path.join(os.environ["DKP_DUMP"], f"dkp_k{k}_n{i1}_r{roots}.npy"), t)
