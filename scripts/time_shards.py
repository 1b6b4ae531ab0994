"""Per-rank time of the bench step for a 1/G shard (what each rank computes
at G GPUs; the step has no collective): GEMM DD n=4096 / TD / QD n=2048 on
a row block of A (n/G rows, full B) and QD Horner on 2^24/G points, on one
GPU.  Projects the whole-job rate at G GPUs as total MP-ops / per-rank step
time (perfectly parallel ranks) and its efficiency vs G x (G = 1 rate)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import gen
from paper_2603_14926_b200.linalg import gemm_into
from paper_2603_14926_b200.poly import horner_into

BF = mw.Variant.BRANCH_FREE
parts = [(2, 4096), (3, 2048), (4, 2048)]
mats = {k: [torch.from_numpy(t).cuda() for t in gen.config3_gemm(k, n)] for k, n in parts}
coeffs, x = gen.config4_horner()
c4, x4 = torch.from_numpy(coeffs).cuda(), torch.from_numpy(x).cuda()
y4 = torch.empty_like(x4)
total = sum(2 * n ** 3 for _, n in parts) + 2 * x4.shape[1] * 1024


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


base = None
for G in (1, 2, 4, 8):
    row = []
    step = 0.0
    for k, n in parts:
        A, B = mats[k]
        rows = n // G
        a = A[:, :rows].contiguous()
        c = torch.empty((k, rows, n), dtype=torch.float64, device="cuda")
        ms = timed(lambda: gemm_into(a, B, c, BF))
        step += ms
        row.append(f"gemm k{k} {ms:7.2f}")
    npts = x4.shape[1] // G
    xs, ys = x4[:, :npts].contiguous(), torch.empty((4, npts), dtype=torch.float64, device="cuda")
    ms = timed(lambda: horner_into(c4, xs, ys, BF))
    step += ms
    row.append(f"horner {ms:7.2f}")
    rate = total / (step / 1e3) / 1e9
    base = base or rate
    print(f"G={G}: " + " | ".join(row) + f" | step {step:7.2f} ms -> {rate:7.1f} G MP-ops/s, "
          f"efficiency {rate / (G * base):.3f}", flush=True)
