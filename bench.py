#!/usr/bin/env python
"""Benchmark: DD/TD/QD GEMM and batched Horner on B200 vs the FP64 roofline.

Metric (BASELINE.json): "DD/TD/QD GEMM and Horner Gops/s vs FP64 FMA
roofline, 1/2/4/8 B200".  One step = one pass of the metric's workloads:
  config 3: C = A B, DD n=4096, TD n=2048, QD n=2048 (naive order, bit-exact)
  config 4: QD Horner, degree 1024, 2^24 points
Units: multi-precision ops (MP-ops; one K-word add or mul; a MAC = 2), so a
step is 2*4096^3 + 2*2048^3 + 2*2048^3 + 2*2^24*1024 MP-ops.  `value` is
the whole-job MP-op rate with inputs resident in HBM; `e2e` is the same
workload through the public Python API with host (pinned) buffers copied in
and results copied out inside the timed region.  Multi-GPU: GEMM by row
blocks of C (B replicated), Horner by point shards; no collective on the
data path ("weak"-style partition of a fixed total: scaling="strong").

The roofline denominator is the FP64 pipe rate measured live by a DFMA
microbenchmark (8 independent chains per thread, all SMs), counting one
DADD/DMUL/DFMA as one FP64 op; algorithmic FP64 ops per MAC are
DD 29, TD 96, QD 209.

--impl reference times the UNMODIFIED reference package (baseline/_ref,
installed by scripts/install_reference.sh) through its own public calls,
sharded over host processes, on a bounded sample per step; the C
restatement in oracle/ (the port) is timed beside it.  `--gpus N` without a
torchrun environment re-executes itself under torchrun with N ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# algorithmic FP64 ops per MAC (mul + add) and per MP-op
MAC_OPS = {2: 29, 3: 96, 4: 209}
GEMM_PARTS = [(2, 4096), (3, 2048), (4, 2048)]
HORNER = dict(k=4, degree=1024, npts=1 << 24)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--quick", action="store_true", help="small sizes (debug)")
    ap.add_argument("--no-secondary", action="store_true", help="skip configs 1, 2 and 5")
    ap.add_argument("--peer-exchange", "--peer-dk", dest="peer_dk", action="store_true",
                    help="N > 1: also time the dot and the DK sweep with the exchange fused into the kernel "
                         "(DotPeer / DKPeerGraph, cudaIpc peer memory); off by default until it has been run "
                         "on a multi-GPU node")
    ap.add_argument("--secondary-timeout", type=float, default=480.0,
                    help="seconds the secondary rows may take before the line is printed without the rest")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo only to exercise the multi-rank "
                         "logic where fewer GPUs than ranks exist; never for timing)")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while running."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def shard(total, rank, world):
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def mp_ops_gemm(n):
    return 2 * n**3


def fp64_ops_gemm(k, n):
    return MAC_OPS[k] * n**3


def step_mp_ops(gemm_parts, horner):
    return sum(mp_ops_gemm(n) for _, n in gemm_parts) + 2 * horner["npts"] * horner["degree"]


def measure_fp64_peak(torch, lib, dev_stream):
    """DFMA microbenchmark: ops/s of the FP64 pipe (1 DFMA = 1 op)."""
    sms = lib.mw_device_sm_count()
    blocks, threads = sms * 8, 256
    sink = torch.empty(blocks * threads, dtype=torch.float64, device="cuda")
    res = {}
    for op, name in ((0, "dfma"), (1, "dadd")):
        iters = 2000
        lib.mw_fp64_peak_kernel(op, blocks, threads, iters, sink.data_ptr(), dev_stream())
        torch.cuda.synchronize()
        # size for ~250 ms
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.mw_fp64_peak_kernel(op, blocks, threads, iters, sink.data_ptr(), dev_stream())
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        iters = max(1, int(iters * 0.25 / max(t, 1e-6)))
        best = 0.0
        for _ in range(3):
            e0.record()
            lib.mw_fp64_peak_kernel(op, blocks, threads, iters, sink.data_ptr(), dev_stream())
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            best = max(best, blocks * threads * iters * 64 / t)
        res[name] = best
    return res


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed
    ncu --set full capture summary (profiles/ncu_summary.json), or None."""
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        summ = json.load(open(path))
        ent = summ.get(kernel) or summ.get(kernel.replace(">", ",0>"))
        if ent is None:
            return None, None
        return int(ent["dram_bytes_per_launch"]), f"profiles/ncu_summary.json ({ent['round']}, {ent['report']})"
    except (OSError, ValueError, KeyError):
        return None, None


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2603_14926_b200 as mw
    from paper_2603_14926_b200 import _lib, gen
    from paper_2603_14926_b200.linalg import gemm_into
    from paper_2603_14926_b200.poly import horner_into

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.backend == "nccl" and torch.cuda.device_count() < world:
        print(f"bench.py: {world} NCCL ranks need {world} GPUs, {torch.cuda.device_count()} visible "
              "(use --backend gloo to exercise the multi-rank logic on fewer GPUs)", file=sys.stderr)
        sys.exit(3)
    dev_index = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev_index)
    if world > 1:
        from datetime import timedelta

        # bounded collectives: a lost peer ends the run instead of hanging it
        if args.backend == "nccl":
            # the communicator's INIT lines (nranks / rank / device) stay visible to the driver
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index), timeout=timedelta(seconds=300))
        else:
            dist.init_process_group("gloo", timeout=timedelta(seconds=300))
    lib = _lib.load()
    stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731

    gemm_parts = [(k, 512 if args.quick else n) for k, n in GEMM_PARTS]
    horner = dict(HORNER)
    if args.quick:
        horner["npts"] = 1 << 18
    BF = mw.Variant.BRANCH_FREE

    # ---- inputs: every rank draws the same seeded arrays, keeps its shard
    t_gen = time.time()
    gdata = []
    for k, n in gemm_parts:
        a, b = gen.config3_gemm(k, n)
        lo, hi = shard(n, rank, world)
        gdata.append(dict(k=k, n=n, lo=lo, hi=hi, a_host=a, b_host=b))
    coeffs, xh = gen.config4_horner(npts=horner["npts"], degree=horner["degree"], k=horner["k"])
    plo, phi = shard(horner["npts"], rank, world)
    if rank == 0:
        print(f"[bench] inputs generated in {time.time() - t_gen:.1f}s", file=sys.stderr)

    # device-resident copies (A row block, full B, C row block)
    dev = []
    for g in gdata:
        k, n, lo, hi = g["k"], g["n"], g["lo"], g["hi"]
        a = torch.from_numpy(np.ascontiguousarray(g["a_host"][:, lo:hi])).cuda()
        b = torch.from_numpy(g["b_host"]).cuda()
        c = torch.empty((k, hi - lo, n), dtype=torch.float64, device="cuda")
        dev.append((k, n, a, b, c))
    cdev = torch.from_numpy(coeffs).cuda()
    xdev = torch.from_numpy(np.ascontiguousarray(xh[:, plo:phi])).cuda()
    ydev = torch.empty_like(xdev)

    n_parts = len(dev) + 1
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(n_parts + 1)] for _ in range(args.steps)]

    def step(evs=None):
        if evs:
            evs[0].record()
        for i, (k, n, a, b, c) in enumerate(dev):
            if a.shape[1] > 0:
                gemm_into(a, b, c, BF)
            if evs:
                evs[i + 1].record()
        if xdev.shape[1] > 0:
            horner_into(cdev, xdev, ydev, BF)
        if evs:
            evs[n_parts].record()

    def barrier():
        if world > 1:
            dist.barrier()

    with ClockSampler(dev_index) as peak_clk:
        peak = measure_fp64_peak(torch, lib, stream)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev_index) as clk:
        t0.record()
        for s in range(args.steps):
            step(ev[s])
        t1.record()
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms_total = t0.elapsed_time(t1)
    part_ms = np.zeros(n_parts)
    for s in range(args.steps):
        for i in range(n_parts):
            part_ms[i] += ev[s][i].elapsed_time(ev[s][i + 1])
    part_ms /= args.steps
    my_shard = {"rank": rank, "device": dev_index, "ms_per_step": round(ms_total / args.steps, 3),
                "gemm_rows": [[g["lo"], g["hi"]] for g in gdata], "horner_points": [plo, phi]}
    rank_shards = [my_shard]
    if world > 1:
        rank_shards = [None] * world
        dist.all_gather_object(rank_shards, my_shard)
        tt = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total = float(tt.item())
    ms_step = ms_total / args.steps
    total_mp = step_mp_ops(gemm_parts, horner)
    value = total_mp / (ms_step / 1e3) / 1e9  # G MP-ops/s, whole job

    # ---- the same step with FULL QD points (low words non-zero), on record
    # beside the headline: config 4's points are plain doubles, for which the
    # Horner kernel takes its bit-identical 63-instruction product; with
    # non-zero low words it runs the reference's full 106-instruction
    # product.  Outside the timed region; 1 GPU only.
    full_pts = None
    if world == 1 and xdev.shape[1] > 0 and horner["k"] == 4:
        xfull = xdev.clone()
        xfull[1:] = xfull[0:1] * torch.tensor([2.0 ** -54, 2.0 ** -108, 2.0 ** -162], dtype=torch.float64,
                                              device=xdev.device).reshape(3, 1)
        horner_into(cdev, xfull, ydev, BF)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        horner_into(cdev, xfull, ydev, BF)
        f1.record()
        torch.cuda.synchronize()
        hf_ms = f0.elapsed_time(f1)
        step_full = float(part_ms[:-1].sum()) + hf_ms
        full_pts = {"horner_ms": round(hf_ms, 3), "ms_per_step": round(step_full, 3),
                    "value": round(total_mp / (step_full / 1e3) / 1e9, 3), "unit": "G MP-ops/s",
                    "note": "the GEMM parts as timed above + Horner at points whose low words are non-zero "
                            "(full 209-instruction step); the headline's points are the config's double-valued ones"}
        del xfull
        horner_into(cdev, xdev, ydev, BF)  # ydev back to the headline's result
        torch.cuda.synchronize()

    # ---- e2e: public API, host buffers in / results out, every step
    e2e = None
    if not args.no_e2e:
        # pinned host buffers, pre-split into row / point chunks so each chunk
        # streams in (and its result out) while the previous one computes.
        # Order: the first Horner point chunk (a small transfer) starts the
        # step, so the GEMM inputs stream in behind its compute; the GEMMs
        # follow smallest-input first (not split: a row chunk would add a
        # partial last wave per launch); the remaining Horner chunks end the
        # step, so only one small chunk's input and one small chunk's output
        # are not hidden behind compute.
        NCH_G = 1
        # Horner chunks of whole waves (resident CTAs x 256 points; the QD
        # kernel holds 8 CTAs per SM) so no chunk but the last ends on a
        # partially filled wave
        wave_pts = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count * 8 * 256
        a_pin, b_pin, c_pin = [], [], []
        for g in sorted(gdata, key=lambda g: g["k"] * g["n"] ** 2):
            lo, hi = g["lo"], g["hi"]
            cuts = np.linspace(lo, hi, NCH_G + 1).astype(int)
            a_pin.append([torch.from_numpy(np.ascontiguousarray(g["a_host"][:, r0:r1])).pin_memory()
                          for r0, r1 in zip(cuts[:-1], cuts[1:]) if r1 > r0])
            b_pin.append(torch.from_numpy(g["b_host"]).pin_memory())
            c_pin.append([torch.empty((g["k"], r1 - r0, g["n"]), dtype=torch.float64).pin_memory()
                          for r0, r1 in zip(cuts[:-1], cuts[1:]) if r1 > r0])
        pcuts = np.unique(np.r_[np.arange(plo, phi, 4 * wave_pts), phi]).astype(int)
        x_pin = [torch.from_numpy(np.ascontiguousarray(xh[:, p0:p1])).pin_memory()
                 for p0, p1 in zip(pcuts[:-1], pcuts[1:]) if p1 > p0]
        y_pin = [torch.empty_like(t).pin_memory() for t in x_pin]
        c_pin_coeffs = torch.from_numpy(coeffs).pin_memory()
        h2d = (sum(t.numel() * 8 for ts in a_pin for t in ts) + sum(t.numel() * 8 for t in b_pin)
               + sum(t.numel() * 8 for t in x_pin) + c_pin_coeffs.numel() * 8)
        d2h = sum(t.numel() * 8 for ts in c_pin for t in ts) + sum(t.numel() * 8 for t in y_pin)
        plan = mw.MatMulPlan(scheme="naive", variant=BF)
        h2d_stream = torch.cuda.Stream()
        d2h_stream = torch.cuda.Stream()

        def e2e_step():
            """Public API end to end (MWMatrix / matmul / MWPolynomial /
            horner_eval_batched) over pinned host buffers: every input chunk
            is copied H2D on a copy stream, computed on the current stream as
            soon as it lands, and its result copied D2H on a second copy stream
            behind it, so transfers overlap compute."""
            cur = torch.cuda.current_stream()
            # no wait on `cur` here: the next step's inputs may stream in
            # while this step still computes (the device buffers are fresh
            # allocations, released to the allocator only after the compute
            # stream's use: record_stream below)

            def stage(host):
                dev_t = host.to("cuda", non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
                return dev_t, ev

            staged = []
            with torch.cuda.stream(h2d_stream):
                cf = c_pin_coeffs.to("cuda", non_blocking=True)
                xs = [stage(x_pin[0])] if x_pin else []
                for bp, chunks in zip(b_pin, a_pin):
                    B = bp.to("cuda", non_blocking=True)
                    staged.append((B, [stage(ap) for ap in chunks]))
                xs += [stage(xp) for xp in x_pin[1:]]

            def drain(dev_t, host_t):
                d2h_stream.wait_stream(cur)
                with torch.cuda.stream(d2h_stream):
                    host_t.copy_(dev_t, non_blocking=True)
                dev_t.record_stream(d2h_stream)

            P = None

            def horner_chunk(i):
                nonlocal P
                X, ev = xs[i]
                cur.wait_event(ev)
                X.record_stream(cur)
                if P is None:
                    cf.record_stream(cur)
                    P = mw.MWPolynomial(cf)
                drain(mw.horner_eval_batched(P, mw.LaneBatch(X), BF).planes, y_pin[i])

            if xs:
                horner_chunk(0)
            for (B, parts), cps in zip(staged, c_pin):
                Bm = None
                for (A, ev), cp in zip(parts, cps):
                    cur.wait_event(ev)
                    A.record_stream(cur)
                    if Bm is None:
                        B.record_stream(cur)
                        Bm = mw.MWMatrix(B)
                    drain(mw.matmul(mw.MWMatrix(A), Bm, plan).planes, cp)
            for i in range(1, len(xs)):
                horner_chunk(i)
            cur.wait_stream(d2h_stream)

        for _ in range(max(1, min(args.warmup, 2))):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": round(total_mp / (ems / args.steps / 1e3) / 1e9, 3), "unit": "G MP-ops/s",
               "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
               "ms_per_step": round(ems / args.steps, 3)}

    # ---- roofline of the dominant kernel (largest share of the step)
    parts = []
    for i, (k, n, a, b, c) in enumerate(dev):
        rows = a.shape[1]
        ops = MAC_OPS[k] * rows * n * n
        parts.append(dict(name=f"gemm_{['', '', 'dd', 'td', 'qd'][k]}_n{n}", kernel=f"gemm_kernel<{k},1,0>",
                          ms=part_ms[i], fp64_ops=ops,
                          mp_ops=2 * rows * n * n))
    hp = phi - plo
    # config 4's points are plain doubles (x, 0, 0, 0): the kernel's product
    # for such points issues 63 FP64 instructions instead of qw_mul_bf's 106
    # (the operations +0 low words determine are removed; bit-identical,
    # csrc/mw_eft.cuh qd_mul_bf_d), so a step EXECUTES 63 + 103 = 166, not
    # 209.  The roofline counts what is executed; MP-ops count the K-word
    # operations of the reference sequence (one mul + one add per step).
    horner_step_ops = (63 + ADD_OPS[4]) if horner["k"] == 4 else MAC_OPS[horner["k"]]
    parts.append(dict(name=f"horner_qd_deg{horner['degree']}_pts{horner['npts']}", kernel="horner_kernel<4,1>",
                      ms=part_ms[-1],
                      fp64_ops=horner_step_ops * hp * horner["degree"], mp_ops=2 * hp * horner["degree"],
                      fp64_ops_reference=MAC_OPS[horner["k"]] * hp * horner["degree"]))
    for p in parts:
        p["fp64_tops"] = p["fp64_ops"] / (p["ms"] / 1e3) / 1e12 if p["ms"] > 0 else 0.0
        p["frac_of_fp64_peak"] = p["fp64_tops"] * 1e12 / peak["dfma"]
        p["gmpops"] = p["mp_ops"] / (p["ms"] / 1e3) / 1e9 if p["ms"] > 0 else 0.0
    for p, (k, n, a, b, c) in zip(parts, dev):
        p["alg_bytes"] = (a.numel() + b.numel() + c.numel()) * 8
    parts[-1]["alg_bytes"] = (xdev.numel() + ydev.numel() + cdev.numel()) * 8
    dom = max(parts, key=lambda p: p["ms"])
    peak_t = peak["dfma"] / 1e12
    roofline = {
        "bound": "fp64", "kernel": dom["name"],
        "achieved": round(dom["fp64_tops"], 3), "peak": round(peak_t, 3),
        "unit": "T FP64-op/s (DADD/DMUL/DFMA = 1 op)",
        "frac": round(dom["fp64_tops"] / peak_t, 4),
        "traffic": ncu_traffic(dom["kernel"])[0],
        "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
        "traffic_source": ncu_traffic(dom["kernel"])[1],
        "algorithmic_bytes": dom["alg_bytes"],
        "peak_source": "measured live: DFMA microbenchmark, 8 chains/thread, all SMs (mw_fp64_peak_kernel)",
    }
    if "fp64_ops_reference" in dom:
        roofline["ops_note"] = (
            "achieved counts the FP64 instructions the kernel issues: 166 per Horner step for double-valued QD "
            "points (63-instruction product qd_mul_bf_d + 103-instruction add; bit-identical with the reference's "
            "106 + 103 = 209, whose rate would be "
            f"{dom['fp64_ops_reference'] / (dom['ms'] / 1e3) / 1e12:.3f} T/s)")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample(gemm_parts, horner)

    sec = {}
    line = {
        "metric": "DD/TD/QD GEMM and Horner Gops/s vs FP64 FMA roofline, 1/2/4/8 B200",
        "value": round(value, 3), "unit": "G MP-ops/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64 (DD/TD/QD multi-word)", "data": "synthetic (seeded, SURVEY §8(d) G_K)",
        "config": {
            "workload": "config3 GEMM DD n4096 + TD n2048 + QD n2048, config4 QD Horner deg1024 x 2^24 pts",
            "gemm": [f"k{k} n{n}" for k, n in gemm_parts], "horner": horner,
            "parallelism": f"rows/points sharded over {world} GPU(s), no collective",
            "ranks": world, "backend": args.backend if world > 1 else None,
            "shards": rank_shards,
            "shared_gpus": (world > torch.cuda.device_count()) or None,
            "l2": "inputs larger than L2 (GEMM DD A+B 537 MB, Horner x 537 MB); no flush",
            "bit_exact": "GEMM naive order and Horner per point, vs reference",
            "horner_points": "double-valued QD points (x, 0, 0, 0) as SURVEY 8(d) config 4 specifies; the kernel "
                             "takes its bit-identical 63-instruction product for them (secondary."
                             "paper_comparisons.horner_qd_deg1024_pts2p20_full_qd_points times full QD points)",
        },
        "parts": [{"name": p["name"], "ms": round(p["ms"], 3), "G_MPops": round(p["gmpops"], 2),
                   "fp64_Tops": round(p["fp64_tops"], 3), "frac": round(p["frac_of_fp64_peak"], 4)}
                  for p in parts],
        "fp64_peak_measured": {"dfma_Tops": round(peak["dfma"] / 1e12, 3), "dadd_Tops": round(peak["dadd"] / 1e12, 3),
                               "method": "8 independent DFMA / DADD chains per thread, 8 CTAs x 256 threads per SM, "
                                         "~0.75 s per op (best of 3)",
                               "clocks": peak_clk.summary()},
        "roofline": roofline,
        "full_qd_points": full_pts,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": args.steps * (len(dev) + 1),
        "clocks": clk.summary(),
        "secondary": sec if not args.no_secondary else None,
    }

    # The headline is complete here.  The secondary rows run under a
    # watchdog: if they have not finished in time (a stuck collective at
    # N > 1, say), the line is printed with what was measured and the
    # process exits -- the headline is never lost to a secondary row.
    import threading

    printed = threading.Event()

    def emit(note=None):
        if printed.is_set():
            return
        printed.set()
        if note:
            line["secondary_note"] = note
        if rank == 0:
            print(json.dumps(line), flush=True)

    def on_timeout():
        emit(f"secondary rows stopped by the {args.secondary_timeout:.0f} s watchdog")
        sys.stdout.flush()
        os._exit(0)

    if not args.no_secondary:
        dog = threading.Timer(args.secondary_timeout, on_timeout)
        dog.daemon = True
        dog.start()
        try:
            secondary(args, torch, dist, mw, world, rank, peak, out=sec)
        except Exception as e:  # reported in the line; the headline stands on its own
            sec["error"] = f"{type(e).__name__}: {e}"[:300]
        dog.cancel()
    emit()
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------ secondary configs 1, 2, 5
ADD_OPS = {2: 20, 3: 57, 4: 103}
MUL_OPS = {2: 9, 3: 39, 4: 106}


def secondary(args, torch, dist, mw, world, rank, peak, out=None):
    """The other §8 rows, measured on the same run (not the headline):
    config 1 dot/axpy (DD n=65536), config 2 GEMV (TD/QD 2048^2),
    config 5 DK (TD/QD n=512, 200 sweeps; roots sharded + one all-gather
    per sweep when N > 1).  Device time via CUDA events, max over ranks."""
    from paper_2603_14926_b200 import blas, gen
    from paper_2603_14926_b200 import dist as mwdist
    from paper_2603_14926_b200.roots import INT32_MAX, sweep_into

    BF = mw.Variant.BRANCH_FREE
    hbm = 6538.9e9
    try:
        hbm = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
    except (OSError, ValueError, KeyError):
        pass
    out = {} if out is None else out  # filled in place: a watchdog may print it early
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > L2 (126 MB)

    def timed(fn, reps, flush_l2=False):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        for e0, e1 in evs:
            if flush_l2:
                flush.fill_(1)
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def timed_graph(fn, calls=100, reps=10):
        """Per-call device time of `calls` back-to-back calls captured in one
        CUDA graph (removes host launch overhead); median over replays."""
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(calls):
                fn()
        g.replay()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for e0, e1 in evs:
            e0.record()
            g.replay()
            e1.record()
        torch.cuda.synchronize()
        ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs) / calls
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    flush_rd = None

    def timed_graph_flushed(fn, reps=20, clean=False):
        """Device time of ONE call (captured alone in a CUDA graph, so the
        host-side API cost cannot leave the GPU idle inside the timed
        region), L2 flushed before every replay; median over replays.
        The flush writes a 256 MB buffer, which leaves L2 full of DIRTY
        lines: the timed call then pays their write-back as it streams its
        operand in.  clean=True also reads a second 256 MB buffer after
        the write, so the call starts from a cold but clean L2 (the state
        ncu's cache control leaves)."""
        nonlocal flush_rd
        if clean and flush_rd is None:
            flush_rd = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for e0, e1 in evs:
            flush.fill_(1)
            if clean:
                flush_rd.view(torch.int64).sum()  # reads 256 MB: clean lines replace the dirty ones
            e0.record()
            g.replay()
            e1.record()
        torch.cuda.synchronize()
        ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # ---- config 1: dot and axpy, DD n = 65536 (2 MiB: L2-resident, launch-bound)
    x, y, alpha = gen.config1_dot()
    n1 = x.shape[1]
    lo, hi = mwdist.aligned_shard_range(n1, rank, world, mwdist.DOT_PARTIAL_SPAN)
    X, Y = mw.LaneBatch(x), mw.LaneBatch(y)
    ms_dot_graph = ms_axpy_graph = None
    if world == 1:
        dres = torch.empty(2, dtype=torch.float64, device="cuda")
        ms_dot = timed(lambda: blas.dot_tensor(X, Y, BF, out=dres), 200)
        ms_dot_graph = timed_graph(lambda: blas.dot_tensor(X, Y, BF, out=dres))
    else:
        be = mwdist.gpu_dot_backend(BF)
        ms_dot = timed(lambda: mwdist.dot_allgather(X.planes, Y.planes, be), 50)
    # the all-gather-then-sum fused into one kernel per rank (DotPeer)
    peer_dot = None
    if world == 1 or (args.backend == "nccl" and args.peer_dk):
        try:
            dp = mwdist.DotPeer(2, n1, BF, device=X.planes.device)
            pres = torch.empty(2, dtype=torch.float64, device="cuda")
            ms_p = timed(lambda: dp(X.planes, Y.planes, out=pres), 200)
            ms_pg = timed_graph(lambda: dp(X.planes, Y.planes, out=pres)) if world == 1 else None
            dp.check()
            dp.close()
            peer_dot = {"us_per_call": round(ms_p * 1e3, 2),
                        "us_per_call_graph": None if ms_pg is None else round(ms_pg * 1e3, 2)}
        except Exception as e:  # reported, never fatal to the bench line
            peer_dot = {"error": f"{type(e).__name__}: {e}"[:200]}
    Xs, Ys = mw.LaneBatch(x[:, lo:hi]), mw.LaneBatch(y[:, lo:hi])
    ms_axpy = timed(lambda: blas.axpy_(tuple(alpha), Xs, Ys, BF), 200)
    if world == 1:
        ms_axpy_graph = timed_graph(lambda: blas.axpy_(tuple(alpha), Xs, Ys, BF))
    def host_us(fn, calls=2000):
        """Host cost of the public API per call: wall time of back-to-back
        calls (the device work queues behind them), synchronised at the end."""
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(calls):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / calls * 1e6

    if world == 1:
        host_dot = host_us(lambda: blas.dot_tensor(X, Y, BF, out=dres))
        host_axpy = host_us(lambda: blas.axpy_(tuple(alpha), Xs, Ys, BF))
    else:
        host_dot = host_axpy = None
    out["config1_dot_dd_n65536"] = {
        "host_us_per_call": None if host_dot is None else round(host_dot, 2),
        "us_per_call": round(ms_dot * 1e3, 2), "G_MPops": round(2 * n1 / (ms_dot / 1e3) / 1e9, 3),
        "us_per_call_graph": None if ms_dot_graph is None else round(ms_dot_graph * 1e3, 2),
        "G_MPops_graph": None if ms_dot_graph is None else round(2 * n1 / (ms_dot_graph / 1e3) / 1e9, 3),
        "hbm_frac": round(2 * 2 * n1 * 8 / (ms_dot / 1e3) / hbm, 4),
        "order": "tree (256 strided partials per 4096-element block + pairwise tree)" + (", all-gather-then-sum over ranks" if world > 1 else ""),
        "note": "2 MiB input is L2-resident and launch-bound; hbm_frac is bytes/time vs HBM copy peak; "
                "us_per_call = one eager API call between CUDA events (launch latency included), "
                "host_us_per_call = host cost per call issued back to back (PyTorch extension path)",
        "fused_peer_exchange": peer_dot}
    out["config1_axpy_dd_n65536"] = {
        "host_us_per_call": None if host_axpy is None else round(host_axpy, 2),
        "us_per_call": round(ms_axpy * 1e3, 2), "G_MPops": round(2 * n1 / (ms_axpy / 1e3) / 1e9, 3),
        "us_per_call_graph": None if ms_axpy_graph is None else round(ms_axpy_graph * 1e3, 2),
        "hbm_frac": round(3 * 2 * (hi - lo) * 8 * world / (ms_axpy / 1e3) / hbm, 4)}

    # ---- config 1's kernels at a streaming size (DD, n = 2^26: 1 GiB per
    # operand, far above L2), where dot and axpy are HBM-bound: GB/s vs the
    # HBM peak.  Timing-only inputs drawn on the device (BF cost is
    # data-independent).
    if world == 1 and not args.quick:
        nbig = 1 << 26
        gdev = torch.Generator(device="cuda")
        gdev.manual_seed(0)

        def dd_planes():
            t = torch.empty((2, nbig), dtype=torch.float64, device="cuda")
            t[0].uniform_(-1, 1, generator=gdev)
            t[1].uniform_(-1, 1, generator=gdev)
            t[1].mul_(t[0]).mul_(2.0 ** -53)
            return t

        Xb, Yb = mw.LaneBatch(dd_planes()), mw.LaneBatch(dd_planes())
        dres_b = torch.empty(2, dtype=torch.float64, device="cuda")
        ms_dot_b = timed(lambda: blas.dot_tensor(Xb, Yb, BF, out=dres_b), 10, flush_l2=True)
        ms_axpy_b = timed(lambda: blas.axpy_(tuple(alpha), Xb, Yb, BF), 10, flush_l2=True)
        out["config1_kernels_dd_n2p26_stream"] = {
            "dot_us": round(ms_dot_b * 1e3, 1),
            "dot_GBps": round(32 * nbig / (ms_dot_b / 1e3) / 1e9, 1),
            "dot_hbm_frac": round(32 * nbig / (ms_dot_b / 1e3) / hbm, 4),
            "axpy_us": round(ms_axpy_b * 1e3, 1),
            "axpy_GBps": round(48 * nbig / (ms_axpy_b / 1e3) / 1e9, 1),
            "axpy_hbm_frac": round(48 * nbig / (ms_axpy_b / 1e3) / hbm, 4),
            "bytes": {"dot": 32 * nbig, "axpy": 48 * nbig},
            "l2": "flushed before each call", "note": "same kernels as config 1 at n = 2^26 (HBM-bound regime)"}
        del Xb, Yb

    # ---- config 2: GEMV TD / QD 2048 x 2048, row blocks per rank, L2 flushed
    for k in (3, 4):
        a, xv = gen.config2_gemv(k)
        m = a.shape[1]
        rlo, rhi = mwdist.shard_range(m, rank, world)
        A, XV = mw.MWMatrix(a), mw.LaneBatch(xv)
        yb = torch.empty((k, rhi - rlo), dtype=torch.float64, device="cuda")
        ms_eager = timed(lambda: blas.gemv(A, XV, BF, "tree", rlo, rhi, out=yb), 20, flush_l2=True)
        ms = timed_graph_flushed(lambda: blas.gemv(A, XV, BF, "tree", rlo, rhi, out=yb))
        ms_clean = timed_graph_flushed(lambda: blas.gemv(A, XV, BF, "tree", rlo, rhi, out=yb), clean=True)
        ms_warm = timed_graph(lambda: blas.gemv(A, XV, BF, "tree", rlo, rhi, out=yb), calls=20)
        fp = MAC_OPS[k] * m * m
        out[f"config2_gemv_{'td' if k == 3 else 'qd'}_n2048"] = {
            "ms": round(ms, 4), "G_MPops": round(2 * m * m / (ms / 1e3) / 1e9, 2),
            "fp64_frac": round(fp / (ms / 1e3) / peak["dfma"] / world, 4),
            "hbm_GBps": round(k * m * m * 8 / (ms / 1e3) / 1e9, 1), "order": "tree (128 partials per row)",
            "fp64_bound_us": round(fp / peak["dfma"] / world * 1e6, 1),
            "hbm_bound_us": round(k * m * m * 8 / hbm / world * 1e6, 1),
            "l2": "flushed before each call",
            "timing": "one call per CUDA-graph replay (device time, no host API gap); ms_eager = the same call launched eagerly through the Python API",
            "ms_eager": round(ms_eager, 4),
            "ms_clean_flush": round(ms_clean, 4),
            "ms_back_to_back": round(ms_warm, 4),
            "flush_note": "ms: after a 256 MB write (dirty L2: the call pays the write-backs); ms_clean_flush: "
                          "write then a 256 MB read (cold, clean L2); ms_back_to_back: 20 calls per graph"}
        del A

    # ---- config 3 with the reference's benchmark scheme (Strassen; 1 GPU):
    # effective rate = 2 n^3 / time (fewer MACs are executed: not comparable
    # to the bit-exact naive headline; the reference's own Strassen order)
    if world == 1:
        for k, n in GEMM_PARTS if not args.quick else ():
            a, b = gen.config3_gemm(k, n)
            A, B = mw.MWMatrix(a), mw.MWMatrix(b)
            cut = 128 if k < 4 else 64
            plan = mw.MatMulPlan(scheme="strassen", variant=BF, strassen_cutoff=cut)
            ms = timed(lambda: mw.matmul(A, B, plan), 2)
            lv = 0
            m_ = n
            while m_ > cut:
                lv, m_ = lv + 1, m_ // 2
            out[f"config3_strassen_{['', '', 'dd', 'td', 'qd'][k]}_n{n}"] = {
                "ms": round(ms, 2), "cutoff": cut, "levels": lv,
                "G_MPops_effective": round(2 * n ** 3 / (ms / 1e3) / 1e9, 1),
                "mac_fraction_executed": round((7 / 8) ** lv, 4),
                "note": "bit-exact with the reference's matmul(scheme='strassen') at this cutoff"}
            del A, B

    # ---- the paper's comparisons on the GPU (1 GPU): branch-free vs
    # Standard (renormalising, per-lane branches) kernels, and Horner vs
    # Estrin (§4.1).  Same generators, smaller sizes; both variants
    # are bit-exact with the reference's own kernels.
    if world == 1 and not args.quick:
        from paper_2603_14926_b200.linalg import gemm_into
        from paper_2603_14926_b200.poly import horner_into

        STD = mw.Variant.STANDARD
        cmp = {}
        for k in (2, 3, 4):
            a, b = gen.config3_gemm(k, 1024)
            A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
            C = torch.empty_like(A)
            ms_bf = timed(lambda: gemm_into(A, B, C, BF), 3)
            ms_std = timed(lambda: gemm_into(A, B, C, STD), 3)
            cmp[f"gemm_{['', '', 'dd', 'td', 'qd'][k]}_n1024"] = {
                "bf_ms": round(ms_bf, 3), "std_ms": round(ms_std, 3), "bf_speedup": round(ms_std / ms_bf, 3)}
            del A, B, C
        coeffs4, x4 = gen.config4_horner(npts=1 << 20)
        c4, xd4 = torch.from_numpy(coeffs4).cuda(), torch.from_numpy(x4).cuda()
        y4 = torch.empty_like(xd4)
        ms_bf = timed(lambda: horner_into(c4, xd4, y4, BF), 3)
        ms_std = timed(lambda: horner_into(c4, xd4, y4, STD), 3)
        cmp["horner_qd_deg1024_pts2p20"] = {
            "bf_ms": round(ms_bf, 3), "std_ms": round(ms_std, 3), "bf_speedup": round(ms_std / ms_bf, 3)}
        # the same Horner at points with non-zero low words (full QD points):
        # the kernel then issues the reference's 209 FP64 instructions per
        # step instead of the 166 of the double-point product the headline's
        # config 4 takes -- reported so both rates are on record
        xf = gen.g_k(np.random.default_rng(44), 4, 1 << 20)
        xfd = torch.from_numpy(xf).cuda()
        ms_full = timed(lambda: horner_into(c4, xfd, y4, BF), 3)
        hops = (1 << 20) * (c4.shape[1] - 1)
        cmp["horner_qd_deg1024_pts2p20_full_qd_points"] = {
            "ms": round(ms_full, 3), "ms_double_points": round(ms_bf, 3),
            "G_MPops": round(2 * hops / (ms_full / 1e3) / 1e9, 1),
            "fp64_frac": round(MAC_OPS[4] * hops / (ms_full / 1e3) / peak["dfma"], 4),
            "fp64_frac_double_points": round((63 + ADD_OPS[4]) * hops / (ms_bf / 1e3) / peak["dfma"], 4),
            "note": "full product 106 + add 103 = 209 FP64 instructions per step; double-valued points 63 + 103 = 166 (bit-identical)"}
        del xfd
        P4, X4 = mw.MWPolynomial(c4), mw.LaneBatch(xd4)
        ms_est = timed(lambda: mw.estrin_eval_batched(P4, X4, BF), 3)
        npts4, deg4 = xd4.shape[1], c4.shape[1] - 1
        lv = max(1, (deg4).bit_length())  # levels after padding deg+1 coefficients to 2^lv
        est_mp = (2 * ((1 << lv) - 1) + (lv - 1)) * npts4  # every padded node: mul + add; squarings
        hor_mp = 2 * deg4 * npts4
        cmp["estrin_vs_horner_qd_deg1024_pts2p20"] = {
            "horner_ms": round(ms_bf, 3), "estrin_ms": round(ms_est, 3),
            "estrin_over_horner": round(ms_est / ms_bf, 3),
            "horner_G_MPops": round(hor_mp / (ms_bf / 1e3) / 1e9, 1),
            "estrin_G_MPops": round(est_mp / (ms_est / 1e3) / 1e9, 1),
            "note": "the reference's Estrin zero-pads 1025 coefficients to 2048 and evaluates every node: 2x Horner's K-word ops per point; per-op rates compare the kernels"}
        # the paper's root-finding benchmark: Durand-Kerner
        # on the Chebyshev test polynomial of degree 64, to convergence from
        # the Aberth start, NoBF (Standard) vs BF; the reference order (bit-
        # exact with mwfloat's dk_solve, sweep count included) and the tree order
        from paper_2603_14926_b200 import roots as mwroots

        for k in (3, 4):
            q = mwroots.chebyshev_coeffs(64, k)
            row = {}
            for vname, var in (("std", STD), ("bf", BF)):
                for order, exact in (("exact", True), ("tree", False)):
                    st0 = mwroots.aberth_init(q, var)
                    mwroots.dk_solve(q, var, state=st0, exact_order=exact)  # warm-up
                    torch.cuda.synchronize()
                    ts = []
                    for _ in range(3):
                        t = time.perf_counter()
                        _, iters = mwroots.dk_solve(q, var, state=st0, exact_order=exact)
                        torch.cuda.synchronize()
                        ts.append(time.perf_counter() - t)
                    row[f"{vname}_{order}_ms"] = round(statistics.median(ts) * 1e3, 2)
                    row[f"{vname}_{order}_sweeps"] = iters
            row["paper_epyc_s"] = {"nobf": 0.306 if k == 3 else 0.989, "bf_simd": 0.156 if k == 3 else 0.415}
            row["note"] = ("wall time of dk_solve from the Aberth start (host loop over device sweeps, one read-back "
                           "per chunk); paper: EPYC 9354P, its own C library (PAPER.md:443-447)")
            cmp[f"dk_chebyshev_n64_{'td' if k == 3 else 'qd'}"] = row
        out["paper_comparisons"] = cmp
        del c4, xd4, y4, P4, X4

    # ---- config 5: DK, n = 512, 200 sweeps (near-root init)
    for k in (3, 4):
        coeffs = torch.from_numpy(gen.config5_poly(k)).cuda()
        zre0, zim0 = (torch.from_numpy(t).cuda() for t in gen.config5_init(k))
        n5 = zre0.shape[1]
        mp_sweep = n5 * (20 * n5 + 31)
        fp_sweep = n5 * (n5 * (6 * MUL_OPS[k] + 14 * ADD_OPS[k]) + 20 * MUL_OPS[k] + 11 * ADD_OPS[k])
        # the tree order executes fewer FP64 instructions per (i, j) than the
        # reference's op sequence: its complex products are 4 mul + 2 add
        # instead of 3 mul + 5 add and the Horner step adds the real
        # coefficient to the real part only -- 8 mul + 7 add per pair
        fp_sweep_tree = n5 * (n5 * (8 * MUL_OPS[k] + 7 * ADD_OPS[k]) + 20 * MUL_OPS[k] + 11 * ADD_OPS[k])
        for exact in (False, True):
            sweeps = 200
            if world == 1:
                from paper_2603_14926_b200.roots import DKSweepGraph

                g = DKSweepGraph(mw.MonicPoly(coeffs), mw.RootState(re=zre0, im=zim0), sweeps, BF, exact_order=exact)
                ms = timed(g.replay, 3)
                g.result()  # raises on a collision
            elif args.backend == "nccl":
                g = mwdist.DKShardedGraph(coeffs, zre0, zim0, sweeps, BF, exact_order=exact)
                ms = timed(g.replay, 3)  # 200 x (sweep kernel + NCCL all-gather) in one graph
            else:
                ms = timed(lambda: mwdist.dk_sweeps_sharded(coeffs, zre0, zim0, sweeps, BF, exact_order=exact), 2)
            # the exchange fused into the sweep kernel (peer stores over
            # NVLink + completion slots; at N = 1 this times the protocol's
            # overhead: self stores, ticket, slot publication and wait)
            peer = None
            if world == 1 or (args.backend == "nccl" and args.peer_dk):
                try:
                    pg = mwdist.DKPeerGraph(coeffs, zre0, zim0, sweeps, BF, exact_order=exact)
                    ms_p = timed(pg.replay, 3)
                    pg.result()
                    pg.close()
                    peer = {"ms_200_sweeps": round(ms_p, 3), "us_per_sweep": round(ms_p * 1e3 / sweeps, 2)}
                except Exception as e:  # reported, never fatal to the bench line
                    peer = {"error": f"{type(e).__name__}: {e}"[:200]}
            out[f"config5_dk_{'td' if k == 3 else 'qd'}_n512_{'exact' if exact else 'tree'}"] = {
                "ms_200_sweeps": round(ms, 3), "us_per_sweep": round(ms * 1e3 / sweeps, 2),
                "G_MPops": round(mp_sweep * sweeps / (ms / 1e3) / 1e9, 3),
                "fp64_frac": round(fp_sweep * sweeps / (ms / 1e3) / peak["dfma"] / world, 4),
                "fp64_frac_executed": round((fp_sweep if exact else fp_sweep_tree) * sweeps / (ms / 1e3)
                                            / peak["dfma"] / world, 4),
                "ops_note": ("fp64_frac counts the reference's op sequence per sweep (6 mul + 14 add per (i, j), "
                             "SURVEY 8(d)); fp64_frac_executed what this order issues"
                             + ("" if exact else " (8 mul + 7 add per (i, j): four-multiplication complex products)")),
                "collective": ("all_gather of (re, im) K-planes per sweep"
                               + (", sweeps + NCCL captured in one CUDA graph" if args.backend == "nccl" else ""))
                if world > 1 else None,
                "fused_peer_exchange": peer}
    return out


# ---------------------------------------------------------- CPU baseline
def cpu_sample(gemm_parts, horner, budget_rows=None, horner_pts=1 << 19):
    """Reference algorithm (C restatement, oracle/) on all host threads over
    a bounded sample: GEMM rows (per K) and Horner points.  Returns the
    cpu_baseline dict in the same unit (G MP-ops/s)."""
    import oracle
    from paper_2603_14926_b200 import gen

    oracle.set_threads(os.cpu_count() or 1)  # torchrun exports OMP_NUM_THREADS=1: use every host thread
    threads = oracle.max_threads()
    sample_rows = {2: 64, 3: 64, 4: 32} if budget_rows is None else budget_rows
    tot_mp = 0.0
    tot_s = 0.0
    desc = []
    for k, n in gemm_parts:
        a, b = gen.config3_gemm(k, n)
        r = min(sample_rows[k], n)
        t = time.perf_counter()
        oracle.gemm(a[:, :r], b, "bf")
        dt = time.perf_counter() - t
        tot_mp += 2 * n**3
        tot_s += dt * (n / r)  # per-row work is uniform: scale to the full matrix
        desc.append(f"gemm k{k} n{n}: {r} rows in {dt:.2f}s")
    coeffs, x = gen.config4_horner(npts=horner["npts"], degree=horner["degree"], k=horner["k"])
    pts = min(horner_pts, horner["npts"])
    t = time.perf_counter()
    oracle.horner(coeffs, x[:, :pts], "bf")
    dt = time.perf_counter() - t
    desc.append(f"horner: {pts} pts in {dt:.2f}s")
    tot_s += dt * (horner["npts"] / pts)
    tot_mp += 2 * horner["npts"] * horner["degree"]
    return {"value": round(tot_mp / tot_s / 1e9, 4), "unit": "G MP-ops/s", "cores": threads, "kind": "port",
            **host_description(),
            "sample": "; ".join(desc) + " -- extrapolated linearly to the full step (uniform work per row/point)",
            "seconds_per_step_extrapolated": round(tot_s, 2)}


# ------------------------------------------- the unmodified reference (CPU)
REF_DIR = os.path.join(REPO, "baseline", "_ref")
_REF_DATA = {}


def host_description():
    """CPU model (the reference's cli.hardware_tag recipe, cli.py:72-82),
    logical and physical core counts."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.lower().startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    phys = None
    try:
        import psutil

        phys = psutil.cpu_count(logical=False)
    except Exception:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "physical_cores": phys}


def _ref_import():
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import mwfloat  # noqa: F401  (baseline/_ref: the unmodified reference package)
    from mwfloat import batch, linalg
    from mwfloat.multiword import Variant

    return batch, linalg, Variant


def _ref_gemm_rows(job):
    """linalg.matmul(A[r0:r1], B, naive, bf) -- the reference's own public
    call on one row block (its partition, linalg.py:352-365), one process."""
    k, r0, r1 = job
    _, linalg, Variant = _ref_import()
    a, b = _REF_DATA[("gemm", k)]
    t = time.perf_counter()
    linalg.matmul(linalg.MWMatrix(tuple(np.ascontiguousarray(a[c, r0:r1]) for c in range(k))),
                  linalg.MWMatrix(tuple(b[c] for c in range(k))),
                  linalg.MatMulPlan(scheme="naive", variant="bf"))
    return time.perf_counter() - t


def _ref_horner_chunk(job):
    """Lane-batched Horner over the reference's own dispatch table
    (_BATCH_MUL/_BATCH_ADD[(4, BF)], batch.py:178-194): bitwise equal to
    poly.horner_eval per point (poly.py:89-96)."""
    p0, p1 = job
    batch, _, Variant = _ref_import()
    coeffs, x = _REF_DATA["horner"]
    k = coeffs.shape[0]
    add, mul = batch._BATCH_ADD[k, Variant.BRANCH_FREE], batch._BATCH_MUL[k, Variant.BRANCH_FREE]
    xs = tuple(np.ascontiguousarray(x[c, p0:p1]) for c in range(k))
    t = time.perf_counter()
    deg = coeffs.shape[1] - 1
    acc = tuple(np.full(p1 - p0, coeffs[c, deg]) for c in range(k))
    for i in range(deg - 1, -1, -1):
        acc = add(mul(acc, xs), tuple(float(coeffs[c, i]) for c in range(k)))
    return time.perf_counter() - t


def reference_sample(gemm_parts, horner, procs, rows_per_proc, pts_per_proc, pool):
    """One bounded sample of the step on the unmodified reference, sharded
    across `procs` processes: per GEMM, `procs` row blocks
    of rows_per_proc[k] rows; Horner, `procs` chunks of pts_per_proc points.
    Returns (measured wall seconds, MP-ops done, extrapolated full-step
    seconds, description)."""
    wall = mp = full_s = 0.0
    desc = []
    for k, n in gemm_parts:
        r = rows_per_proc[k]
        jobs = [(k, i * r, (i + 1) * r) for i in range(procs) if (i + 1) * r <= n]
        t = time.perf_counter()
        pool.map(_ref_gemm_rows, jobs)
        dt = time.perf_counter() - t
        done = 2 * len(jobs) * r * n * n
        wall += dt
        mp += done
        full_s += dt * (2 * n**3) / done
        desc.append(f"gemm k{k} n{n}: {len(jobs) * r} rows in {dt:.2f}s")
    c = pts_per_proc
    jobs = [(i * c, (i + 1) * c) for i in range(procs)]
    t = time.perf_counter()
    pool.map(_ref_horner_chunk, jobs)
    dt = time.perf_counter() - t
    done = 2 * len(jobs) * c * horner["degree"]
    wall += dt
    mp += done
    full_s += dt * (2 * horner["npts"] * horner["degree"]) / done
    desc.append(f"horner: {len(jobs) * c} pts in {dt:.2f}s")
    return wall, mp, full_s, "; ".join(desc)


def run_reference(args):
    """The reference arm: the UNMODIFIED reference package (baseline/_ref,
    scripts/install_reference.sh) through its own public calls, sharded
    over processes on the host cores, each step a bounded sample of the
    workload (rates extrapolate linearly: uniform work per row / point).
    Under torchrun only rank 0 runs.  The C restatement (oracle/, the
    port) is timed beside it and reported under `port`."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp_

    from paper_2603_14926_b200 import gen

    gemm_parts = [(k, 512 if args.quick else n) for k, n in GEMM_PARTS]
    horner = dict(HORNER)
    if args.quick:
        horner["npts"] = 1 << 16
    host = host_description()
    procs = max(1, min(os.cpu_count() or 1, 64))
    have_ref = os.path.exists(os.path.join(REF_DIR, "mwfloat", "__init__.py"))
    kind = "reference" if have_ref else "port"
    port = None
    steps_s = []
    if have_ref:
        for k, n in gemm_parts:
            _REF_DATA[("gemm", k)] = gen.config3_gemm(k, n)
        _REF_DATA["horner"] = gen.config4_horner(npts=procs * 4096, degree=horner["degree"], k=horner["k"])
        _ref_import()
        rows = {2: 1, 3: 1, 4: 1}
        pts = 1024 if args.quick else 2048
        with mp_.get_context("fork").Pool(procs) as pool:
            for _ in range(args.warmup):
                reference_sample(gemm_parts, horner, procs, rows, 256, pool)
            vals, walls = [], []
            for _ in range(args.steps):
                wall, done, full_s, desc = reference_sample(gemm_parts, horner, procs, rows, pts, pool)
                vals.append(step_mp_ops(gemm_parts, horner) / full_s / 1e9)
                walls.append(wall)
                steps_s.append(full_s)
        v = statistics.median(vals)
        sample = (f"unmodified reference (baseline/_ref mwfloat), {procs} processes x 1 thread: " + desc
                  + " per step (median of steps); rates extrapolated linearly to the full step")
        ms_step = statistics.median(walls) * 1e3
        try:  # the C restatement of the same algorithm, for comparison
            port = cpu_sample(gemm_parts, horner, budget_rows={2: 16, 3: 16, 4: 8}, horner_pts=1 << 18)
        except Exception as e:
            port = {"error": f"{type(e).__name__}: {e}"[:200]}
    else:
        small = {2: 16, 3: 16, 4: 8}
        for _ in range(args.warmup):
            cpu_sample(gemm_parts, horner, budget_rows={k: 1 for k in small}, horner_pts=4096)
        vals, walls = [], []
        for _ in range(args.steps):
            t = time.perf_counter()
            r = cpu_sample(gemm_parts, horner, budget_rows=small, horner_pts=1 << 18)
            walls.append(time.perf_counter() - t)
            vals.append(r["value"])
            steps_s.append(r["seconds_per_step_extrapolated"])
            desc = r
        v = statistics.median(vals)
        procs = desc["cores"]
        sample = "C restatement (oracle/, port; baseline/_ref absent): " + desc["sample"]
        ms_step = statistics.median(walls) * 1e3
    print(json.dumps({
        "metric": "DD/TD/QD GEMM and Horner Gops/s vs FP64 FMA roofline, 1/2/4/8 B200",
        "impl": "reference", "value": round(v, 5), "unit": "G MP-ops/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (DD/TD/QD multi-word)", "data": "synthetic (seeded, SURVEY §8(d) G_K)",
        "ms_per_step": round(ms_step, 1),
        "extrapolated": True,
        "ms_per_full_step_extrapolated": round(statistics.median(steps_s) * 1e3, 1),
        "config": {
            "workload": "config3 GEMM DD n4096 + TD n2048 + QD n2048, config4 QD Horner deg1024 x 2^24 pts",
            "gemm": [f"k{k} n{n}" for k, n in gemm_parts], "horner": horner,
            "parallelism": f"rows/points sharded over {procs} host processes (CPU), no collective",
            "l2": "n/a (CPU)", "bit_exact": "the reference itself",
            "horner_points": "double-valued QD points (x, 0, 0, 0) as SURVEY 8(d) config 4 specifies; the reference "
                             "runs its full qw_mul_bf on them",
            "sample": "each step is a bounded sample (ms_per_step = its measured wall time); value = the "
                      "sample's MP-op rate, i.e. the full step extrapolated linearly",
        },
        "host": host,
        "cpu_baseline": {"value": round(v, 5), "unit": "G MP-ops/s", "cores": procs, "kind": kind, "sample": sample,
                         **host},
        "port": port,
        "e2e": {"value": round(v, 5), "unit": "G MP-ops/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def launch_cmd(nproc: int, argv: list, port: int) -> list:
    """torchrun command line that re-runs this script with one rank per GPU
    (the driver's own launch form: 127.0.0.1 rendezvous, one node)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def self_launch(args, argv) -> int | None:
    """`--gpus N` without a torchrun environment: re-execute under torchrun
    with N ranks and return its exit code.  Under torchrun, a world size that
    differs from --gpus is an error (exit 2), never a silent 1-rank run."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            print(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}; refusing to run", file=sys.stderr)
            return 2
        return None
    if args.gpus <= 1:
        return None
    import socket
    import subprocess

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    if args.backend == "nccl":
        env.setdefault("NCCL_DEBUG", "INFO")  # the communicator lines (nranks) for the driver
    print(f"[bench] self-launch: {args.gpus} ranks under torchrun (backend {args.backend})", file=sys.stderr)
    return subprocess.call(launch_cmd(args.gpus, argv, port), env=env)


if __name__ == "__main__":
    a = parse()
    rc = self_launch(a, sys.argv[1:])
    if rc is not None:
        sys.exit(rc)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
