"""Multi-GPU host logic on CPU: world_size 2 over torch.distributed gloo.

The per-rank compute hooks are the CPU oracle (the kernels need a GPU);
what is tested is the partitioning, the collective pattern and the combine
order of paper_2603_14926_b200.dist -- and that the sharded results equal
the single-process results bit for bit (GPU-count invariance).
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import assert_bitwise
from paper_2603_14926_b200 import dist as mwdist
from paper_2603_14926_b200 import gen

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_dot_backend():
    span = mwdist.DOT_PARTIAL_SPAN

    def partials(x, y):
        xn, yn = x.numpy(), y.numpy()
        n = xn.shape[1]
        cols = []
        for b in range(0, n, span):
            cols.append(oracle.dot(xn[:, b:b + span], yn[:, b:b + span], "bf", order=1))
        return torch.from_numpy(np.stack(cols, axis=1)) if cols else torch.zeros((xn.shape[0], 0), dtype=torch.float64)

    def fold(p):
        return torch.from_numpy(oracle.tree_fold(p.numpy(), "bf"))

    return mwdist.DotBackend(partials, fold)


def _worker(rank, port, outdir, job):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        if job == "dot":
            for k, n in ((2, 65536), (3, 10000), (4, 4097), (2, 100)):
                rng = np.random.default_rng(n + k)
                x, y = gen.g_k(rng, k, n), gen.g_k(rng, k, n)
                r = mwdist.dot_allgather(torch.from_numpy(x), torch.from_numpy(y), _oracle_dot_backend())
                np.save(os.path.join(outdir, f"dot_{k}_{n}_{rank}.npy"), r.numpy())
        elif job == "dk":
            k, n = 3, 64
            rng = np.random.default_rng(11)
            coeffs = gen.g_k(rng, k, n) * 0.5
            ang = 2 * np.pi * np.arange(n) / n + 0.1
            zre = np.zeros((k, n)); zim = np.zeros((k, n))
            zre[0] = 1.3 * np.cos(ang); zim[0] = 1.3 * np.sin(ang)

            def sweep_fn(c, a, b, orr, oii, mag, flag, i0, i1):
                nre, nim, m, coll = oracle.dk_sweep(c.numpy(), a.numpy(), b.numpy(), "bf", exact=True, rows=(i0, i1))
                orr[:, i0:i1] = torch.from_numpy(nre[:, i0:i1])
                oii[:, i0:i1] = torch.from_numpy(nim[:, i0:i1])
                if coll is not None:
                    flag.fill_(coll[0] * n + coll[1])

            re, im, first = mwdist.dk_sweeps_sharded(torch.from_numpy(coeffs), torch.from_numpy(zre),
                                                     torch.from_numpy(zim), 4, "bf", sweep_fn=sweep_fn)
            assert first is None
            np.save(os.path.join(outdir, f"dk_{rank}.npy"), np.stack([re.numpy(), im.numpy()]))
        elif job == "gemm":
            k, m, kd, n = 3, 37, 23, 29
            rng = np.random.default_rng(5)
            a, b = gen.g_k(rng, k, (m, kd)), gen.g_k(rng, k, (kd, n))
            lo, hi = mwdist.shard_range(m, rank, WORLD)
            block = oracle.gemm(a, b, "bf", rows=(lo, hi))[:, lo:hi]  # (k, rows, n)
            counts = [mwdist.shard_range(m, r, WORLD)[1] - mwdist.shard_range(m, r, WORLD)[0] for r in range(WORLD)]
            flat = torch.from_numpy(np.ascontiguousarray(block.transpose(0, 2, 1).reshape(k * n, -1)))
            full = mwdist.allgather_planes(flat, counts)  # (k*n, m)
            c = full.numpy().reshape(k, n, m).transpose(0, 2, 1)
            np.save(os.path.join(outdir, f"gemm_{rank}.npy"), np.ascontiguousarray(c))
    finally:
        dist.destroy_process_group()


def _run(job):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(_free_port(), d, job), nprocs=WORLD, join=True)
        return {f: np.load(os.path.join(d, f)) for f in os.listdir(d)}


def test_shard_ranges_cover_and_align():
    for total in (0, 1, 7, 4096, 65536, 100003):
        for world in (1, 2, 3, 8):
            rs = [mwdist.shard_range(total, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            al = [mwdist.aligned_shard_range(total, r, world, 4096) for r in range(world)]
            assert al[0][0] == 0 and al[-1][1] == total
            assert all(a[1] == b[0] and a[1] % 4096 == 0 for a, b in zip(al, al[1:]) if a[1] < total)


def test_dot_allgather_then_sum_is_gpu_count_invariant():
    out = _run("dot")
    for k, n in ((2, 65536), (3, 10000), (4, 4097), (2, 100)):
        rng = np.random.default_rng(n + k)
        x, y = gen.g_k(rng, k, n), gen.g_k(rng, k, n)
        want = oracle.dot(x, y, "bf", order=1)  # the 1-GPU tree dot
        for r in range(WORLD):
            assert_bitwise(out[f"dot_{k}_{n}_{r}.npy"], want)


def test_dk_sharded_sweeps_equal_single_process():
    out = _run("dk")
    k, n = 3, 64
    rng = np.random.default_rng(11)
    coeffs = gen.g_k(rng, k, n) * 0.5
    ang = 2 * np.pi * np.arange(n) / n + 0.1
    zre = np.zeros((k, n)); zim = np.zeros((k, n))
    zre[0] = 1.3 * np.cos(ang); zim[0] = 1.3 * np.sin(ang)
    for _ in range(4):
        zre, zim, _, _ = oracle.dk_sweep(coeffs, zre, zim, "bf", exact=True)
    for r in range(WORLD):
        got = out[f"dk_{r}.npy"]
        assert_bitwise(got[0], zre)
        assert_bitwise(got[1], zim)


def test_gemm_row_blocks_reassemble():
    out = _run("gemm")
    k, m, kd, n = 3, 37, 23, 29
    rng = np.random.default_rng(5)
    a, b = gen.g_k(rng, k, (m, kd)), gen.g_k(rng, k, (kd, n))
    want = oracle.gemm(a, b, "bf")
    for r in range(WORLD):
        assert_bitwise(out[f"gemm_{r}.npy"], want)
