"""Multi-GPU partitioning: one process per GPU, torch.distributed plumbing.

Only the paths that shard naturally are partitioned:

* GEMM     -- row blocks of C (A row block local, B replicated): no
              collective on the data path.
* GEMV     -- row blocks of A / y: no collective.
* Horner   -- contiguous point shards, coefficients replicated: none.
* axpy     -- contiguous lane shards: none.
* DK sweep -- roots [i0, i1) per rank update from the frozen full vector
              (Jacobi), then ONE all-gather of the new (re, im) K-planes per
              sweep rebuilds the full state on every rank.  The exact-order
              kernel makes the result bitwise independent of the GPU count.
* dot      -- all-gather-then-sum: each rank produces the tree partials of
              its slice (slices cut at multiples of 4096 elements, one
              partial per 4096), all ranks all-gather them and fold the full
              partial list with the same pairwise tree -- bit-identical to
              the 1-GPU tree dot and on every rank.  NCCL's sum would not be
              error-free, so no reduction collective is used.

Every partition is over disjoint outputs with a fixed combine order, so
results are invariant to the number of GPUs (the reference's thread
invariance, test_linalg.py:134-143).

The per-rank compute hooks are injectable (``DotBackend``) so the host-side
logic -- shard arithmetic, gather order, fold -- is exercised by CPU
``gloo`` tests with the oracle standing in for the kernels.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

__all__ = ["shard_range", "aligned_shard_range", "DotBackend", "gpu_dot_backend", "dot_allgather",
           "dk_sweeps_sharded", "allgather_planes", "DKShardedGraph"]

DOT_PARTIAL_SPAN = 4096  # elements per dot partial (mw_dot_partials)


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous near-equal split [lo, hi) of ``total`` items."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def aligned_shard_range(total: int, rank: int, world: int, align: int) -> tuple[int, int]:
    """Split at multiples of ``align`` (the last shard takes the ragged tail)."""
    units = (total + align - 1) // align
    lo_u, hi_u = shard_range(units, rank, world)
    return min(lo_u * align, total), min(hi_u * align, total)


@dataclass
class DotBackend:
    """partials(x_slice, y_slice) -> (K, P) tensor of tree partials;
    fold(all_partials (K, total P)) -> (K,) tensor."""

    partials: Callable
    fold: Callable


def gpu_dot_backend(variant) -> DotBackend:
    from . import _lib
    from .multiword import variant_code

    v = variant_code(variant)

    def partials(x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        k, n = x.shape
        lib = _lib.load()
        npart = lib.mw_dot_num_partials(n)
        out = torch.empty((k, max(npart, 0)), dtype=torch.float64, device=x.device)
        if npart:
            rc = lib.mw_dot_partials(k, v, x.data_ptr(), x.stride(0), y.data_ptr(), y.stride(0), n,
                                     out.data_ptr(), npart, _lib.stream_handle(x.device))
            _lib.check(rc, "mw_dot_partials")
        return out

    def fold(p: torch.Tensor) -> torch.Tensor:
        k, cnt = p.shape
        lib = _lib.load()
        p = p.contiguous()
        out = torch.empty(k, dtype=torch.float64, device=p.device)
        wsn = lib.mw_tree_fold_workspace(k, cnt)
        ws = torch.empty(max(wsn, 1), dtype=torch.float64, device=p.device)
        rc = lib.mw_tree_fold(k, v, p.data_ptr(), cnt, cnt, ws.data_ptr(), out.data_ptr(),
                              _lib.stream_handle(p.device))
        _lib.check(rc, "mw_tree_fold")
        return out

    return DotBackend(partials, fold)


def allgather_planes(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """Concatenate per-rank (K, c_r) blocks along axis 1 in rank order.
    Uneven counts are padded to the max for the collective."""
    world = len(counts)
    k = local.shape[0]
    cmax = max(counts) if counts else 0
    buf = torch.zeros((k, cmax), dtype=local.dtype, device=local.device)
    buf[:, : local.shape[1]] = local
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf.contiguous(), group=group)
    return torch.cat([g[:, :c] for g, c in zip(gathered, counts)], dim=1)


def dot_allgather(x: torch.Tensor, y: torch.Tensor, backend: DotBackend, group=None) -> torch.Tensor:
    """Sharded tree dot.  x, y: full (K, n) planes visible to every rank
    (each rank touches only its slice).  Returns the (K,) result on every
    rank, bitwise equal to the 1-GPU tree dot."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n = x.shape[1]
    lo, hi = aligned_shard_range(n, rank, world, DOT_PARTIAL_SPAN)
    part = backend.partials(x[:, lo:hi], y[:, lo:hi])
    counts = []
    for r in range(world):
        a, b = aligned_shard_range(n, r, world, DOT_PARTIAL_SPAN)
        counts.append((b - a + DOT_PARTIAL_SPAN - 1) // DOT_PARTIAL_SPAN)
    allp = allgather_planes(part, counts, group)
    return backend.fold(allp)


def dk_sweeps_sharded(coeffs: torch.Tensor, zre: torch.Tensor, zim: torch.Tensor, sweeps: int, variant,
                      exact_order: bool = True, group=None, sweep_fn=None):
    """Run ``sweeps`` DK sweeps with roots sharded over the ranks of
    ``group``; after each sweep the new root slices are all-gathered so
    every rank holds the full state.  Returns (re, im, first_collision)
    where first_collision is None or (sweep, code).

    ``sweep_fn(coeffs, zre, zim, out_re, out_im, mag, flag, i0, i1)`` is the
    per-rank compute (default: the mw_dk_sweep kernel)."""
    from .roots import INT32_MAX, sweep_into

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    k, n = zre.shape
    lo, hi = shard_range(n, rank, world)
    counts = [shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world)]
    if sweep_fn is None:
        def sweep_fn(c, a, b, orr, oii, mag, flag, i0, i1):
            sweep_into(c, a, b, orr, oii, mag, flag, variant, exact_order, i0, i1)
    cur_re, cur_im = zre.clone(), zim.clone()
    out_re, out_im = torch.empty_like(zre), torch.empty_like(zim)
    mag = torch.empty(n, dtype=torch.float64, device=zre.device)
    flags = torch.full((max(sweeps, 1),), INT32_MAX, dtype=torch.int32, device=zre.device)
    for s in range(sweeps):
        sweep_fn(coeffs, cur_re, cur_im, out_re, out_im, mag, flags[s : s + 1], lo, hi)
        both = torch.cat([out_re[:, lo:hi], out_im[:, lo:hi]], dim=0)
        full = allgather_planes(both, counts, group)
        cur_re = full[:k].contiguous()
        cur_im = full[k:].contiguous()
    # first collision over ranks: MIN over the per-sweep flags
    f = flags.clone()
    if world > 1:
        dist.all_reduce(f, op=dist.ReduceOp.MIN, group=group)
    fl = f.cpu().tolist()
    first = next(((s, c) for s, c in enumerate(fl[:sweeps]) if c != INT32_MAX), None)
    return cur_re, cur_im, first


class DKShardedGraph:
    """``sweeps`` root-sharded DK sweeps with their per-sweep all-gathers,
    captured once in a CUDA graph (kernel + NCCL all_gather_into_tensor +
    re-interleave per sweep), so a fixed-sweep run is one graph launch per
    rank ("capture 200 sweeps + NCCL in a CUDA graph").
    Requires n divisible by the world size (equal shards)."""

    def __init__(self, coeffs: torch.Tensor, zre: torch.Tensor, zim: torch.Tensor, sweeps: int, variant,
                 exact_order: bool = True, group=None):
        from .roots import INT32_MAX, sweep_into

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        k, n = zre.shape
        if n % self.world:
            raise ValueError("root count must be divisible by the world size")
        self.k, self.n, self.sweeps = k, n, sweeps
        per = n // self.world
        lo, hi = self.rank * per, (self.rank + 1) * per
        dev = zre.device
        self.src = torch.cat([zre, zim], 0).contiguous()  # (2K, n) initial state
        self.cur = torch.empty_like(self.src)
        self.out = torch.empty_like(self.src)
        self.send = torch.empty((2 * k, per), dtype=torch.float64, device=dev)
        self.recv = torch.empty((self.world, 2 * k, per), dtype=torch.float64, device=dev)
        self.mag = torch.empty(n, dtype=torch.float64, device=dev)
        self.flags = torch.empty(sweeps, dtype=torch.int32, device=dev)

        def body():
            self.cur.copy_(self.src)
            self.flags.fill_(INT32_MAX)
            for s in range(sweeps):
                sweep_into(coeffs, self.cur[:k], self.cur[k:], self.out[:k], self.out[k:], self.mag,
                           self.flags[s:s + 1], variant, exact_order, lo, hi)
                self.send.copy_(self.out[:, lo:hi])
                dist.all_gather_into_tensor(self.recv, self.send, group=group)
                # recv[r] holds rank r's slice: lay the slices back side by side
                self.cur.view(2 * k, self.world, per).copy_(self.recv.permute(1, 0, 2))

        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            body()  # warm-up (lazy kernel init, NCCL communicator setup)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            body()
        self.group = group

    def replay(self):
        self.graph.replay()

    def result(self):
        """(re, im, first_collision) like dk_sweeps_sharded."""
        from .roots import INT32_MAX

        f = self.flags.clone()
        if self.world > 1:
            dist.all_reduce(f, op=dist.ReduceOp.MIN, group=self.group)
        fl = f.cpu().tolist()
        first = next(((s, c) for s, c in enumerate(fl) if c != INT32_MAX), None)
        return self.cur[: self.k].clone(), self.cur[self.k:].clone(), first
