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
             ``DKPeerGraph`` fuses that exchange into the sweep kernel
              itself: each finished root is stored straight into every
              rank's next-state buffer over NVLink (cudaIpc peer memory)
              while the other roots are still being computed, and a
              per-source completion slot replaces the collective.
* dot      -- all-gather-then-sum: each rank produces the tree partials of
              its slice (slices cut at multiples of 4096 elements, one
              partial per 4096), all ranks all-gather them and fold the full
              partial list with the same pairwise tree -- bit-identical to
              the 1-GPU tree dot and on every rank.  NCCL's sum would not be
              error-free, so no reduction collective is used.  ``DotPeer``
              does the same inside one kernel per rank: block roots are
              stored straight into every rank's root buffer over NVLink and
              the last block folds them after a bounded completion wait.

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
           "dk_sweeps_sharded", "allgather_planes", "DKShardedGraph", "PeerLayout", "peer_tables",
           "exchange_handles", "PeerBuffer", "DKPeerGraph", "DotPeer"]

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


# ---------------------------------------------------------------------------
# Fused compute + exchange over peer memory (mw_dk_sweep_peer)


@dataclass(frozen=True)
class PeerLayout:
    """One cudaMalloc buffer per rank, identical layout on every rank:
    state parity 0 | state parity 1 | world u64 completion slots.  A state
    is (2K, n) float64 planes: K re planes, then K im planes."""

    k: int
    n: int
    world: int

    @property
    def state_bytes(self) -> int:
        return 2 * self.k * self.n * 8

    def state_off(self, parity: int) -> int:
        return parity * self.state_bytes

    @property
    def slot_off(self) -> int:
        return 2 * self.state_bytes

    @property
    def total_bytes(self) -> int:
        return self.slot_off + 8 * self.world


def peer_tables(bases: list[int], layout: PeerLayout):
    """Device-pointer tables for mw_dk_sweep_peer from the per-rank buffer
    bases (own base for self, the IPC-mapped address for peers).  Sweep s
    reads parity s % 2 and writes parity 1 - s % 2, so
    ``outs[parity][p]`` = rank p's write buffer for a sweep reading
    ``parity``; ``slots[p]`` = rank p's slot array."""
    outs = [[b + layout.state_off(1 - par) for b in bases] for par in (0, 1)]
    slots = [b + layout.slot_off for b in bases]
    return outs, slots


def exchange_handles(local: bytes, group=None) -> list[bytes]:
    """All ranks' 64-byte IPC handles, in rank order."""
    world = dist.get_world_size(group)
    out: list = [None] * world
    dist.all_gather_object(out, local, group=group)
    return out


class _DevView:
    """Zero-copy torch view of raw device memory (CUDA array interface)."""

    def __init__(self, addr: int, shape: tuple):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f8", "data": (addr, False), "version": 3,
                                         "strides": None}


class PeerBuffer:
    """One zeroed cudaMalloc buffer per rank, cross-mapped into every rank
    with cudaIpc handles (exchanged over ``group``).  ``bases[p]`` is rank
    p's buffer as seen from this process (own pointer for p == rank).
    Construction and ``close()`` are collective."""

    def __init__(self, nbytes: int, device: torch.device, group=None):
        import ctypes

        from . import _lib

        self._lib = lib = _lib.load()
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = device
        buf = ctypes.c_void_p()
        with torch.cuda.device(device):
            _lib.check(lib.mw_peer_alloc(nbytes, ctypes.byref(buf)), "mw_peer_alloc")
        self.base = buf.value
        self._opened: list[int] = []
        self.bases = [self.base] * self.world
        if self.world > 1:
            h = (ctypes.c_char * 64)()
            _lib.check(lib.mw_ipc_get_handle(self.base, h), "mw_ipc_get_handle")
            handles = exchange_handles(bytes(h), group)
            for p, hp in enumerate(handles):
                if p == self.rank:
                    continue
                q = ctypes.c_void_p()
                with torch.cuda.device(device):
                    _lib.check(lib.mw_ipc_open_handle(hp, ctypes.byref(q)), "mw_ipc_open_handle")
                self._opened.append(q.value)
                self.bases[p] = q.value
            torch.cuda.synchronize(device)
            dist.barrier(group)  # every buffer allocated, zeroed and mapped before the first peer store

    def view(self, offset: int, shape: tuple) -> torch.Tensor:
        """float64 tensor view of this rank's buffer at byte ``offset``."""
        return torch.as_tensor(_DevView(self.base + offset, shape), device=self.device)

    def close(self):
        if self.base is None:
            return
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            dist.barrier(self.group)  # no peer still storing into our buffer
        for q in self._opened:
            self._lib.mw_ipc_close_handle(q)
        self._opened = []
        if self.world > 1:
            dist.barrier(self.group)  # every peer unmapped our buffer
        self._lib.mw_peer_free(self.base)
        self.base = None


class DKPeerGraph:
    """``sweeps`` root-sharded DK sweeps whose state exchange happens inside
    the sweep kernel (mw_dk_sweep_peer): no collective on the data path.
    Same interface as ``DKShardedGraph`` (replay / result) and bitwise the
    same result for either order.  All sweeps are captured in one CUDA
    graph; replays need no reset (completion slots are monotonic across
    replays through a device-side epoch).  Requires n divisible by the
    world size.  ``spin_limit`` bounds every completion wait (~0.25 us per
    poll); a wait that expires makes ``result()`` raise instead of hanging."""

    def __init__(self, coeffs: torch.Tensor, zre: torch.Tensor, zim: torch.Tensor, sweeps: int, variant,
                 exact_order: bool = True, group=None, spin_limit: int = 8_000_000):
        from . import _lib
        from .multiword import variant_code
        from .roots import INT32_MAX

        lib = _lib.load()
        _lib.require_cuda(coeffs, zre, zim)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        k, n = zre.shape
        if n % self.world:
            raise ValueError("root count must be divisible by the world size")
        if sweeps < 1:
            raise ValueError("sweeps must be >= 1")
        self.k, self.n, self.sweeps = k, n, sweeps
        per = n // self.world
        lo, hi = self.rank * per, (self.rank + 1) * per
        dev = zre.device
        self.layout = lay = PeerLayout(k, n, self.world)
        self._buf = PeerBuffer(lay.total_bytes, dev, group)
        bases = self._buf.bases
        outs, slots = peer_tables(bases, lay)
        self._outs = [torch.tensor(o, dtype=torch.int64, device=dev) for o in outs]
        self._slots = torch.tensor(slots, dtype=torch.int64, device=dev)
        self._state = [self._buf.view(lay.state_off(par), (2 * k, n)) for par in (0, 1)]
        my_slot = self._buf.base + lay.slot_off
        self._done = torch.zeros(1, dtype=torch.int32, device=dev)
        self._epoch = torch.zeros(1, dtype=torch.int64, device=dev)
        self._timeout = torch.zeros(1, dtype=torch.int32, device=dev)
        self.src = torch.cat([zre, zim], 0).contiguous()
        self.mag = torch.empty(n, dtype=torch.float64, device=dev)
        self.flags = torch.empty(sweeps, dtype=torch.int32, device=dev)
        self._coeffs = coeffs.contiguous()
        self._ws = torch.empty(max(lib.mw_dk_sweep_workspace(k, lo, hi), 1), dtype=torch.float64, device=dev)
        v = variant_code(variant)
        exact = 1 if exact_order else 0

        def body(start: int):
            # sweeps are numbered globally across runs (g = run * sweeps + s)
            # and sweep g reads parity g % 2: the buffer holding a finished
            # run's result is then only rewritten by this rank's own next
            # start copy, never by a peer that is already one run ahead
            stream = _lib.stream_handle(dev)
            self._state[start].copy_(self.src)
            self.flags.fill_(INT32_MAX)
            for s in range(sweeps):
                par = (start + s) & 1
                rc = lib.mw_dk_sweep_peer(
                    k, v, self._coeffs.data_ptr(), self._coeffs.shape[1], n, self._state[par].data_ptr(), lo, hi,
                    self._outs[par].data_ptr(), self._slots.data_ptr(), self._state[1 - par].data_ptr(), my_slot,
                    self._done.data_ptr(), self._epoch.data_ptr(), self._timeout.data_ptr(), self.world,
                    self.rank, s, sweeps, spin_limit, self.mag.data_ptr(), self.flags[s:s + 1].data_ptr(), exact,
                    self._ws.data_ptr(), stream)
                _lib.check(rc, "mw_dk_sweep_peer")

        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            body(0)  # warm-up run (every rank runs it: epochs stay in step)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self._runs = 1
        self._check_timeout()
        # start parity of run r is (r * sweeps) % 2: one graph for an even
        # sweep count, two alternating graphs for an odd one
        self.graphs = {}
        for start in sorted({(r * sweeps) & 1 for r in (1, 2)}):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                body(start)
            self.graphs[start] = g

    def _check_timeout(self):
        if int(self._timeout.item()):
            raise RuntimeError("DKPeerGraph: a peer completion wait expired (a rank stalled or diverged)")

    def replay(self):
        self.graphs[(self._runs * self.sweeps) & 1].replay()
        self._runs += 1

    def result(self):
        """(re, im, first_collision) of the latest run, like
        DKShardedGraph.result() (call it before the next replay)."""
        from .roots import INT32_MAX

        self._check_timeout()
        f = self.flags.clone()
        if self.world > 1:
            dist.all_reduce(f, op=dist.ReduceOp.MIN, group=self.group)
        fl = f.cpu().tolist()
        first = next(((s, c) for s, c in enumerate(fl) if c != INT32_MAX), None)
        fin = self._state[(self._runs * self.sweeps) & 1]
        return fin[: self.k].clone(), fin[self.k:].clone(), first

    def close(self):
        """Release the peer mappings and the buffer (collective: every rank
        calls it, after its last replay)."""
        self.graphs = None
        self._state = None
        self._buf.close()


class DotPeer:
    """Sharded tree dot with the all-gather-then-sum inside ONE kernel per
    rank (mw_dot_peer): each block's subtree root is stored into every
    rank's root buffer over NVLink, the last block waits for all ranks'
    roots (bounded) and folds them with the pairwise tree.  Same shards and
    bits as ``dot_allgather`` (the 1-GPU tree dot) on every rank, no NCCL
    on the data path.  One instance per (k, n); calls are stream-ordered
    and graph-capturable (device-side epoch selects the root-buffer
    parity)."""

    def __init__(self, k: int, n: int, variant, device=None, group=None, spin_limit: int = 8_000_000):
        from . import _lib
        from .multiword import variant_code

        if n < 1:
            raise ValueError("n must be >= 1")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.k, self.n, self.v = k, n, variant_code(variant)
        self.nbt = (n + DOT_PARTIAL_SPAN - 1) // DOT_PARTIAL_SPAN
        if self.nbt > 256 * 256:
            raise ValueError("n too large for the fused dot (at most 2^28 elements)")
        self._buf = PeerBuffer(2 * k * self.nbt * 8 + 8 * (dist.get_world_size(group) if dist.is_initialized()
                                                              else 1), dev, group)
        self.world, self.rank = self._buf.world, self._buf.rank
        self.lo, self.hi = aligned_shard_range(n, self.rank, self.world, DOT_PARTIAL_SPAN)
        slot_off = 2 * k * self.nbt * 8
        self._roots = torch.tensor(self._buf.bases, dtype=torch.int64, device=dev)
        self._slots = torch.tensor([b + slot_off for b in self._buf.bases], dtype=torch.int64, device=dev)
        self._my_slot = self._buf.base + slot_off
        self._done = torch.zeros(1, dtype=torch.int32, device=dev)
        self._epoch = torch.zeros(1, dtype=torch.int64, device=dev)
        self._timeout = torch.zeros(1, dtype=torch.int32, device=dev)
        self.spin_limit = spin_limit
        self.device = dev
        self._lib = _lib

    def __call__(self, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """x, y: the full (K, n) planes (each rank reads only its slice).
        Returns the (K,) dot on every rank."""
        _lib = self._lib
        if x.shape != (self.k, self.n) or y.shape != (self.k, self.n):
            raise ValueError("operand shape does not match this DotPeer")
        if x.device != self.device or y.device != self.device:
            raise ValueError("operands on a different device")
        if x.stride(1) != 1 or y.stride(1) != 1:
            raise ValueError("planes must be contiguous along the element axis")
        out = torch.empty(self.k, dtype=torch.float64, device=self.device) if out is None else out
        nl = self.hi - self.lo
        rc = _lib.load().mw_dot_peer(
            self.k, self.v, x.data_ptr() + 8 * self.lo, x.stride(0), y.data_ptr() + 8 * self.lo, y.stride(0), nl,
            self.lo // DOT_PARTIAL_SPAN, self.nbt, self._roots.data_ptr(), self._slots.data_ptr(), self._my_slot,
            self._done.data_ptr(), self._epoch.data_ptr(), self._timeout.data_ptr(), self.world, self.rank,
            self.spin_limit, out.data_ptr(), _lib.stream_handle(self.device))
        _lib.check(rc, "mw_dot_peer")
        return out

    def check(self):
        """Raise if any completion wait expired."""
        if int(self._timeout.item()):
            raise RuntimeError("DotPeer: a peer completion wait expired (a rank stalled or diverged)")

    def close(self):
        self._buf.close()
