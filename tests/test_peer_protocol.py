"""Host-side checks of the fused-exchange DK sweep (dist.DKPeerGraph,
mw_dk_sweep_peer in csrc/dk.cu) that need no GPU:

* the buffer layout and the pointer tables the kernel receives;
* the IPC-handle exchange over a world-size-2 gloo group;
* a model of the completion protocol, run under many random interleavings
  of W ranks: the per-sweep state reads, the peer stores of each finished
  root, the per-source completion slots (st.release.sys value
  run * sweeps + s + 1) and the bounded waits, plus the start-of-run copy
  and the host's result read between runs.  The model asserts that no rank
  reads an entry of the wrong sweep, that no store lands in a buffer a
  peer has not finished reading, and that each run's result is intact
  when the host reads it.  Variants that publish completion before the
  stores, or that restart every run from parity 0, are caught by the same
  model (so it has teeth);
* the same for the fused dot (mw_dot_peer): roots stored, slot published,
  wait, then the fold reads every root; a single (not double) root buffer
  is caught.
"""

import os
import random
import tempfile

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_14926_b200 import dist as mwdist

from test_dist_gloo import _free_port


def test_layout_and_tables():
    lay = mwdist.PeerLayout(k=3, n=4096, world=4)
    assert lay.state_bytes == 2 * 3 * 4096 * 8
    assert lay.state_off(0) == 0 and lay.state_off(1) == lay.state_bytes
    assert lay.slot_off == 2 * lay.state_bytes and lay.slot_off % 16 == 0
    assert lay.total_bytes == lay.slot_off + 8 * 4
    bases = [0x10000000 * (p + 1) for p in range(4)]
    outs, slots = mwdist.peer_tables(bases, lay)
    for par in (0, 1):
        # a sweep reading parity `par` writes parity 1 - par on every rank
        assert outs[par] == [b + lay.state_off(1 - par) for b in bases]
    assert slots == [b + lay.slot_off for b in bases]


def _hworker(rank, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        mine = bytes([rank + 1]) * 64
        got = mwdist.exchange_handles(mine)
        np.save(os.path.join(outdir, f"h{rank}.npy"), np.frombuffer(b"".join(got), dtype=np.uint8))
    finally:
        dist.destroy_process_group()


def test_exchange_handles_rank_order():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_hworker, args=(_free_port(), d), nprocs=2, join=True)
        for r in range(2):
            h = np.load(os.path.join(d, f"h{r}.npy"))
            assert h.tolist() == [1] * 64 + [2] * 64


class _Hazard(AssertionError):
    pass


def _model(world, sweeps, runs, per, seed, publish_first=False, fixed_start=False):
    """Interleave the per-rank programs at random; each ``yield`` is one
    memory action.  Entries carry the global sweep number g of the state
    they belong to (run r, sweep s -> g = r * sweeps + s)."""
    rng = random.Random(seed)
    n = world * per
    buf = [[[None] * n for _ in range(2)] for _ in range(world)]
    slots = [[0] * world for _ in range(world)]
    epoch = [0] * world
    reading = [None] * world  # (parity) while a rank's sweep reads
    results = []

    def check(cond, msg):
        if not cond:
            raise _Hazard(msg)

    def program(r):
        for run in range(runs):
            start = 0 if fixed_start else (run * sweeps) & 1
            for i in range(n):
                buf[r][start][i] = run * sweeps
                yield
            for s in range(sweeps):
                g = run * sweeps + s
                par = (start + s) & 1
                reading[r] = par
                order = list(range(n))
                rng.shuffle(order)
                for i in order:  # CTAs read the frozen state over time
                    check(buf[r][par][i] == g, f"rank {r} sweep {g} read entry {i} = {buf[r][par][i]}")
                    yield
                reading[r] = None
                v = epoch[r] * sweeps + s + 1
                if publish_first:
                    for p in range(world):
                        slots[p][r] = v
                        yield
                for i in range(r * per, (r + 1) * per):
                    peers = list(range(world))
                    rng.shuffle(peers)
                    for p in peers:
                        check(reading[p] != 1 - par, f"rank {r} stored into rank {p}'s buffer under read")
                        old = buf[p][1 - par][i]
                        check(old is None or old <= g - 1 or old == g + 1,
                              f"rank {r} overwrote live entry {old} on rank {p}")
                        buf[p][1 - par][i] = g + 1
                        yield
                if not publish_first:
                    for p in range(world):
                        slots[p][r] = v
                        yield
                for src in range(world):
                    while slots[r][src] < v:
                        yield
                if s == sweeps - 1:
                    epoch[r] += 1
            fin = (start + sweeps) & 1
            for _ in range(rng.randrange(3)):  # host latency before result()
                yield
            for i in range(n):
                check(buf[r][fin][i] == (run + 1) * sweeps, f"rank {r} run {run} result entry {i} overwritten")
            results.append((r, run))
            yield

    progs = [program(r) for r in range(world)]
    live = set(range(world))
    steps = 0
    while live:
        r = rng.choice(sorted(live))
        try:
            next(progs[r])
        except StopIteration:
            live.discard(r)
        steps += 1
        assert steps < 2_000_000, "model did not terminate (deadlock)"
    assert len(results) == world * runs


def test_protocol_model_random_interleavings():
    for seed in range(60):
        world = 2 + seed % 3
        sweeps = 1 + seed % 4  # odd and even sweep counts (start-parity alternation)
        _model(world, sweeps, runs=3, per=2, seed=seed)


def _breaks(**kw):
    broke = 0
    for seed in range(100):
        try:
            _model(seed=seed, **kw)
        except _Hazard:
            broke += 1
    return broke


def test_model_catches_early_publication():
    assert _breaks(world=3, sweeps=2, runs=1, per=2, publish_first=True) > 0


def test_model_catches_fixed_start_parity_with_odd_sweeps():
    """Restarting every run at parity 0 with an odd sweep count lets a peer
    already in the next run overwrite the previous result."""
    assert _breaks(world=3, sweeps=3, runs=3, per=2, fixed_start=True) > 0


def _dot_model(world, calls, seed, single_buffer=False):
    """The mw_dot_peer protocol: per call c each rank stores its root into
    slot [rank] of every rank's buffer (parity c % 2), publishes c + 1,
    waits for all sources, then folds (reads) its own buffer."""
    rng = random.Random(seed)
    buf = [[[None] * world for _ in range(2)] for _ in range(world)]
    slots = [[0] * world for _ in range(world)]

    def check(cond, msg):
        if not cond:
            raise _Hazard(msg)

    def program(r):
        for c in range(calls):
            par = 0 if single_buffer else c & 1
            peers = list(range(world))
            rng.shuffle(peers)
            for p in peers:
                buf[p][par][r] = c
                yield
            for p in range(world):
                slots[p][r] = c + 1
                yield
            for src in range(world):
                while slots[r][src] < c + 1:
                    yield
            order = list(range(world))
            rng.shuffle(order)
            for i in order:  # the last block's fold reads every root
                check(buf[r][par][i] == c, f"rank {r} call {c} folded root {i} = {buf[r][par][i]}")
                yield

    progs = [program(r) for r in range(world)]
    live = set(range(world))
    steps = 0
    while live:
        r = rng.choice(sorted(live))
        try:
            next(progs[r])
        except StopIteration:
            live.discard(r)
        steps += 1
        assert steps < 1_000_000, "deadlock"


def test_dot_protocol_model():
    for seed in range(80):
        _dot_model(2 + seed % 4, calls=4, seed=seed)


def test_dot_model_catches_single_buffer():
    broke = 0
    for seed in range(100):
        try:
            _dot_model(3, calls=4, seed=seed, single_buffer=True)
        except _Hazard:
            broke += 1
    assert broke > 0
