"""Durand-Kerner simultaneous root iteration in complex K-word arithmetic.

Drop-in for mwfloat.roots (pkg/src/mwfloat/roots.py): ``MonicPoly``
(73-131), ``RootState`` (134-159), ``CollisionError`` / ``NoConvergence``
(61-70), ``default_tolerance`` (162-164), ``radius_estimate`` (167-185),
``aberth_init`` (188-221), ``dk_iterate`` (240-315) and ``dk_solve``
(318-340), same signatures.

The sweep is one mw_dk_sweep launch.  ``exact_order=True`` (default)
replays the reference's op order bit for bit (numerator Horner and ordered
denominator on two independent lanes per root); ``exact_order=False`` is
the warp-per-root tree kernel (reassociated, within the n 2^-p bound).
``dk_sweeps`` runs a fixed number of sweeps with no host round trip (the
benchmark form of config 5) and can capture them in a CUDA graph.

Initialization needs pi, cos, sin and fractional powers to ~300 bits; the
reference uses its BigFloat oracle, here mpmath at 400 bits, both rounded
to K words by greedy nearest-double extraction.  This is host-side setup,
not the hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import torch

from . import _lib
from .batch import LaneBatch, as_planes, batch_add, batch_div, batch_mul, coefficient_planes
from .multiword import BITS, Variant, from_basefloat, from_fraction, variant_code

__all__ = [
    "MonicPoly",
    "RootState",
    "CollisionError",
    "NoConvergence",
    "aberth_init",
    "radius_estimate",
    "dk_iterate",
    "dk_sweeps",
    "DKSweepGraph",
    "dk_solve",
    "default_tolerance",
    "chebyshev_coeffs",
    "residual_check",
]

INT32_MAX = 2**31 - 1


class CollisionError(ValueError):
    """A denominator factor z_i - z_j vanished: two approximations are equal
    and the simultaneous update is undefined (roots.py:61-64)."""


class NoConvergence(RuntimeError):
    """The sweep budget ran out before the tolerance was met; ``state``
    holds the last iterate (roots.py:67-74)."""

    def __init__(self, message, state):
        super().__init__(message)
        self.state = state


class MonicPoly:
    """q(x) = x^n + sum c_i x^i with K-word coefficients c[0..n-1]."""

    __slots__ = ("planes",)

    def __init__(self, comps, device=None):
        self.planes = as_planes(comps, 1, device)
        if self.planes.shape[1] < 1:
            raise ValueError("monic polynomial needs degree >= 1")

    @property
    def comps(self) -> tuple:
        return tuple(self.planes[c] for c in range(self.k))

    @property
    def k(self) -> int:
        return self.planes.shape[0]

    @property
    def n(self) -> int:
        return self.planes.shape[1]

    @property
    def device(self):
        return self.planes.device

    @classmethod
    def from_coeffs(cls, coeffs, k: int | None = None, device=None) -> "MonicPoly":
        return cls(coefficient_planes(coeffs, k), device=device)

    @classmethod
    def from_polynomial(cls, p, variant: Variant = Variant.STANDARD) -> "MonicPoly":
        """Divide through by the leading coefficient (roots.py:93-101)."""
        an = p.coeff(p.degree)
        if all(c == 0.0 for c in an):
            raise ValueError("leading coefficient is zero")
        num = LaneBatch(p.planes[:, : p.degree].contiguous())
        den = LaneBatch(torch.tensor(an, dtype=torch.float64, device=p.device).reshape(-1, 1).expand(-1, p.degree).contiguous())
        return cls(batch_div(num, den, variant).planes)

    def coeff(self, i: int) -> tuple:
        return tuple(float(v) for v in self.planes[:, i].cpu())

    def __repr__(self):
        return f"MonicPoly(k={self.k}, n={self.n}, device={self.device})"


@dataclass
class RootState:
    """Simultaneous approximations: (K, n) re / im planes."""

    re: torch.Tensor
    im: torch.Tensor
    iteration: int = 0
    converged: bool = False
    last_max_update: float = math.inf

    def __post_init__(self):
        self.re = as_planes(self.re, 1)
        self.im = as_planes(self.im, 1, self.re.device)
        if self.re.shape != self.im.shape:
            raise ValueError("re/im shape mismatch")

    @property
    def n(self) -> int:
        return self.re.shape[1]

    @property
    def k(self) -> int:
        return self.re.shape[0]

    def root(self, i: int):
        return (
            tuple(float(v) for v in self.re[:, i].cpu()),
            tuple(float(v) for v in self.im[:, i].cpu()),
        )

    def roots(self) -> list:
        re = self.re.cpu().numpy()
        im = self.im.cpu().numpy()
        return [
            (tuple(float(v) for v in re[:, i]), tuple(float(v) for v in im[:, i]))
            for i in range(self.n)
        ]


def default_tolerance(k: int) -> float:
    """Relative step threshold 2^(-bits + 10)."""
    return math.ldexp(1.0, -BITS[k] + 10)


# ------------------------------------------------------------ init (host)
def _mp():
    import mpmath

    mpmath.mp.prec = 400
    return mpmath


def _mpf_fraction(x) -> Fraction:
    """Exact value of a finite mpmath mpf."""
    sign, man, exp, _ = x._mpf_
    v = Fraction(int(man)) * (Fraction(2) ** int(exp))
    return -v if sign else v


def radius_estimate(q: MonicPoly, variant: Variant = Variant.STANDARD) -> tuple:
    """r = max over nonzero c_i of |n_nz c_i|^(1/(n-i)), K words
    (roots.py:167-185); all coefficients zero gives r = 1."""
    mp = _mp()
    n = q.n
    arr = q.planes.cpu().numpy()
    nz = [i for i in range(n) if np.any(arr[:, i] != 0.0)]
    if not nz:
        return from_basefloat(1.0, q.k)
    n_nz = len(nz) + 1
    best = None
    for i in nz:
        mag = abs(sum(Fraction(float(c)) for c in arr[:, i]))
        x = mp.mpf(n_nz * mag.numerator) / mag.denominator
        r_i = mp.root(x, n - i)
        if best is None or r_i > best:
            best = r_i
    return from_fraction(_mpf_fraction(best), q.k)


def _check_distinct(state: RootState):
    zre = state.re[0].cpu().numpy()
    zim = state.im[0].cpu().numpy()
    n = state.n
    for i in range(n):
        d2 = (zre - zre[i]) ** 2 + (zim - zim[i]) ** 2
        d2[i] = np.inf
        j = int(np.argmin(d2))
        if d2[j] == 0.0 and state.root(i) == state.root(j):
            raise CollisionError(f"approximations {i} and {j} coincide")


def aberth_init(q: MonicPoly, variant: Variant = Variant.STANDARD, radius=None) -> RootState:
    """Points -c_{n-1}/n + r exp(i (2(j-1)pi/n + 3/(2n))), j = 1..n
    (roots.py:188-221).  ``radius`` overrides radius_estimate (e.g. the
    R0 = 1.5 circle SURVEY §8(d) uses for the degree-512 problem)."""
    mp = _mp()
    n, k = q.n, q.k
    dev = q.device
    cn = LaneBatch(q.planes[:, n - 1 : n].contiguous())
    nn = LaneBatch(np.array(from_basefloat(float(n), k)).reshape(k, 1), device=dev)
    center = tuple(-c for c in batch_div(cn, nn, variant).lane(0))
    if radius is None:
        rad = radius_estimate(q, variant)
    elif isinstance(radius, (int, float)):
        rad = from_basefloat(float(radius), k)
    else:
        rad = tuple(getattr(radius, "comps", radius))
    if len(rad) != k:
        rad = from_basefloat(float(rad[0]), k)
    cosv = np.zeros((k, n))
    sinv = np.zeros((k, n))
    two_over_n = mp.mpf(2) / n
    offset = mp.mpf(3) / (2 * n)
    for j in range(1, n + 1):
        theta = (j - 1) * two_over_n * mp.pi + offset
        cosv[:, j - 1] = from_fraction(_mpf_fraction(mp.cos(theta)), k)
        sinv[:, j - 1] = from_fraction(_mpf_fraction(mp.sin(theta)), k)
    radb = LaneBatch(np.tile(np.array(rad).reshape(k, 1), (1, n)), device=dev)
    cenb = LaneBatch(np.tile(np.array(center).reshape(k, 1), (1, n)), device=dev)
    zre = batch_add(cenb, batch_mul(radb, LaneBatch(cosv, device=dev), variant), variant)
    zim = batch_mul(radb, LaneBatch(sinv, device=dev), variant)
    state = RootState(re=zre.planes, im=zim.planes)
    _check_distinct(state)
    return state


# ---------------------------------------------------------------- sweep
def sweep_into(coeffs: torch.Tensor, zre: torch.Tensor, zim: torch.Tensor, out_re: torch.Tensor,
               out_im: torch.Tensor, step_mag: torch.Tensor, flag: torch.Tensor, variant,
               exact_order: bool = True, i0: int = 0, i1: int | None = None, tuning=None,
               max_bits: torch.Tensor | None = None) -> None:
    """Raw launch: roots [i0, i1) of the frozen state -> out planes at the
    same indices (plane stride n).  ``flag`` (int32 device scalar) must hold
    INT32_MAX beforehand; it is lowered to min(j*n + i) on a collision.
    ``tuning``: an optional _lib.Tuning (launch shape only; same bits).
    ``max_bits`` (two int64 on the device, zero beforehand) receive the bit
    patterns of the largest step_mag written (the sweep's max update) and
    of the largest new |z| = hypot(re0, im0)."""
    # the tree order's stream-ordered scratch (lane-per-root powers kernel)
    # is allocated in the extension from torch's caching allocator
    _lib.ext().dk_sweep(variant_code(variant), coeffs, zre, zim, out_re, out_im, step_mag, flag, bool(exact_order),
                        i0, -1 if i1 is None else i1,
                        **_lib.tune_kw(tuning, "dk_tree_roots", "dk_exact_roots", "dk_exact_split"),
                        max_bits=max_bits)


def _raise_collision(code: int, n: int):
    j, i = divmod(int(code), n)
    raise CollisionError(f"z_{i} equals z_{j}; denominator vanishes")


def dk_iterate(q: MonicPoly, state: RootState, variant: Variant = Variant.STANDARD,
               exact_order: bool = True) -> RootState:
    """One simultaneous sweep: z_i <- z_i - q(z_i) / prod_{j != i}(z_i - z_j),
    all i from the frozen previous state; a zero factor raises
    CollisionError."""
    if state.k != q.k:
        raise ValueError("mixed word counts")
    if state.n != q.n:
        raise ValueError("state size does not match the polynomial degree")
    _lib.require_cuda(q.planes, state.re, state.im)
    dev = state.re.device
    out_re = torch.empty_like(state.re)
    out_im = torch.empty_like(state.im)
    mag = torch.empty(state.n, dtype=torch.float64, device=dev)
    # three int64, uploaded by a copy (no fill kernel): [0] low word = the
    # collision flag (INT32_MAX = none), [1] / [2] = the max-update and
    # max-|z| bits the sweep kernel raises atomically (no torch reduction)
    status = torch.tensor([INT32_MAX, 0, 0], dtype=torch.int64).to(dev, non_blocking=True)
    sweep_into(q.planes, state.re, state.im, out_re, out_im, mag, status.view(torch.int32)[0:1], variant,
               exact_order, max_bits=status[1:3])
    host = status.cpu().numpy()  # one read-back per sweep
    code = int(host[0])
    if code != INT32_MAX:
        _raise_collision(code, state.n)
    return RootState(
        re=out_re, im=out_im, iteration=state.iteration + 1, converged=False,
        last_max_update=float(host[1:2].view(np.float64)[0]),
    )


def dk_sweeps(q: MonicPoly, state: RootState, sweeps: int, variant: Variant = Variant.BRANCH_FREE,
              exact_order: bool = True, check: bool = True, tuning=None) -> RootState:
    """``sweeps`` sweeps back to back on the device (ping-pong buffers, no
    host synchronisation in between).  Collision flags are kept per sweep
    and checked once at the end (first colliding sweep reported)."""
    _lib.require_cuda(q.planes, state.re, state.im)
    dev = state.re.device
    bufs = [(state.re.clone(), state.im.clone()), (torch.empty_like(state.re), torch.empty_like(state.im))]
    mag = torch.empty(state.n, dtype=torch.float64, device=dev)
    flags = torch.full((max(sweeps, 1),), INT32_MAX, dtype=torch.int32, device=dev)
    for s in range(sweeps):
        src, dst = bufs[s & 1], bufs[(s + 1) & 1]
        sweep_into(q.planes, src[0], src[1], dst[0], dst[1], mag, flags[s : s + 1], variant, exact_order,
                   tuning=tuning)
    fin = bufs[sweeps & 1]
    if check and sweeps > 0:
        f = flags.cpu().numpy()
        bad = np.nonzero(f != INT32_MAX)[0]
        if bad.size:
            _raise_collision(int(f[bad[0]]), state.n)
    return RootState(
        re=fin[0], im=fin[1], iteration=state.iteration + sweeps, converged=False,
        last_max_update=float(mag.max().item()) if sweeps > 0 else state.last_max_update,
    )


class DKSweepGraph:
    """``sweeps`` DK sweeps captured once into a CUDA graph (state reset,
    flag reset and every sweep launch), so a fixed-sweep run costs one
    graph launch instead of ``sweeps`` host round trips.

        g = DKSweepGraph(q, state, 200, Variant.BRANCH_FREE)
        g.replay()              # rerun from `state` (or g.load(new_state))
        final = g.result()      # RootState; raises CollisionError
    """

    def __init__(self, q: MonicPoly, state: RootState, sweeps: int, variant: Variant = Variant.BRANCH_FREE,
                 exact_order: bool = True, tuning=None):
        _lib.require_cuda(q.planes, state.re, state.im)
        if sweeps < 1:
            raise ValueError("sweeps must be >= 1")
        self.q, self.n, self.sweeps = q, state.n, sweeps
        self.iteration0 = state.iteration
        dev = state.re.device
        self.src = (state.re.clone(), state.im.clone())
        self.bufs = [(torch.empty_like(state.re), torch.empty_like(state.im)) for _ in range(2)]
        self.mag = torch.empty(state.n, dtype=torch.float64, device=dev)
        self.flags = torch.empty(sweeps, dtype=torch.int32, device=dev)

        def body():
            self.bufs[0][0].copy_(self.src[0])
            self.bufs[0][1].copy_(self.src[1])
            self.flags.fill_(INT32_MAX)
            for s_ in range(sweeps):
                a, b = self.bufs[s_ & 1], self.bufs[(s_ + 1) & 1]
                sweep_into(q.planes, a[0], a[1], b[0], b[1], self.mag, self.flags[s_ : s_ + 1], variant,
                           exact_order, tuning=tuning)

        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            body()  # warm-up outside capture (lazy init of kernels / attributes)
        torch.cuda.current_stream(dev).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            body()

    def load(self, state: RootState):
        self.src[0].copy_(state.re)
        self.src[1].copy_(state.im)
        self.iteration0 = state.iteration

    def replay(self):
        self.graph.replay()

    def result(self, check: bool = True) -> RootState:
        if check:
            f = self.flags.cpu().numpy()
            bad = np.nonzero(f != INT32_MAX)[0]
            if bad.size:
                _raise_collision(int(f[bad[0]]), self.n)
        fin = self.bufs[self.sweeps & 1]
        return RootState(re=fin[0].clone(), im=fin[1].clone(), iteration=self.iteration0 + self.sweeps,
                         converged=False, last_max_update=float(self.mag.max().item()))


def dk_solve(q: MonicPoly, variant: Variant = Variant.STANDARD, tol: float | None = None, max_iter: int = 200,
             state: RootState | None = None, exact_order: bool = True):
    """Iterate until the largest update falls below tol * max|z| or the
    budget runs out (NoConvergence carrying the state).  Returns
    (state, iterations) (roots.py:318-340).

    Same sweeps, same per-sweep test and the same result as calling
    dk_iterate until converged, but the sweeps run in growing chunks (2, 4,
    ..., 32) back to back on the device, each sweep writing its own state,
    update magnitudes and collision flag; the per-sweep convergence test is
    evaluated on the device and the host reads one small vector per chunk
    and returns the first converged sweep's state (a collision raises at
    its own sweep, before that sweep's convergence test, as in the
    reference loop).  The up to 31 sweeps computed past convergence cost
    device time only.

    The iterates are bit-identical to the reference's sweep by sweep (exact
    order), and the test is the reference's comparison evaluated on the
    host in binary64; its two magnitudes, however, are CUDA's hypot (<= 2
    ulp, taken inside the sweep kernel) where the reference uses np.hypot
    (roots.py:308, 336), so when the largest update lands within a few ulp
    of tol * max|z| the first converged sweep can differ from the
    reference loop's by one."""
    if tol is None:
        tol = default_tolerance(q.k)
    if tol <= 0:
        raise ValueError("tol must be positive")
    if state is None:
        state = aberth_init(q, variant)
    if state.k != q.k:
        raise ValueError("mixed word counts")
    if state.n != q.n:
        raise ValueError("state size does not match the polynomial degree")
    _lib.require_cuda(q.planes, state.re, state.im)
    dev = state.re.device
    k, n = state.k, state.n
    cur_re, cur_im, it = state.re, state.im, state.iteration
    done, chunk = 0, 2
    last = state
    while done < max_iter:
        m = min(chunk, max_iter - done)
        res_re = torch.empty((m, k, n), dtype=torch.float64, device=dev)
        res_im = torch.empty_like(res_re)
        mag = torch.empty((m, n), dtype=torch.float64, device=dev)
        # per sweep: [collision flag (low word), max-update bits, max-|z|
        # bits], raised by the sweep kernels themselves; uploaded and read
        # back once per chunk (no torch kernels on this path)
        status = torch.from_numpy(np.tile(np.array([INT32_MAX, 0, 0], dtype=np.int64), (m, 1))).to(dev)
        flags32 = status.view(torch.int32)  # (m, 6): column 0 is each row's low word
        src_re, src_im = cur_re, cur_im
        for s in range(m):
            sweep_into(q.planes, src_re, src_im, res_re[s], res_im[s], mag[s], flags32[s, 0:1], variant,
                       exact_order, max_bits=status[s, 1:3])
            src_re, src_im = res_re[s], res_im[s]
        host = status.cpu().numpy()
        upd_all = host[:, 1].copy().view(np.float64)
        zmag_all = host[:, 2].copy().view(np.float64)
        for s in range(m):
            if int(host[s, 0]) != INT32_MAX:
                _raise_collision(int(host[s, 0]), n)
            upd, zmag = float(upd_all[s]), float(zmag_all[s])
            if upd <= tol * max(zmag, 1e-300):  # the reference's test, on the host (roots.py:336-337)
                st = RootState(re=res_re[s], im=res_im[s], iteration=it + s + 1, converged=True,
                               last_max_update=upd)
                return st, st.iteration
        last = RootState(re=res_re[m - 1], im=res_im[m - 1], iteration=it + m, converged=False,
                         last_max_update=float(upd_all[m - 1]))
        cur_re, cur_im, it = last.re, last.im, last.iteration
        done += m
        chunk = min(2 * chunk, 32)
    raise NoConvergence(f"no convergence in {max_iter} sweeps", last)


# ------------------------------------------------------ test problems (host)
def chebyshev_coeffs(n: int, k: int, weight=None, device=None) -> MonicPoly:
    """Even-coefficient integration test polynomial of degree n
    (roots.py:343-368): a_n = 1, odd-from-top coefficients zero,
    a_{n-2m} = -sum_{j=1..m} weight(j) a_{n-2(m-j)}, default weight
    1/(2j+1); exact rationals rounded per coefficient to K words."""
    if n < 2:
        raise ValueError("n must be >= 2")
    if weight is None:
        def weight(j):
            return Fraction(1, 2 * j + 1)
    b = [Fraction(1)]
    for m in range(1, n // 2 + 1):
        b.append(-sum(weight(j) * b[m - j] for j in range(1, m + 1)))
    arr = np.zeros((k, n))
    for i in range(n):
        d = n - i
        if d % 2 == 0:
            arr[:, i] = from_fraction(b[d // 2], k)
    return MonicPoly(arr, device=device)


def residual_check(q: MonicPoly, roots) -> float:
    """max_i |q(z_i)| evaluated exactly (roots.py:371-385 uses a 300-bit
    oracle; here exact rationals, then rounded to a float)."""
    arr = q.planes.cpu().numpy()
    coeffs = [sum(Fraction(float(c)) for c in arr[:, i]) for i in range(q.n)] + [Fraction(1)]
    worst = 0.0
    for zre, zim in roots:
        zr = sum(Fraction(float(c)) for c in zre)
        zi = sum(Fraction(float(c)) for c in zim)
        ar, ai = coeffs[-1], Fraction(0)
        for c in reversed(coeffs[:-1]):
            ar, ai = ar * zr - ai * zi + c, ar * zi + ai * zr
        mag2 = ar * ar + ai * ai
        if mag2:
            worst = max(worst, math.sqrt(float(mag2)) if float(mag2) > 0 else
                        2.0 ** ((mag2.numerator.bit_length() - mag2.denominator.bit_length()) / 2.0))
    return worst
