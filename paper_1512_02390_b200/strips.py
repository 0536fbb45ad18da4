"""Element-row strip decomposition of the V-cycle and the outer solvers
across ranks (one process per GPU).

Rank g owns element rows [g s, (g+1) s) (s = n_y / world) and keeps G = 2
ghost element rows on each side.  Its local arrays are the (p (s + 2G), N_x)
row window of the global (N_y, N_x) field, and every per-level operator,
smoother and transfer runs UNCHANGED on the local mesh
``MeshConfig(n_x, s + 2G, l_x, dy (s + 2G))`` treated as periodic: outputs on
owned rows are exact as long as the ghost rows hold the neighbours' data,
because

* ``r = f - A u`` on owned rows reads u one element row beyond them;
* the Schwarz windows of the first ghost element row reach n_o < p rows into
  the strip and read r up to n_o rows beyond it, i.e. inside the second
  ghost row -- so with two ghost rows of r, every correction landing on an
  owned row is exact (the outer ghost row's windows wrap onto garbage, but
  they only touch ghost rows);
* restriction of owned coarse rows reads the element row below; the
  prolongation of owned fine rows reads the coarse vertex row above.

Ghost rows are refreshed by row-slab exchanges with the two neighbours (the
layout is row-major, so a slab is contiguous: no packing), inner products
are summed over owned rows and all-reduced, and the singular p = 1 coarse
problem is all-gathered and solved redundantly on every rank (it is tiny),
each rank keeping its window of the solution.  Redundant work: 2G/s extra
element rows per strip (12% at s = 32).

The driver is written against two small interfaces so the same code runs
(a) one process per GPU over NCCL (``TorchTransport``), (b) CPU gloo ranks
in the tests with an oracle engine, and (c) several ranks emulated by
threads on one GPU (``ThreadTransport``) for single-device validation.
"""

from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass

import numpy as np

from .metrics import ConvergenceReport

G = 2  # ghost element rows on each side


@dataclass(frozen=True)
class StripPlan:
    n_x: int
    n_y: int
    l_x: float
    l_y: float
    world: int
    rank: int

    def __post_init__(self):
        if self.n_y % self.world:
            raise ValueError(f"{self.n_y} element rows do not split into {self.world} strips")
        if self.n_y // self.world < 1:
            raise ValueError("empty strip")

    @property
    def s(self) -> int:
        return self.n_y // self.world

    @property
    def ey0(self) -> int:
        return self.rank * self.s

    @property
    def local_ny(self) -> int:
        return self.s + 2 * G

    @property
    def dy(self) -> float:
        return self.l_y / self.n_y

    def local_mesh_args(self):
        return (self.n_x, self.local_ny, self.l_x, self.dy * self.local_ny)

    def own(self, p: int) -> slice:
        """Owned node rows in the local array of level p."""
        return slice(G * p, (G + self.s) * p)

    def global_rows(self, p: int) -> np.ndarray:
        """Global node row of every local row of level p (periodic)."""
        N_y = p * self.n_y
        return (np.arange(p * self.local_ny) + (self.ey0 - G) * p) % N_y

    def below(self) -> int:
        return (self.rank - 1) % self.world

    def above(self) -> int:
        return (self.rank + 1) % self.world


# ---------------------------------------------------------------------------
# transports


class TorchTransport:
    """torch.distributed point-to-point + collectives (NCCL for CUDA tensors,
    gloo for CPU tensors)."""

    def __init__(self, plan: StripPlan, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.plan = plan
        self.group = group
        # gloo cannot move CUDA tensors point-to-point: stage through the host
        self.host_staged = dist.get_backend(group) != "nccl"

    def exchange(self, t, p: int, k: int):
        """Fill k ghost element rows on each side of t (level p) from the neighbours."""
        import torch
        pl = self.plan
        own = pl.own(p)
        lo, hi = own.start, own.stop
        R = k * p
        if pl.world == 1:
            t[lo - R:lo] = t[hi - R:hi]
            t[hi:hi + R] = t[lo:lo + R]
            return
        dist = self.dist
        send_down = t[lo:lo + R].contiguous()
        send_up = t[hi - R:hi].contiguous()
        if self.host_staged and t.is_cuda:
            send_down, send_up = send_down.cpu(), send_up.cpu()
        recv_top = torch.empty_like(send_down)
        recv_bot = torch.empty_like(send_down)
        ops = [dist.P2POp(dist.isend, send_down, pl.below(), self.group),
               dist.P2POp(dist.isend, send_up, pl.above(), self.group),
               dist.P2POp(dist.irecv, recv_top, pl.above(), self.group),
               dist.P2POp(dist.irecv, recv_bot, pl.below(), self.group)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        t[hi:hi + R] = recv_top
        t[lo - R:lo] = recv_bot

    def allreduce(self, x: float) -> float:
        import torch
        dev = "cpu" if self.host_staged else "cuda"
        v = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(v, group=self.group)
        return float(v.item())

    def allgather_rows(self, own, full):
        """full[(N_y, N_x)] <- concatenation of every rank's owned rows `own`."""
        import torch
        src = own.contiguous()
        if self.host_staged and src.is_cuda:
            src = src.cpu()
        parts = [torch.empty_like(src) for _ in range(self.plan.world)]
        self.dist.all_gather(parts, src, group=self.group)
        full.copy_(torch.cat(parts, 0))


class ThreadTransport:
    """Several ranks emulated by threads of one process (one GPU): exchanges
    are device copies between the ranks' arrays between barriers."""

    def __init__(self, plan: StripPlan, shared):
        self.plan = plan
        self.sh = shared  # dict with 'barrier', 'slots'

    def _sync(self):
        import torch
        torch.cuda.synchronize()
        self.sh["barrier"].wait()

    def exchange(self, t, p: int, k: int):
        pl = self.plan
        own = pl.own(p)
        lo, hi = own.start, own.stop
        R = k * p
        self.sh["slots"][pl.rank] = t
        self._sync()
        below = self.sh["slots"][pl.below()]
        above = self.sh["slots"][pl.above()]
        top = above[lo:lo + R].clone()
        bot = below[hi - R:hi].clone()
        self._sync()
        t[hi:hi + R] = top
        t[lo - R:lo] = bot
        self._sync()

    def allreduce(self, x: float) -> float:
        self.sh["slots"][self.plan.rank] = x
        self._sync()
        v = math.fsum(self.sh["slots"][r] for r in range(self.plan.world))
        self._sync()
        return v

    def allgather_rows(self, own, full):
        import torch
        self.sh["slots"][self.plan.rank] = own
        self._sync()
        parts = [self.sh["slots"][r] for r in range(self.plan.world)]
        full.copy_(torch.cat(parts, 0))
        self._sync()


def run_threads(world: int, fn):
    """Run fn(rank, shared) on `world` threads (emulated ranks); returns results."""
    shared = {"barrier": threading.Barrier(world), "slots": [None] * world}
    out = [None] * world
    err = []

    def body(r):
        try:
            out[r] = fn(r, shared)
        except BaseException as e:  # surface the first failure
            err.append(e)
            shared["barrier"].abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


# ---------------------------------------------------------------------------
# the strip-parallel algorithm (engine-agnostic)


class StripSolver:
    """V-cycle, MG and MGCG on one rank's strip.

    ``engine`` provides, per level l (0 = p=1 coarse), on LOCAL arrays:
      orders            list of level orders
      n_pre, n_post     smoothing counts per level
      zeros(l)          new local array
      residual(l, u, f, out)   out = f - A u     (f None: out = A u)
      correct(l, r, u, zero)   u += M r  (zero: u := M r)
      restrict(l, fine, out)   out (level l-1) = P^T fine
      prolong_add(l, coarse, fine)
      coarse_full(f0_full) -> u0_full            (global p=1 solve)
      full_zeros0()     new global p=1 array
      local_dot(a, b)   sum over owned rows (caller passes own slices)
      copy(dst, src)
    """

    def __init__(self, plan: StripPlan, engine, transport):
        self.plan, self.eng, self.tr = plan, engine, transport
        self.L = len(engine.orders) - 1

    # -- helpers
    def own(self, l):
        return self.plan.own(self.eng.orders[l])

    def dot(self, a, b, l=None):
        l = self.L if l is None else l
        o = self.own(l)
        return self.tr.allreduce(self.eng.local_dot(a[o], b[o]))

    def _smooth(self, l, u, f, n_it, zero):
        e, p = self.eng, self.eng.orders[l]
        for it in range(n_it):
            z = zero and it == 0
            if z:
                self.tr.exchange(f, p, G)          # r = f needs 2 ghost rows for the windows
                e.correct(l, f, u, True)
            else:
                r = e.work(l)
                self.tr.exchange(u, p, 1)
                e.residual(l, u, f, r)
                self.tr.exchange(r, p, G)
                e.correct(l, r, u, False)

    def v_cycle(self, u, f, u_zero=False):
        """Algorithm 3 (multigrid.py:231-251) on the strip; u updated in place."""
        e = self.eng
        L = self.L
        us, fs = e.us, e.fs
        us[L], fs[L] = u, f
        for l in range(L, 0, -1):
            p = e.orders[l]
            zero = u_zero if l == L else True
            if e.n_pre[l]:
                self._smooth(l, us[l], fs[l], e.n_pre[l], zero)
                zero = False
            elif zero:
                e.fill_zero(us[l])
            r = e.work(l)
            if zero:
                e.copy(r, fs[l])
            else:
                self.tr.exchange(us[l], p, 1)
                e.residual(l, us[l], fs[l], r)
            self.tr.exchange(r, p, 1)
            e.restrict(l, r, fs[l - 1])
        # replicated coarse solve
        p0 = e.orders[0]
        f0_full = e.full_zeros0()
        self.tr.allgather_rows(fs[0][self.own(0)], f0_full)
        u0_full = e.coarse_full(f0_full)
        e.copy(us[0], u0_full[self.plan.global_rows(p0)])
        for l in range(1, L + 1):
            self.tr.exchange(us[l - 1], e.orders[l - 1], 1)
            e.prolong_add(l, us[l - 1], us[l])
            if e.n_post[l]:
                self._smooth(l, us[l], fs[l], e.n_post[l], False)
        return u

    def _norm(self, r):
        return math.sqrt(self.dot(r, r))

    def solve_mg(self, f, u, tol=1e10, max_cycles=200):
        """krylov.py:49-67 on strips; f, u local (u = initial guess, updated)."""
        t0 = time.perf_counter()
        e, L = self.eng, self.L
        r = e.zeros(L)
        p = e.orders[L]
        self.tr.exchange(u, p, 1)
        e.residual(L, u, f, r)
        res = [self._norm(r)]
        r_max = res[0] / tol
        ok = res[0] <= r_max
        cycles = 0
        while not ok and cycles < max_cycles:
            self.v_cycle(u, f)
            cycles += 1
            self.tr.exchange(u, p, 1)
            e.residual(L, u, f, r)
            res.append(self._norm(r))
            ok = res[-1] <= r_max
        return u, ConvergenceReport(res, ok, cycles, time.perf_counter() - t0)

    def solve_mgcg(self, f, u, tol=1e10, max_cycles=200):
        """krylov.py:70-115 on strips (beta = z^T (r - r_old) / delta as coded)."""
        t0 = time.perf_counter()
        e, L = self.eng, self.L
        p_ = e.orders[L]
        r = e.zeros(L)
        self.tr.exchange(u, p_, 1)
        e.residual(L, u, f, r)
        res = [self._norm(r)]
        r_max = res[0] / tol
        ok = res[0] <= r_max
        broke = False
        cycles = 0
        if not ok:
            d = e.zeros(L)
            self.v_cycle(d, e.clone(r), u_zero=True)
            delta = self.dot(d, r)
            r_old = None
            q = e.zeros(L)
            for _ in range(max_cycles):
                self.tr.exchange(d, p_, 1)
                e.residual(L, d, None, q)
                pq = self.dot(d, q)
                if pq <= 0.0:
                    broke = True
                    break
                alpha = delta / pq
                e.axpy(alpha, d, u)
                r_new = e.clone(r)
                e.axpy(-alpha, q, r_new)
                r_prev, r = r, r_new
                cycles += 1
                res.append(self._norm(r))
                if res[-1] <= r_max:
                    ok = True
                    break
                z = e.zeros(L)
                self.v_cycle(z, e.clone(r), u_zero=True)
                diff = e.clone(r)
                if r_old is not None:
                    e.axpy(-1.0, r_old, diff)
                beta = self.dot(z, diff) / delta
                e.xpby(z, beta, d)              # d = z + beta d
                delta = self.dot(z, r)
                r_old = r
        rep = ConvergenceReport(res, ok, cycles, time.perf_counter() - t0)
        rep.breakdown = broke
        return u, rep


# ---------------------------------------------------------------------------
# GPU engine: the library's kernels on the local mesh


class GpuEngine:
    """Per-level device handles built on the rank's local (strip + ghosts) mesh."""

    def __init__(self, plan: StripPlan, p: int, rule, kind="w5", n_pre=1, n_post=0, orders=None,
                 nu_hat=None, nu_shift=0.2, coarse=None, coarse_tol=1e-12):
        import torch
        from . import multigrid as MG
        from .mesh import MeshConfig
        from .operators import diffusivity_field
        self.torch = torch
        self.plan = plan
        lm = MeshConfig(*plan.local_mesh_args())
        gm = MeshConfig(plan.n_x, plan.n_y, plan.l_x, plan.l_y)
        # the local hierarchy: same kernels on the local periodic mesh (its own
        # coarse level is never used: the coarse problem is solved globally)
        if nu_hat is None:
            self.h = MG.build_hierarchy(lm, p, rule, weight=kind, n_pre=n_pre, n_post=n_post, orders=orders,
                                        coarse="cg", coarse_tol=coarse_tol)
        else:  # nu sampled at GLOBAL coordinates
            self.h = _local_diffusion_hierarchy(plan, lm, gm, p, rule, kind, n_pre, n_post, orders, nu_hat,
                                                nu_shift, coarse_tol, diffusivity_field)
        levels = self.h.levels
        self.orders = [lv.basis.p for lv in levels]
        self.n_pre = [lv.n_pre for lv in levels]
        self.n_post = [lv.n_post for lv in levels]
        self.us = [lv.u for lv in levels]
        self.fs = [lv.f for lv in levels]
        self._work = [lv.work for lv in levels]
        # global p=1 coarse problem, replicated on every rank
        self.hc = _coarse_only(gm, nu_hat, nu_shift, coarse, coarse_tol)

    def zeros(self, l):
        return self.torch.zeros(self.h.levels[l].op.layout.shape, dtype=self.torch.float64, device="cuda")

    def work(self, l):
        return self._work[l]

    def clone(self, a):
        return a.clone()

    def copy(self, dst, src):
        dst.copy_(src)

    def fill_zero(self, a):
        a.zero_()

    def residual(self, l, u, f, out):
        self.h.levels[l].op.residual_into(u, f, out)

    def correct(self, l, r, u, zero):
        from . import _native as N
        lv = self.h.levels[l]
        N.check(N.lib().smg_schwarz_smooth(lv.smoother._h.raw, lv.op._handle.raw, N.ptr(u), N.ptr(r),
                                           N.ptr(self._work[l]), N.ptr(lv.smoother.ring), 1, 1 if zero else 0,
                                           N.stream())
                if zero else N.lib().smg_schwarz_correct(lv.smoother._h.raw, N.ptr(r), N.ptr(u),
                                                         N.ptr(lv.smoother.ring), N.stream()),
                "strip correct")

    def restrict(self, l, fine, out):
        from . import _native as N
        N.check(N.lib().smg_restrict(self.h.levels[l].transfer.handle.raw, N.ptr(fine), N.ptr(out), N.stream()),
                "strip restrict")

    def prolong_add(self, l, coarse, fine):
        from . import _native as N
        N.check(N.lib().smg_prolongate(self.h.levels[l].transfer.handle.raw, N.ptr(coarse), N.ptr(fine), 1,
                                       N.stream()), "strip prolong")

    def full_zeros0(self):
        return self.torch.zeros((self.plan.n_y, self.plan.n_x), dtype=self.torch.float64, device="cuda")

    def coarse_full(self, f0_full):
        from .multigrid import coarse_solve
        return coarse_solve(self.hc, f0_full)

    def local_dot(self, a, b):
        return float(self.torch.sum(a * b).item())

    def axpy(self, alpha, x, y):
        y.add_(x, alpha=alpha)

    def xpby(self, x, beta, y):
        y.mul_(beta).add_(x)


def _local_diffusion_hierarchy(plan, lm, gm, p, rule, kind, n_pre, n_post, orders, nu_hat, nu_shift,
                               coarse_tol, diffusivity_field):
    """Diffusion hierarchy on the local mesh with nu sampled at GLOBAL coordinates."""
    import torch
    from . import multigrid as MG
    from .basis import gll_basis, interp_matrix
    from .mesh import layout_for
    from .operators import DiffusionOperator
    from .schwarz import AdditiveSchwarz
    if orders is None:
        orders = [1 << l for l in range(p.bit_length())]
    levels = []
    depth = len(orders) - 1
    for l, p_l in enumerate(orders):
        b = gll_basis(p_l)
        nu_g = diffusivity_field(gm, b, nu_hat, nu_shift)
        nu_l = nu_g[plan.global_rows(p_l)]
        op = DiffusionOperator(b, lm, nu_l)
        lay = layout_for(lm, p_l)
        if l == 0:
            lv = MG.Level(l, b, op, None, 0, 0, 0)
        else:
            n_o = rule.layers(p_l)
            sm = AdditiveSchwarz(b, lay, lm.dx, lm.dy, n_o, kind, nu_bar=op.element_mean_nu())
            lv = MG.Level(l, b, op, sm, n_pre, n_post, n_o)
            lv.transfer = MG._Transfer(orders[l - 1], p_l, lm.n_x, lm.n_y, interp_matrix(levels[-1].basis, b).matrix)
        lv.u = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
        lv.f = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
        lv.work = torch.empty(lay.shape, dtype=torch.float64, device="cuda")
        levels.append(lv)
    return MG.MultigridHierarchy(lm, levels, coarse_tol=coarse_tol, coarse="cg")


def _coarse_only(gm, nu_hat, nu_shift, coarse, coarse_tol):
    """A hierarchy holding only the global p=1 level (for coarse_solve)."""
    import torch
    from . import multigrid as MG
    from .basis import gll_basis
    from .operators import DiffusionOperator, PoissonOperator, diffusivity_field
    b = gll_basis(1)
    op = PoissonOperator(b, gm) if nu_hat is None else DiffusionOperator(b, gm, diffusivity_field(gm, b, nu_hat, nu_shift))
    lv = MG.Level(0, b, op, None, 0, 0, 0)
    lv.u = torch.zeros(op.layout.shape, dtype=torch.float64, device="cuda")
    lv.f = torch.zeros(op.layout.shape, dtype=torch.float64, device="cuda")
    if coarse is None:
        coarse = "pinv" if nu_hat is None else "pcg"
    return MG.MultigridHierarchy(gm, [lv], coarse_tol=coarse_tol, coarse=coarse)


def local_window(plan: StripPlan, full, p: int):
    """The rank's local (strip + ghosts) rows of a global level-p array."""
    return full[plan.global_rows(p)]
