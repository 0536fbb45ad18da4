"""Outer solvers: stand-alone MG and inexact MG-preconditioned CG (reference krylov.py).

All vectors live on the device; the CG scalars (delta, p.q, ||r||^2, beta)
stay in a device array and are combined by the BLAS-1 kernels, so the only
host synchronisation per cycle is the read of ||r|| (and the breakdown
flag) that the reference's convergence test needs.

Between two such reads everything is stream-ordered device work; for
hierarchies whose V-cycle is graph-capturable (coarse="pinv", additive
smoother) that segment is captured once as a CUDA graph and replayed, so the
~30 launches of a cycle cost one graph launch instead of a host loop the GPU
waits on after every sync (C2 MGCG: 96 us of launch gap per 264 us cycle).
SMG_SOLVE_GRAPH=0 runs the same launches eagerly (bitwise the same results).
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .metrics import ConvergenceReport
from .multigrid import MultigridHierarchy, _v_cycle
from .operators import to_device

__all__ = ["SolveConfig", "solve", "solve_mg", "solve_mgcg", "random_initial_guess"]


@dataclass(frozen=True)
class SolveConfig:
    """krylov.py:20-33."""
    solver: str = "mg"
    tol_reduction: float = 1e10
    max_cycles: int = 200
    seed: int = 0

    def __post_init__(self):
        if self.tol_reduction <= 1.0:
            raise ValueError("tol_reduction must exceed 1")
        if self.max_cycles < 1:
            raise ValueError("max_cycles must be >= 1")
        if self.solver not in ("mg", "mgcg"):
            raise ValueError(f"unknown solver {self.solver!r}")


def random_initial_guess(h: MultigridHierarchy, seed: int) -> np.ndarray:
    """U[0,1) from numpy's PCG64 -- the reference's exact bits (krylov.py:36-39)."""
    return np.random.default_rng(seed).random(h.top.op.layout.shape)


def solve(h: MultigridHierarchy, f, cfg: SolveConfig, u0=None):
    """krylov.py:42-46; returns (u on the device, ConvergenceReport)."""
    if cfg.solver == "mg":
        return solve_mg(h, f, cfg, u0)
    return solve_mgcg(h, f, cfg, u0)


class _Scalars:
    """Device scalar block + pinned host mirror for the per-cycle read."""

    def __init__(self):
        self.dev = torch.zeros(8, dtype=torch.float64, device="cuda")
        self.flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.host = torch.zeros(8, dtype=torch.float64).pin_memory()
        self.host_flag = torch.zeros(1, dtype=torch.int32).pin_memory()

    def read(self):
        self.host.copy_(self.dev, non_blocking=True)
        self.host_flag.copy_(self.flag, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.host, int(self.host_flag[0])


def _graphable(h: MultigridHierarchy) -> bool:
    from .schwarz import MultiplicativeSchwarz
    if os.environ.get("SMG_SOLVE_GRAPH", "1") == "0" or h.coarse != "pinv":
        return False
    return not any(isinstance(lv.smoother, MultiplicativeSchwarz) for lv in h.levels[1:])


class _Segment:
    """A stream-ordered launch sequence run eagerly the first time, then
    captured as a CUDA graph and replayed (buffers must stay fixed)."""

    def __init__(self, fn, graph: bool):
        self.fn, self.graph, self.g, self.calls = fn, graph, None, 0

    def __call__(self):
        self.calls += 1
        if not self.graph or self.calls == 1:
            self.fn()            # eager first call: sets kernel attributes, allocates nothing later
            return
        if self.g is None:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self.fn()
            torch.cuda.current_stream().wait_stream(side)
            self.g = g
        self.g.replay()


class _SolveState:
    """Per-hierarchy solver workspace: the iterate, right-hand side and CG
    vectors live in fixed buffers across solve() calls, so the cycle segments
    are captured as CUDA graphs once per hierarchy and replayed by every later
    solve (the caller gets a copy of the iterate)."""

    def __init__(self, h: MultigridHierarchy):
        shape = h.top.op.layout.shape
        mk = lambda: torch.zeros(shape, dtype=torch.float64, device="cuda")  # noqa: E731
        self.u, self.f, self.r_cur, self.r_new, self.p, self.q, self.z = (mk() for _ in range(7))
        self.s = _Scalars()
        self.graph = _graphable(h)
        self.segs = {}

    def seg(self, key, fn):
        if key not in self.segs:
            self.segs[key] = _Segment(fn, self.graph)
        return self.segs[key]


def _state(h: MultigridHierarchy) -> _SolveState:
    st = getattr(h, "_solve_state", None)
    if st is None or st.graph != _graphable(h):
        st = _SolveState(h)
        h._solve_state = st
    return st


def _start(h, f, cfg, u0):
    shape = h.top.op.layout.shape
    ws = _state(h)
    ws.f.copy_(to_device(f, shape))
    ws.u.copy_(to_device(random_initial_guess(h, cfg.seed) if u0 is None else u0, shape))
    ws.s.dev.zero_()
    ws.s.flag.zero_()
    return ws.f, ws.u


def solve_mg(h: MultigridHierarchy, f, cfg: SolveConfig, u0=None):
    """Repeated V-cycles with per-cycle residual norms (krylov.py:49-67)."""
    t0 = time.perf_counter()
    h.reset_smoothers()
    op = h.top.op
    f, u = _start(h, f, cfg, u0)
    ws = _state(h)
    r = ws.r_cur
    s = ws.s
    op.residual_into(u, f, r, norm2=s.dev[2:3])
    host, _ = s.read()
    res = [math.sqrt(float(host[2]))]
    r_max = res[0] / cfg.tol_reduction
    converged = res[0] <= r_max
    cycles = 0

    def cycle():
        _v_cycle(h, u, f)
        op.residual_into(u, f, r, norm2=s.dev[2:3])
    seg = ws.seg("mg", cycle)
    while not converged and cycles < cfg.max_cycles:
        seg()
        cycles += 1
        host, _ = s.read()
        res.append(math.sqrt(float(host[2])))
        converged = res[-1] <= r_max
    return u.clone(), ConvergenceReport(res, converged, cycles, time.perf_counter() - t0)


def solve_mgcg(h: MultigridHierarchy, f, cfg: SolveConfig, u0=None):
    """Inexact MG-preconditioned CG, Polak-Ribiere beta = z^T(r - r_old)/delta
    as coded at krylov.py:108 (krylov.py:70-115)."""
    t0 = time.perf_counter()
    h.reset_smoothers()
    lib = N.lib()
    op = h.top.op
    f, u = _start(h, f, cfg, u0)
    W = _state(h)
    n = u.numel()
    r_cur, r_new, p, q, z = W.r_cur, W.r_new, W.p, W.q, W.z
    ws = h.reduce_ws
    s = W.s
    st = N.stream()
    op.residual_into(u, f, r_cur, norm2=s.dev[2:3])
    host, _ = s.read()
    res = [math.sqrt(float(host[2]))]
    r_max = res[0] / cfg.tol_reduction
    breakdown = False
    converged = res[0] <= r_max
    cycles = 0
    if not converged:
        def step(ra, rb):
            # krylov.py:91-103: q = A p, alpha = delta / p.q, u += alpha p, rb = ra - alpha q
            def run():
                st = N.stream()
                # q = A p and p . q in one call (fused in the warp-per-element Poisson kernel)
                N.check(lib.smg_op_apply_dot(op._handle.raw, N.ptr(p), N.ptr(q), N.ptr(s.dev[1:2]),
                                             N.ptr(op.partials), op.ring_ptr(), st), "apply_dot")
                N.check(lib.smg_cg_update2(N.ptr(u), N.ptr(ra), N.ptr(rb), N.ptr(p), N.ptr(q), n,
                                           N.ptr(s.dev), N.ptr(s.flag), N.ptr(ws), st), "cg_update")
            return run

        def precond(rb, ra_old):
            # krylov.py:104-110: z = V(r), beta = z.(r - r_old) / delta, delta = z.r, p = z + beta p
            def run():
                st = N.stream()
                _v_cycle(h, z, rb, u_zero=True)
                N.check(lib.smg_cg_beta(N.ptr(z), N.ptr(rb), N.ptr(ra_old) if ra_old is not None else None, n,
                                        N.ptr(s.dev), N.ptr(ws), st), "cg_beta")
                N.check(lib.smg_cg_direction(N.ptr(p), N.ptr(z), n, N.ptr(s.dev), st), "cg_direction")
            return run

        def start():
            # p = V(r0), delta = p.r0, then the first step
            st = N.stream()
            _v_cycle(h, p, r_cur, u_zero=True)
            N.check(lib.smg_dot(N.ptr(p), N.ptr(r_cur), n, N.ptr(s.dev[0:1]), N.ptr(ws), st), "dot")
            step(r_cur, r_new)()

        # segments between two host reads: the start, the first precondition
        # (r_old = 0) and the two buffer parities of the steady state
        seg = [W.seg("cg0", lambda: (precond(r_new, None)(), step(r_new, r_cur)())),
               W.seg("cg1", lambda: (precond(r_cur, r_new)(), step(r_cur, r_new)())),
               W.seg("cg2", lambda: (precond(r_new, r_cur)(), step(r_new, r_cur)()))]
        W.seg("cgs", start)()
        for it in range(cfg.max_cycles):
            host, flag = s.read()
            if flag:
                breakdown = True
                break
            cycles += 1
            res.append(math.sqrt(float(host[2])))
            if res[-1] <= r_max or it + 1 >= cfg.max_cycles:
                converged = res[-1] <= r_max
                break
            seg[0 if it == 0 else (1 if it % 2 == 1 else 2)]()
    report = ConvergenceReport(res, converged, cycles, time.perf_counter() - t0)
    report.breakdown = breakdown
    return u.clone(), report
