"""Outer solvers: stand-alone MG and inexact MG-preconditioned CG (reference krylov.py).

All vectors live on the device; the CG scalars (delta, p.q, ||r||^2, beta)
stay in a device array and are combined by the BLAS-1 kernels, so the only
host synchronisation per cycle is the read of ||r|| (and the breakdown
flag) that the reference's convergence test needs.
"""

from __future__ import annotations

import math
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


def _start(h, f, cfg, u0):
    shape = h.top.op.layout.shape
    f = to_device(f, shape)
    u = to_device(random_initial_guess(h, cfg.seed) if u0 is None else u0, shape).clone()
    return f, u


def solve_mg(h: MultigridHierarchy, f, cfg: SolveConfig, u0=None):
    """Repeated V-cycles with per-cycle residual norms (krylov.py:49-67)."""
    t0 = time.perf_counter()
    h.reset_smoothers()
    op = h.top.op
    f, u = _start(h, f, cfg, u0)
    r = torch.empty_like(u)
    s = _Scalars()
    op.residual_into(u, f, r, norm2=s.dev[2:3])
    host, _ = s.read()
    res = [math.sqrt(float(host[2]))]
    r_max = res[0] / cfg.tol_reduction
    converged = res[0] <= r_max
    cycles = 0
    while not converged and cycles < cfg.max_cycles:
        u = _v_cycle(h, u, f)
        cycles += 1
        op.residual_into(u, f, r, norm2=s.dev[2:3])
        host, _ = s.read()
        res.append(math.sqrt(float(host[2])))
        converged = res[-1] <= r_max
    return u, ConvergenceReport(res, converged, cycles, time.perf_counter() - t0)


def solve_mgcg(h: MultigridHierarchy, f, cfg: SolveConfig, u0=None):
    """Inexact MG-preconditioned CG, Polak-Ribiere beta = z^T(r - r_old)/delta
    as coded at krylov.py:108 (krylov.py:70-115)."""
    t0 = time.perf_counter()
    h.reset_smoothers()
    lib = N.lib()
    op = h.top.op
    f, u = _start(h, f, cfg, u0)
    n = u.numel()
    r_cur = torch.empty_like(u)
    r_new = torch.empty_like(u)
    p = torch.empty_like(u)
    q = torch.empty_like(u)
    z = torch.empty_like(u)
    ws = h.reduce_ws
    s = _Scalars()
    st = N.stream()
    op.residual_into(u, f, r_cur, norm2=s.dev[2:3])
    host, _ = s.read()
    res = [math.sqrt(float(host[2]))]
    r_max = res[0] / cfg.tol_reduction
    breakdown = False
    converged = res[0] <= r_max
    cycles = 0
    if not converged:
        _v_cycle(h, p, r_cur, u_zero=True)
        N.check(lib.smg_dot(N.ptr(p), N.ptr(r_cur), n, N.ptr(s.dev[0:1]), N.ptr(ws), st), "dot")
        for it in range(cfg.max_cycles):
            op.residual_into(p, None, q)
            N.check(lib.smg_dot(N.ptr(p), N.ptr(q), n, N.ptr(s.dev[1:2]), N.ptr(ws), st), "dot")
            N.check(lib.smg_cg_update2(N.ptr(u), N.ptr(r_cur), N.ptr(r_new), N.ptr(p), N.ptr(q), n,
                                       N.ptr(s.dev), N.ptr(s.flag), N.ptr(ws), st), "cg_update")
            host, flag = s.read()
            if flag:
                breakdown = True
                break
            cycles += 1
            res.append(math.sqrt(float(host[2])))
            if res[-1] <= r_max:
                converged = True
                break
            _v_cycle(h, z, r_new, u_zero=True)
            N.check(lib.smg_cg_beta(N.ptr(z), N.ptr(r_new), N.ptr(r_cur) if it > 0 else None, n,
                                    N.ptr(s.dev), N.ptr(ws), st), "cg_beta")
            N.check(lib.smg_cg_direction(N.ptr(p), N.ptr(z), n, N.ptr(s.dev), st), "cg_direction")
            r_cur, r_new = r_new, r_cur
    report = ConvergenceReport(res, converged, cycles, time.perf_counter() - t0)
    report.breakdown = breakdown
    return u, report
