"""Polynomial multigrid on the device (reference multigrid.py).

Levels p_l = 2^l (or an explicit ``orders`` list such as (1, 3, 6, 12, 24)).
Per level the device holds u_l, f_l and one work field; transfers are
element-local sum-factorized kernels (no dense global P), the V-cycle
(Alg. 3) is a sequence of stream-ordered launches with no host sync, and
the singular p = 1 problem is solved either by

* ``coarse="pinv"`` (default for Poisson): the exact pseudo-inverse of the
  periodic p=1 operator by global fast diagonalization -- the quantity the
  reference's CG approximates to 1e-12 (checked in the reference against
  ``np.linalg.pinv``, test_multigrid.py:102-113); graph-capturable; or
* ``coarse="pcg"`` (default for diffusion): CG on the variable-coefficient
  p=1 operator preconditioned by the 1/mean(nu)-scaled constant-coefficient
  pseudo-inverse -- same projections and 1e-12 stopping test as the
  reference, ~tens instead of thousands of iterations; or
* ``coarse="cg"`` (the parity mode): the reference's own plain CG
  (multigrid.py:196-228) on the device.
"""

from __future__ import annotations

import ctypes as C
import logging
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .basis import Basis1D, gll_basis, interp_matrix
from .mesh import MeshConfig, layout_for
from .operators import DiffusionOperator, PoissonOperator, diffusivity_field, diffusivity_field_device, to_device
from .schwarz import AdditiveSchwarz, MultiplicativeSchwarz, SweepCounter, WeightKind

log = logging.getLogger(__name__)

__all__ = ["OverlapRule", "Level", "LevelConfig", "MultigridHierarchy", "build_hierarchy",
           "prolongate", "restrict_residual", "coarse_solve", "v_cycle"]


@dataclass(frozen=True)
class OverlapRule:
    """Per-level overlap layers: fixed, floor(p/8), ceil(p/8), ceil(p/2) (multigrid.py:28-54)."""
    name: str
    k: int = 0

    def layers(self, p_l: int) -> int:
        if self.name == "fixed":
            n_o = self.k
        elif self.name == "floorp8":
            n_o = p_l // 8
        elif self.name == "ceilp8":
            n_o = -(-p_l // 8)
        elif self.name == "ceilp2":
            n_o = -(-p_l // 2)
        else:
            raise ValueError(f"unknown overlap rule {self.name!r}")
        return int(min(max(n_o, 0), p_l - 1))

    @classmethod
    def parse(cls, text: str) -> "OverlapRule":
        if text.startswith("fixed:"):
            return cls("fixed", int(text.split(":", 1)[1]))
        if text in ("floorp8", "ceilp8", "ceilp2"):
            return cls(text)
        raise ValueError(f"unknown overlap rule {text!r}")


@dataclass(eq=False)
class Level:
    """One level (multigrid.py:57-70); ``transfer`` replaces the dense px/py."""
    l: int
    basis: Basis1D
    op: object
    smoother: AdditiveSchwarz | MultiplicativeSchwarz | None
    n_pre: int
    n_post: int
    n_o: int
    transfer: object = None
    u: torch.Tensor = field(default=None, repr=False)
    f: torch.Tensor = field(default=None, repr=False)
    work: torch.Tensor = field(default=None, repr=False)


@dataclass(eq=False)
class LevelConfig:
    l: int
    p_l: int
    n_pre: int
    n_post: int
    n_o: int


class _Transfer:
    """Device handle for the level l-1 <-> l transfers."""

    def __init__(self, p_c, p_f, n_x, n_y, J):
        raw = C.c_void_p()
        j = N.host(J)
        N.check(N.lib().smg_transfer_create(C.byref(raw), p_c, p_f, n_x, n_y, j[1]), "transfer_create")
        self.handle = N.Handle(raw, "smg_transfer_destroy")
        self.J = np.asarray(J)
        # ring workspace of the halo-free restriction (caller-owned scratch, include/smg.h)
        nws = int(N.lib().smg_transfer_ws_doubles(raw))
        self.ws = torch.zeros(nws, dtype=torch.float64, device="cuda") if nws else None

    def ws_ptr(self):
        return N.ptr(self.ws) if self.ws is not None else None


class _CoarsePinv:
    def __init__(self, mesh: MeshConfig):
        raw = C.c_void_p()
        N.check(N.lib().smg_coarse_create(C.byref(raw), mesh.n_x, mesh.n_y, float(mesh.dx), float(mesh.dy)),
                "coarse_create")
        self.handle = N.Handle(raw, "smg_coarse_destroy")
        self.ws = torch.empty(N.lib().smg_coarse_ws_doubles(raw), dtype=torch.float64, device="cuda")


class MultigridHierarchy:
    """multigrid.py:84-109 plus the device workspaces."""

    def __init__(self, mesh: MeshConfig, levels: list, coarse_tol: float = 1e-12,
                 sweep_counter: SweepCounter | None = None, coarse: str = "pinv"):
        self.mesh = mesh
        self.levels = levels
        self.coarse_tol = coarse_tol
        self.coarse_cg_exhausted = 0
        self.coarse_iterations: list[int] = []
        self.sweep_counter = sweep_counter
        if coarse not in ("pinv", "cg", "pcg"):
            raise ValueError(f"unknown coarse solver {coarse!r}")
        diffusion = isinstance(levels[0].op, DiffusionOperator)
        if coarse == "pinv" and diffusion:
            raise ValueError("coarse='pinv' is the constant-coefficient pseudo-inverse; use 'pcg' or 'cg' for diffusion")
        self.coarse = coarse
        self._pinv = _CoarsePinv(mesh) if coarse in ("pinv", "pcg") else None
        # PCG preconditioner scale: 1 / mean(nu) on the coarse nodes
        self._pcg_scale = 1.0 / float(np.mean(levels[0].op.nu)) if diffusion else 1.0
        n0 = levels[0].op.layout.size
        self._cg_ws = None
        self._n0 = n0
        self.reduce_ws = torch.zeros(N.lib().smg_reduce_ws_doubles(), dtype=torch.float64, device="cuda")

    def reset_smoothers(self):
        if self.sweep_counter is not None:
            self.sweep_counter.reset()

    @property
    def depth(self) -> int:
        return len(self.levels) - 1

    @property
    def top(self) -> Level:
        return self.levels[-1]

    def level_configs(self) -> list[LevelConfig]:
        return [LevelConfig(lv.l, lv.basis.p, lv.n_pre, lv.n_post, lv.n_o) for lv in self.levels]


def build_hierarchy(mesh: MeshConfig, p: int, rule: OverlapRule, smoother: str = "add",
                    weight: WeightKind = WeightKind.QUINTIC, n_pre: int = 1, n_post: int = 0,
                    variable: bool = False, nu_hat: float | None = None, nu_shift: float = 0.2,
                    coarse_tol: float = 1e-12, *, orders=None, coarse: str | None = None
                    ) -> MultigridHierarchy:
    """All levels, smoothers and transfers (multigrid.py:127-177).

    Extra keywords (defaults keep the reference behaviour):
      orders -- explicit level orders, e.g. (1, 3, 6, 12, 24) for p=24, which
                the reference can only assemble by hand (multigrid.py:139-140);
      coarse -- "pinv" | "pcg" | "cg" (see module docstring).
    """
    if orders is None:
        if p < 2 or (p & (p - 1)) != 0:
            raise ValueError(f"top-level order must be a power of two >= 2, got {p}")
        orders = [1 << l for l in range(p.bit_length())]
    else:
        orders = [int(o) for o in orders]
        if orders[0] != 1 or orders[-1] != p or any(b <= a for a, b in zip(orders, orders[1:])):
            raise ValueError(f"orders must rise from 1 to p={p}, got {orders}")
    if smoother not in ("add", "mult"):
        raise ValueError(f"smoother must be 'add' or 'mult', got {smoother!r}")
    counter = SweepCounter() if smoother == "mult" else None   # multigrid.py:144
    if coarse is None:
        coarse = "pinv" if nu_hat is None else "pcg"
    depth = len(orders) - 1
    levels: list[Level] = []
    for l, p_l in enumerate(orders):
        basis = gll_basis(p_l)
        layout = layout_for(mesh, p_l)
        if nu_hat is None:
            op = PoissonOperator(basis, mesh)
            nu_bar = None
        else:
            op = DiffusionOperator(basis, mesh, diffusivity_field_device(mesh, basis, nu_hat, nu_shift))
            nu_bar = op.element_mean_nu()
        if l == 0:
            lv = Level(l, basis, op, None, 0, 0, 0)
        else:
            n_o = rule.layers(p_l)
            fac = 2 ** (depth - l) if variable else 1
            if smoother == "add":
                sm = AdditiveSchwarz(basis, layout, mesh.dx, mesh.dy, n_o, weight, nu_bar=nu_bar)
            else:
                sm = MultiplicativeSchwarz(basis, layout, mesh.dx, mesh.dy, n_o, nu_bar=nu_bar, counter=counter)
            lv = Level(l, basis, op, sm, n_pre * fac, n_post * fac, n_o)
            J = interp_matrix(levels[l - 1].basis, basis).matrix
            lv.transfer = _Transfer(orders[l - 1], p_l, mesh.n_x, mesh.n_y, J)
        lv.u = torch.zeros(layout.shape, dtype=torch.float64, device="cuda")
        lv.f = torch.zeros(layout.shape, dtype=torch.float64, device="cuda")
        lv.work = torch.empty(layout.shape, dtype=torch.float64, device="cuda")
        levels.append(lv)
    return MultigridHierarchy(mesh, levels, coarse_tol=coarse_tol, coarse=coarse, sweep_counter=counter)


def prolongate(h: MultigridHierarchy, l: int, coarse) -> torch.Tensor:
    """P_l u_c as a new level-l field (multigrid.py:180-185)."""
    if not 1 <= l <= h.depth:
        raise ValueError(f"level must be in [1, {h.depth}], got {l}")
    lv = h.levels[l]
    uc = to_device(coarse, h.levels[l - 1].op.layout.shape)
    out = torch.empty(lv.op.layout.shape, dtype=torch.float64, device="cuda")
    N.check(N.lib().smg_prolongate(lv.transfer.handle.raw, N.ptr(uc), N.ptr(out), 0, N.stream()), "prolongate")
    return out


def restrict_residual(h: MultigridHierarchy, l: int, fine) -> torch.Tensor:
    """P_l^T f as a new level-(l-1) field (multigrid.py:188-193)."""
    if not 1 <= l <= h.depth:
        raise ValueError(f"level must be in [1, {h.depth}], got {l}")
    lv = h.levels[l]
    ff = to_device(fine, lv.op.layout.shape)
    out = torch.empty(h.levels[l - 1].op.layout.shape, dtype=torch.float64, device="cuda")
    N.check(N.lib().smg_restrict_ws(lv.transfer.handle.raw, N.ptr(ff), N.ptr(out), lv.transfer.ws_ptr(), N.stream()),
            "restrict")
    return out


def _coarse_into(h: MultigridHierarchy, f0: torch.Tensor, u0: torch.Tensor):
    lib = N.lib()
    if h.coarse == "pinv":
        N.check(lib.smg_coarse_pinv(h._pinv.handle.raw, N.ptr(f0), N.ptr(u0), N.ptr(h._pinv.ws), N.stream()),
                "coarse_pinv")
        return
    cap = 10 * h._n0
    it = C.c_int(0)
    if h.coarse == "pcg":
        if h._cg_ws is None:
            h._cg_ws = torch.zeros(lib.smg_coarse_pcg_ws_doubles(h._pinv.handle.raw), dtype=torch.float64,
                                   device="cuda")
        N.check(lib.smg_coarse_pcg(h.levels[0].op._handle.raw, h._pinv.handle.raw, N.ptr(f0), N.ptr(u0),
                                   N.ptr(h._cg_ws), float(h.coarse_tol), cap, float(h._pcg_scale), C.byref(it),
                                   N.stream()), "coarse_pcg")
    else:
        if h._cg_ws is None:
            h._cg_ws = torch.zeros(lib.smg_coarse_cg_ws_doubles(h._n0), dtype=torch.float64, device="cuda")
        N.check(lib.smg_coarse_cg(h.levels[0].op._handle.raw, N.ptr(f0), N.ptr(u0), N.ptr(h._cg_ws),
                                  float(h.coarse_tol), cap, C.byref(it), N.stream()), "coarse_cg")
    h.coarse_iterations.append(abs(it.value))
    if it.value < 0:
        h.coarse_cg_exhausted += 1
        log.warning("coarse CG hit its iteration cap (%d); possible ill-conditioning", cap)


def coarse_solve(h: MultigridHierarchy, f0) -> torch.Tensor:
    """Null-space-projected solve of the singular p = 1 problem (multigrid.py:218-228)."""
    f0 = to_device(f0, h.levels[0].op.layout.shape)
    u0 = torch.empty_like(f0)
    _coarse_into(h, f0, u0)
    return u0


_NVTX = os.environ.get("SMG_NVTX", "0") == "1"


class _Range:
    """NVTX range (SMG_NVTX=1; a no-op otherwise) so that nsys / ncu --nvtx
    timelines show the V-cycle's levels and phases by name."""
    __slots__ = ("name",)

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        if _NVTX:
            torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *exc):
        if _NVTX:
            torch.cuda.nvtx.range_pop()


def _chain_levels(h: MultigridHierarchy) -> int:
    """Levels 1..K whose prolongations run as one launch (smg_prolongate_chain):
    orders 2^l up to p = 16 and no post-smoothing below level K.  Cached per
    hierarchy together with the ctypes argument arrays (pointers into the
    level fields, which the V-cycle keeps, except the caller's top u)."""
    import ctypes as C
    top_ptr = h.top.u.data_ptr() if h.top.u is not None else 0
    # opt-in (SMG_CHAIN=1): bitwise equal, but measured no faster than the
    # per-level launches with PDL on B200 (C2 V-cycle 110.6 vs 110.6 us, C3
    # 1231 vs 1216 us)
    key = (top_ptr, os.environ.get("SMG_CHAIN", "0"))
    if getattr(h, "_chain_key", None) == key:
        return h._chain_K
    K = 0
    if key[1] == "1":
        for l in range(1, min(h.depth, 4) + 1):
            lv = h.levels[l]
            if lv.basis.p != (1 << l) or h.levels[l - 1].basis.p != (1 << (l - 1)):
                break
            K = l
            if lv.n_post:
                break
    h._chain_K = K
    h._chain_key = key
    if K >= 2:
        h._chain_tr = (C.c_void_p * K)(*[h.levels[l].transfer.handle.raw.value for l in range(1, K + 1)])
        h._chain_u = (C.c_void_p * K)(*[h.levels[l].u.data_ptr() for l in range(1, K + 1)])
    return K


def _v_cycle(h: MultigridHierarchy, u: torch.Tensor, f: torch.Tensor, u_zero: bool = False) -> torch.Tensor:
    """Algorithm 3 on device buffers; u is updated in place.  u_zero declares
    the initial guess to be 0 (MGCG preconditioning): u's prior contents are
    never read, the top smoother uses r = f without an operator apply
    (bitwise what A 0 = 0 gives) and WRITES u = correction.  Lower levels
    always start from zero the same way (multigrid.py:240-241)."""
    lib = N.lib()
    st = N.stream()
    L = h.depth
    top = h.top
    top.u, top.f = u, f
    for l in range(L, 0, -1):
        with _Range(f"down p={h.levels[l].basis.p}"):
            lv = h.levels[l]
            zero = u_zero if l == L else True
            if zero and not lv.n_pre:
                lv.u.zero_()
            if lv.n_pre:
                if isinstance(lv.smoother, MultiplicativeSchwarz):
                    if zero:
                        lv.u.zero_()
                    lv.smoother.smooth(lv.op, lv.u, lv.f, lv.n_pre)
                else:
                    N.check(lib.smg_schwarz_smooth_ws(lv.smoother._h.raw, lv.op._handle.raw, N.ptr(lv.u),
                                                      N.ptr(lv.f), N.ptr(lv.work), N.ptr(lv.smoother.ring),
                                                      lv.op.ring_ptr(), lv.n_pre, int(zero), st), "smooth")
                zero = False
            fc = h.levels[l - 1].f
            if zero:
                N.check(lib.smg_restrict_ws(lv.transfer.handle.raw, N.ptr(lv.f), N.ptr(fc), lv.transfer.ws_ptr(), st),
                        "restrict")
            else:
                N.check(lib.smg_residual_restrict_ws(lv.transfer.handle.raw, lv.op._handle.raw, N.ptr(lv.u),
                                                     N.ptr(lv.f), N.ptr(fc), N.ptr(lv.work), lv.transfer.ws_ptr(),
                                                     lv.op.ring_ptr(), st), "residual_restrict")
    with _Range("coarse"):
        _coarse_into(h, h.levels[0].f, h.levels[0].u)
    K = _chain_levels(h)
    if K >= 2:
        # levels 1..K prolongated in one launch (n_post = 0 below level K)
        N.check(lib.smg_prolongate_chain(h._chain_tr, K, N.ptr(h.levels[0].u), h._chain_u, st), "prolongate_chain")
    else:
        K = 0
    for l in range(max(K, 1), L + 1):
        with _Range(f"up p={h.levels[l].basis.p}"):
            lv = h.levels[l]
            if l > K:
                N.check(lib.smg_prolongate(lv.transfer.handle.raw, N.ptr(h.levels[l - 1].u), N.ptr(lv.u), 1, st),
                        "prolongate")
            if lv.n_post:
                if isinstance(lv.smoother, MultiplicativeSchwarz):
                    lv.smoother.smooth(lv.op, lv.u, lv.f, lv.n_post)
                else:
                    N.check(lib.smg_schwarz_smooth_ws(lv.smoother._h.raw, lv.op._handle.raw, N.ptr(lv.u),
                                                      N.ptr(lv.f), N.ptr(lv.work), N.ptr(lv.smoother.ring),
                                                      lv.op.ring_ptr(), lv.n_post, 0, st), "smooth")
    return u


def v_cycle(h: MultigridHierarchy, u, f) -> torch.Tensor:
    """One V-cycle (multigrid.py:231-251).  A CUDA float64 ``u`` is mutated in
    place and returned (the reference's contract); numpy input is copied to
    the device and the device result returned."""
    shape = h.top.op.layout.shape
    if not (isinstance(u, torch.Tensor) and u.is_cuda and u.dtype == torch.float64 and u.is_contiguous()):
        u = to_device(u, shape).clone()
    elif tuple(u.shape) != shape:
        raise ValueError(f"field shape {tuple(u.shape)} does not match layout {shape}")
    f = to_device(f, shape)
    return _v_cycle(h, u, f)
