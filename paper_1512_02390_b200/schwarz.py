"""Weighted additive Schwarz smoother (reference schwarz.py), B200 hot path.

Host side (once per level, numpy float64): subdomain geometry, the smoothed
sign weights of Table 1, the restricted 1D patch matrices and their
generalized eigendecompositions by the reference's own cyclic Jacobi
ordering (schwarz.py:152-197), so S_x, S_y, lambda are the reference's bits.

Device side: ``AdditiveSchwarz.smooth`` runs one fused sm_100a launch per
colour class (``smg_schwarz_correct``: gather windows -> 4 contractions ->
/(lam_y (+) lam_x) -> *W -> /nu_bar -> scatter-add) after the residual
kernel.  ``FastDiagSolver.solve`` runs the same kernel on explicit blocks.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .basis import Basis1D, overlap_width
from .mesh import FieldLayout

__all__ = ["WeightKind", "SubdomainGeometry", "FastDiagSolver", "restricted_1d", "weight_value",
           "build_weight_1d", "build_weight_tensor", "build_fast_diag", "AdditiveSchwarz",
           "MultiplicativeSchwarz", "SweepCounter", "jacobi_eigh", "shape_function",
           "subdomain_geometry"]


class WeightKind(str, Enum):
    """Weighting profiles of the paper's Table 1 (schwarz.py:28-34)."""
    ARITHMETIC = "wa"
    LINEAR = "w1"
    CUBIC = "w3"
    QUINTIC = "w5"
    SEVENTH = "w7"
    TOPHAT = "wt"


_POLY = {  # odd shape-function cores on [-1, 1] (schwarz.py:37-52)
    WeightKind.LINEAR: lambda x: x,
    WeightKind.CUBIC: lambda x: (3 * x - x ** 3) / 2,
    WeightKind.QUINTIC: lambda x: (15 * x - 10 * x ** 3 + 3 * x ** 5) / 8,
    WeightKind.SEVENTH: lambda x: (35 * x - 35 * x ** 3 + 21 * x ** 5 - 5 * x ** 7) / 16,
    WeightKind.TOPHAT: np.sign,
    WeightKind.ARITHMETIC: np.zeros_like,
}


def shape_function(kind: WeightKind, x) -> np.ndarray:
    """Core profile on [-1, 1], sign(x) outside (schwarz.py:55-59)."""
    kind = WeightKind(kind)
    x = np.asarray(x, dtype=float)
    core = _POLY[kind](np.clip(x, -1.0, 1.0))
    return np.where(np.abs(x) <= 1.0, core, np.sign(x))


def weight_value(kind: WeightKind, xi, delta: float) -> np.ndarray:
    """w(xi) = [phi((xi+1)/delta) - phi((xi-1)/delta)] / 2 (schwarz.py:62-67)."""
    if delta <= 0:
        raise ValueError("overlap width must be positive")
    xi = np.asarray(xi, dtype=float)
    return 0.5 * (shape_function(kind, (xi + 1.0) / delta) - shape_function(kind, (xi - 1.0) / delta))


@dataclass(frozen=True)
class SubdomainGeometry:
    """Updated node set of one subdomain (schwarz.py:70-81)."""
    p: int
    n_o: int
    delta: float
    coords: np.ndarray

    @property
    def n_updated(self) -> int:
        return self.p + 1 + 2 * self.n_o


def subdomain_geometry(basis: Basis1D, n_o: int) -> SubdomainGeometry:
    """schwarz.py:84-90."""
    delta = overlap_width(basis, n_o)
    p = basis.p
    coords = np.concatenate([basis.nodes[p - n_o:p] - 2.0, basis.nodes, basis.nodes[1:n_o + 1] + 2.0])
    return SubdomainGeometry(p=p, n_o=n_o, delta=delta, coords=coords)


def build_weight_1d(kind: WeightKind, basis: Basis1D, geom: SubdomainGeometry) -> np.ndarray:
    """1D weights at the updated nodes (schwarz.py:93-119)."""
    kind = WeightKind(kind)
    p, n_o = geom.p, geom.n_o
    own = np.arange(geom.n_updated) - n_o
    if kind is WeightKind.ARITHMETIC:
        # 1 / (number of subdomains updating the node)  (schwarz.py:93-102)
        cover = np.floor((own + n_o) / p) - np.ceil((own - p - n_o) / p) + 1
        return 1.0 / cover.astype(int)
    w = weight_value(kind, geom.coords, geom.delta)
    w[(own > n_o) & (own < p - n_o)] = 1.0
    return w


def build_weight_tensor(kind: WeightKind, basis: Basis1D, geom: SubdomainGeometry) -> np.ndarray:
    w = build_weight_1d(kind, basis, geom)
    return np.outer(w, w)


def restricted_1d(basis: Basis1D, d: float, n_o: int):
    """Three-element periodic patch restricted to the m updated nodes
    (schwarz.py:129-149): returns (L_s, m_s)."""
    p = basis.p
    if not 0 <= n_o <= p - 1:
        raise ValueError(f"overlap layers must be in [0, {p - 1}], got {n_o}")
    q = 3 * p + 1
    L = np.zeros((q, q))
    mass = np.zeros(q)
    for off in (0, p, 2 * p):
        L[off:off + p + 1, off:off + p + 1] += (2.0 / d) * basis.stiff
        mass[off:off + p + 1] += (d / 2.0) * basis.weights
    keep = slice(p - n_o, 2 * p + n_o + 1)
    return np.ascontiguousarray(L[keep, keep]), mass[keep].copy()


def _rotate(m, i, j, c, s, axis):
    """Apply the Jacobi plane rotation to columns (axis=1) or rows (axis=0) i, j."""
    if axis == 1:
        xi, xj = m[:, i], m[:, j]
        new_i, new_j = c * xi - s * xj, s * xi + c * xj
        m[:, i], m[:, j] = new_i, new_j
    else:
        xi, xj = m[i, :], m[j, :]
        new_i, new_j = c * xi - s * xj, s * xi + c * xj
        m[i, :], m[j, :] = new_i, new_j


def jacobi_eigh(a: np.ndarray, tol: float = 1e-14, max_sweeps: int = 50):
    """Cyclic Jacobi eigensolver (schwarz.py:152-197); ascending eigenvalues.

    Same rotation formula, pivot order and stopping rules as the reference,
    so the factors (and the smoother's output) reproduce it exactly.
    """
    a = np.array(a, dtype=float)
    n = a.shape[0]
    v = np.eye(n)
    scale = np.linalg.norm(a)
    if scale == 0.0:
        return np.zeros(n), v
    for _ in range(max_sweeps):
        if np.linalg.norm(a - np.diag(np.diag(a))) < tol * scale:
            break
        for i in range(n - 1):
            for j in range(i + 1, n):
                aij = a[i, j]
                if abs(aij) < 1e-20 * scale:
                    a[i, j] = a[j, i] = 0.0
                    continue
                theta = (a[j, j] - a[i, i]) / (2.0 * aij)
                t = np.sign(theta) / (abs(theta) + np.hypot(theta, 1.0)) if theta != 0.0 else 1.0
                c = 1.0 / np.sqrt(t ** 2 + 1.0)
                s = t * c
                _rotate(a, i, j, c, s, 1)
                _rotate(a, i, j, c, s, 0)
                _rotate(v, i, j, c, s, 1)
    else:
        raise RuntimeError(f"Jacobi eigensolver did not converge within {max_sweeps} sweeps")
    lam = np.diag(a).copy()
    order = np.argsort(lam)
    return lam[order], v[:, order]


def _direction_factors(basis: Basis1D, d: float, n_o: int):
    """S = M^-1/2 Q with S^T M S = I (schwarz.py:225-232)."""
    L_s, m_s = restricted_1d(basis, d, n_o)
    inv_sqrt = 1.0 / np.sqrt(m_s)
    lam, q = jacobi_eigh(inv_sqrt[:, None] * L_s * inv_sqrt[None, :])
    if lam[0] <= 0.0:
        raise RuntimeError("restricted subdomain problem is not definite")
    return inv_sqrt[:, None] * q, lam


class FastDiagSolver:
    """Factored inverse of the tensor-product subdomain operator
    (schwarz.py:200-222).  ``solve`` runs on the device."""

    def __init__(self, S_x, S_y, lam_x, lam_y, weight=None, *, p=None, n_o=None, w1d=None):
        self.S_x, self.S_y, self.lam_x, self.lam_y, self.weight = S_x, S_y, lam_x, lam_y, weight
        self._p, self._n_o = p, n_o
        self._w1d = w1d
        self._handle = None

    def _h(self):
        if self._handle is None:
            m = self.S_x.shape[0]
            # any (p, n_o) with p + 1 + 2 n_o = m works for block mode
            p, n_o = (self._p, self._n_o) if self._p is not None else (m - 1, 0)
            w = self._w1d if self._w1d is not None else np.ones(m)
            self._handle = _make_schwarz(p, n_o, 2, 2, self.S_x, self.S_y, self.lam_x, self.lam_y, w,
                                         None, check_alias=False)
        return self._handle

    def solve(self, blocks):
        """W * (S_y (S_y^T B S_x ./ (lam_y (+) lam_x)) S_x^T) for one or many blocks."""
        lib = N.lib()
        m = self.S_x.shape[0]
        x = _as_device(blocks)
        shape = tuple(x.shape)
        if shape[-2:] != (m, m):
            raise ValueError(f"blocks must end in ({m}, {m}), got {shape}")
        xb = x.reshape(-1, m, m).contiguous()
        out = torch.empty_like(xb)
        N.check(lib.smg_fd_solve_blocks(self._h().raw, N.ptr(xb), N.ptr(out), xb.shape[0],
                                        int(self.weight is not None), N.stream()), "fd_solve")
        return out.reshape(shape)


def build_fast_diag(basis: Basis1D, dx: float, dy: float, n_o: int,
                    kind: WeightKind | None = None) -> FastDiagSolver:
    """schwarz.py:235-244."""
    S_x, lam_x = _direction_factors(basis, dx, n_o)
    S_y, lam_y = _direction_factors(basis, dy, n_o)
    weight = w1 = None
    if kind is not None:
        w1 = build_weight_1d(kind, basis, subdomain_geometry(basis, n_o))
        weight = np.outer(w1, w1)
    return FastDiagSolver(S_x, S_y, lam_x, lam_y, weight, p=basis.p, n_o=n_o, w1d=w1)


def _check_no_alias(layout: FieldLayout, n_o: int):
    """schwarz.py:247-252."""
    m = layout.p + 1 + 2 * n_o
    if m > layout.N_x or m > layout.N_y:
        raise ValueError(f"subdomain window ({m} nodes) wraps onto itself on a "
                         f"{layout.n_x}x{layout.n_y} mesh at p={layout.p}; reduce n_o")


def _as_device(a):
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    return t.to(device="cuda", dtype=torch.float64).contiguous()


def _make_schwarz(p, n_o, n_x, n_y, S_x, S_y, lam_x, lam_y, w1d, inv_nu_dev, check_alias=True):
    lib = N.lib()
    keep = [N.host(a) for a in (S_x, S_y, lam_x, lam_y, w1d, w1d)]
    raw = C.c_void_p()
    if not check_alias:
        # block mode only: use a mesh wide enough for the alias guard
        n_x = n_y = max(2, -(-(p + 1 + 2 * n_o) // max(p, 1)))
    N.check(lib.smg_schwarz_create(C.byref(raw), p, n_o, n_x, n_y, *[k[1] for k in keep],
                                   N.ptr(inv_nu_dev)), "schwarz_create")
    return N.Handle(raw, "smg_schwarz_destroy")


class AdditiveSchwarz:
    """Weighted additive Schwarz sweep over all subdomains (schwarz.py:255-275)."""

    def __init__(self, basis: Basis1D, layout: FieldLayout, dx: float, dy: float, n_o: int,
                 kind: WeightKind, nu_bar=None):
        _check_no_alias(layout, n_o)
        self.n_o = n_o
        self.layout = layout
        self.solver = build_fast_diag(basis, dx, dy, n_o, kind)
        self._inv_nu = None
        if nu_bar is not None:
            nb = np.asarray(nu_bar.cpu() if isinstance(nu_bar, torch.Tensor) else nu_bar, dtype=np.float64)
            self._inv_nu = _as_device(1.0 / nb)
        w1 = self.solver._w1d
        self._h = _make_schwarz(layout.p, n_o, layout.n_x, layout.n_y, self.solver.S_x, self.solver.S_y,
                                self.solver.lam_x, self.solver.lam_y, w1, self._inv_nu)
        self._work = None
        # ring workspace of the tiled kernel (caller-owned scratch, include/smg.h);
        # one per smoother: calls on one smoother are stream-ordered
        self.ring = torch.zeros(max(1, int(N.lib().smg_schwarz_ws_doubles(self._h.raw))), dtype=torch.float64,
                                device="cuda")

    def kernel_info(self):
        """(engine, tile_x, tile_y) of the device kernel behind this smoother: engine is
        'dense', 'tiled-dfma', 'tiled-dmma' or 'pair' (diagnostics and bench labels)."""
        import ctypes as C
        e, tx, ty = C.c_int(0), C.c_int(0), C.c_int(0)
        N.check(N.lib().smg_schwarz_info(self._h.raw, C.byref(e), C.byref(tx), C.byref(ty)), "schwarz_info")
        return ("dense", "tiled-dfma", "tiled-dmma", "pair")[e.value], tx.value, ty.value

    def _workspace(self):
        if self._work is None:
            self._work = torch.empty(self.layout.shape, dtype=torch.float64, device="cuda")
        return self._work

    def correct(self, r, u):
        """u += sum_s R_s^T W A_s^-1 R_s r (/nu_bar), in place (device)."""
        N.check(N.lib().smg_schwarz_correct(self._h.raw, N.ptr(r), N.ptr(u), N.ptr(self.ring), N.stream()),
                "schwarz_correct")
        return u

    def smooth(self, op, u, f, n_it: int, u_is_zero: bool = False):
        """n_it sweeps of r = f - A u; u += correction, in place; returns u."""
        if not isinstance(u, torch.Tensor) or not u.is_cuda:
            raise TypeError("AdditiveSchwarz.smooth mutates u in place: pass a CUDA float64 tensor")
        f = _as_device(f)
        ring = op.ring_ptr() if hasattr(op, "ring_ptr") else None
        N.check(N.lib().smg_schwarz_smooth_ws(self._h.raw, op._handle.raw, N.ptr(u), N.ptr(f),
                                              N.ptr(self._workspace()), N.ptr(self.ring), ring, int(n_it),
                                              int(bool(u_is_zero)),
                                              N.stream()), "schwarz_smooth")
        return u


class SweepCounter:
    """Running count of multiplicative sweeps, shared across a hierarchy
    (schwarz.py:278-291): the traversal direction alternates with it."""

    def __init__(self, i: int = 0):
        self.i = i

    def reset(self):
        self.i = 0


class MultiplicativeSchwarz:
    """Sequential Schwarz sweep with local residual refresh (schwarz.py:293-353;
    SURVEY 8(f) row f3).

    Subdomains in lexicographic (e_y, e_x) order, reversed on every
    even-numbered sweep of the shared ``counter``; unweighted local FD solves
    (kind=None), the correction divided by ``nu_bar`` for diffusion, and the
    residual refreshed by the element kernels of the touched elements.  The
    chain is sequential by construction: one persistent CTA walks it
    (``smg_mult_sweep``, smg_mult.cu)."""

    def __init__(self, basis: Basis1D, layout: FieldLayout, dx: float, dy: float, n_o: int,
                 nu_bar=None, counter: SweepCounter | None = None):
        self.counter = SweepCounter() if counter is None else counter
        _check_no_alias(layout, n_o)
        self.n_o = n_o
        self.layout = layout
        self.solver = build_fast_diag(basis, dx, dy, n_o, kind=None)
        self._nu_bar = None
        if nu_bar is not None:
            nb = np.asarray(nu_bar.cpu() if isinstance(nu_bar, torch.Tensor) else nu_bar, dtype=np.float64)
            self._nu_bar = _as_device(nb)
        keep = [N.host(a) for a in (self.solver.S_x, self.solver.S_y, self.solver.lam_x, self.solver.lam_y)]
        raw = C.c_void_p()
        N.check(N.lib().smg_mult_create(C.byref(raw), layout.p, n_o, layout.n_x, layout.n_y,
                                        *[k[1] for k in keep], N.ptr(self._nu_bar)), "mult_create")
        self._h = N.Handle(raw, "smg_mult_destroy")
        self._work = None

    def _workspace(self):
        if self._work is None:
            self._work = torch.empty(self.layout.shape, dtype=torch.float64, device="cuda")
        return self._work

    def sweep(self, op, u, r, forward: bool):
        """One ordered pass given the residual r (both updated in place)."""
        N.check(N.lib().smg_mult_sweep(self._h.raw, op._handle.raw, N.ptr(u), N.ptr(r), int(bool(forward)),
                                       N.stream()), "mult_sweep")
        return u

    def smooth(self, op, u, f, n_it: int):
        """schwarz.py:336-353: n_it sweeps, r = f - A u before each."""
        if not isinstance(u, torch.Tensor) or not u.is_cuda:
            raise TypeError("MultiplicativeSchwarz.smooth mutates u in place: pass a CUDA float64 tensor")
        f = _as_device(f)
        r = self._workspace()
        for _ in range(int(n_it)):
            self.counter.i += 1
            N.check(N.lib().smg_op_residual(op._handle.raw, N.ptr(u), N.ptr(f), N.ptr(r), N.stream()), "residual")
            self.sweep(op, u, r, self.counter.i % 2 == 1)
        return u
