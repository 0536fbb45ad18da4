"""Matrix-free Poisson and variable-diffusion operators (reference operators.py).

``apply`` / ``residual`` run the sm_100a line-operator kernel
(``smg_op_residual``): one launch, gather-form (no scatter), deterministic.
Fields are CUDA float64 tensors of shape (N_y, N_x); numpy inputs are
copied to the device.  The problem builders (coordinates, nu, manufactured
loads) are host-side input preparation, as in the reference.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .basis import Basis1D
from .mesh import FieldLayout, MeshConfig, layout_for

__all__ = ["PoissonOperator", "DiffusionOperator", "residual", "manufactured_rhs_poisson",
           "manufactured_rhs_diffusion", "nodal_coordinates", "project_mean", "load_vector",
           "diffusivity_field", "poisson_benchmark", "to_device"]


def to_device(a, shape=None) -> torch.Tensor:
    """float64 CUDA contiguous view/copy of a numpy array or tensor."""
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    t = t.to(device="cuda", dtype=torch.float64)
    if not t.is_contiguous():
        t = t.contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"field shape {tuple(t.shape)} does not match layout {tuple(shape)}")
    return t


def _check_layout(layout: FieldLayout, u):
    if tuple(u.shape) != layout.shape:
        raise ValueError(f"field shape {tuple(u.shape)} does not match layout ({layout.N_y}, {layout.N_x})")


class _DeviceOperator:
    """Shared device plumbing for both operators."""
    _kind = 0

    def _create(self, mat, nu_dev):
        lib = N.lib()
        w = N.host(self.basis.weights)
        m = N.host(mat)
        raw = C.c_void_p()
        N.check(lib.smg_op_create(C.byref(raw), self._kind, self.basis.p, self.mesh.n_x, self.mesh.n_y,
                                  float(self.mesh.dx), float(self.mesh.dy), w[1], m[1], N.ptr(nu_dev)),
                "op_create")
        self._handle = N.Handle(raw, "smg_op_destroy")
        self._norm_buf = None
        # per-CTA norm partials (caller-owned scratch of smg_op_residual_norm2)
        self.partials = torch.empty(max(1, int(lib.smg_op_ws_doubles(raw))), dtype=torch.float64, device="cuda")
        # ring workspace of the halo-free element kernel (caller-owned scratch, include/smg.h)
        nring = int(lib.smg_op_ring_doubles(raw))
        self.ring = torch.zeros(nring, dtype=torch.float64, device="cuda") if nring else None

    def ring_ptr(self):
        return N.ptr(self.ring) if self.ring is not None else None

    def apply(self, u) -> torch.Tensor:
        """A u as a new device field (operators.py:49-54 / 86-92)."""
        _check_layout(self.layout, u)
        u = to_device(u)
        out = torch.empty_like(u)
        N.check(N.lib().smg_op_residual_ws(self._handle.raw, N.ptr(u), None, N.ptr(out), self.ring_ptr(), N.stream()),
                "apply")
        return out

    def residual_into(self, u, f, out, norm2=None):
        """out = f - A u (f may be None: out = A u); optional device ||out||^2."""
        lib = N.lib()
        if norm2 is None:
            N.check(lib.smg_op_residual_ws(self._handle.raw, N.ptr(u), N.ptr(f), N.ptr(out), self.ring_ptr(),
                                           N.stream()), "residual")
        else:
            N.check(lib.smg_op_residual_norm2_ws(self._handle.raw, N.ptr(u), N.ptr(f), N.ptr(out), N.ptr(norm2),
                                                 N.ptr(self.partials), self.ring_ptr(), N.stream()), "residual")
        return out


class PoissonOperator(_DeviceOperator):
    """A = M_y (x) L_x + L_y (x) M_x on one level (operators.py:30-54)."""
    _kind = 0

    def __init__(self, basis: Basis1D, mesh: MeshConfig):
        self.basis = basis
        self.mesh = mesh
        self.layout = layout_for(mesh, basis.p)
        self.mass_x = (mesh.dx / 2.0) * basis.weights
        self.mass_y = (mesh.dy / 2.0) * basis.weights
        self.stiff_x = (2.0 / mesh.dx) * basis.stiff
        self.stiff_y = (2.0 / mesh.dy) * basis.stiff
        self._create(basis.stiff, None)

    def element_kernel(self, block, e_x: int = 0, e_y: int = 0):
        """Single-element operator on a host (p+1)^2 block (operators.py:44-47)."""
        block = np.asarray(block, dtype=float)
        return self.mass_y[:, None] * (block @ self.stiff_x) + (self.stiff_y @ block) * self.mass_x[None, :]


class DiffusionOperator(_DeviceOperator):
    """Weak-form -div(nu grad u) with GLL quadrature (operators.py:57-98)."""
    _kind = 1

    def __init__(self, basis: Basis1D, mesh: MeshConfig, nu):
        self.basis = basis
        self.mesh = mesh
        self.layout = layout_for(mesh, basis.p)
        if isinstance(nu, torch.Tensor) and nu.is_cuda:
            # device-generated field (diffusivity_field_device): stays on the
            # device; the host copy is made only if a host-side method needs it
            nu_d = nu.to(torch.float64).contiguous()
            if tuple(nu_d.shape) != self.layout.shape:
                raise ValueError(f"field shape {tuple(nu_d.shape)} does not match layout {self.layout.shape}")
            if bool((nu_d <= 0.0).any()):
                raise ValueError("diffusivity must be positive at every node")
            self._nu_host = None
            self._nu_dev = nu_d
        else:
            nu_h = np.asarray(nu.cpu() if isinstance(nu, torch.Tensor) else nu, dtype=np.float64)
            _check_layout(self.layout, nu_h)
            if np.any(nu_h <= 0.0):
                raise ValueError("diffusivity must be positive at every node")
            self._nu_host = nu_h
            self._nu_dev = to_device(nu_h)
        self._cx = mesh.dy / mesh.dx
        self._cy = mesh.dx / mesh.dy
        self.mass_x = (mesh.dx / 2.0) * basis.weights
        self.mass_y = (mesh.dy / 2.0) * basis.weights
        self._create(basis.diff, self._nu_dev)

    @property
    def nu(self) -> np.ndarray:
        """Nodal diffusivity on the host (copied from the device on first use)."""
        if self._nu_host is None:
            self._nu_host = self._nu_dev.cpu().numpy()
        return self._nu_host

    def _element_nu(self, e_x, e_y):
        p = self.basis.p
        iy = (e_y * p + np.arange(p + 1)) % self.layout.N_y
        ix = (e_x * p + np.arange(p + 1)) % self.layout.N_x
        return self.nu[np.ix_(iy, ix)] * np.outer(self.basis.weights, self.basis.weights)

    def element_kernel(self, block, e_x: int, e_y: int):
        """Single-element operator on a host block (operators.py:79-84)."""
        d = self.basis.diff
        nw = self._element_nu(e_x, e_y)
        block = np.asarray(block, dtype=float)
        return self._cx * ((nw * (block @ d.T)) @ d) + self._cy * (d.T @ (nw * (d @ block)))

    def element_mean_nu(self) -> np.ndarray:
        """Quadrature-weighted element mean of nu, (n_y, n_x) (operators.py:94-98).
        Host setup (feeds the smoother's 1/nu_bar); computed on the device
        when the field was generated there."""
        p = self.basis.p
        if self._nu_host is None:
            out = torch.empty((self.layout.n_y, self.layout.n_x), dtype=torch.float64, device="cuda")
            w = np.ascontiguousarray(self.basis.weights, dtype=np.float64)
            N.check(N.lib().smg_element_mean(p, self.layout.n_x, self.layout.n_y, N.hptr(w), N.ptr(self._nu_dev),
                                             N.ptr(out), N.stream()), "element_mean")
            return out.cpu().numpy()
        L = self.layout
        off = np.arange(p + 1)
        iy = (p * np.arange(L.n_y)[:, None] + off[None, :]) % L.N_y
        ix = (p * np.arange(L.n_x)[:, None] + off[None, :]) % L.N_x
        blocks = self.nu[iy[:, None, :, None], ix[None, :, None, :]]
        w2 = np.outer(self.basis.weights, self.basis.weights)
        return np.einsum("yxij,ij->yx", blocks, w2) / 4.0


def residual(op, u, f) -> torch.Tensor:
    """r = f - op(u) in one fused launch (operators.py:101-103)."""
    u = to_device(u, op.layout.shape)
    f = to_device(f, op.layout.shape)
    out = torch.empty_like(u)
    return op.residual_into(u, f, out)


def project_mean(f):
    """f - mean(f) (operators.py:138-140).  CUDA tensors: device reduction +
    subtract (returns a new tensor); numpy arrays (host input preparation):
    numpy, like the reference."""
    if isinstance(f, torch.Tensor) and f.is_cuda:
        g = f.to(torch.float64).contiguous().clone()
        ws = torch.zeros(N.lib().smg_reduce_ws_doubles(), dtype=torch.float64, device="cuda")
        N.check(N.lib().smg_project_mean(N.ptr(g), g.numel(), N.ptr(ws), N.stream()), "project_mean")
        return g
    f = np.asarray(f, dtype=np.float64)
    return f - f.mean()


# ---------------------------------------------------------------------------
# Host-side problem builders (reference operators.py:110-199)


def nodal_coordinates(mesh: MeshConfig, basis: Basis1D):
    """Global node coordinates (X, Y), each (N_y, N_x) (operators.py:110-120)."""
    loc = (basis.nodes[:-1] + 1) / 2
    x = ((np.arange(mesh.n_x)[:, None] + loc[None, :]) * mesh.dx).ravel()
    y = ((np.arange(mesh.n_y)[:, None] + loc[None, :]) * mesh.dy).ravel()
    return np.meshgrid(x, y)


def _global_quadrature(mesh: MeshConfig, basis: Basis1D):
    """Assembled quadrature weights (operators.py:123-135)."""
    p = basis.p
    L = layout_for(mesh, p)

    def line(n, d, N_):
        w = np.zeros(N_)
        for e in range(n):
            np.add.at(w, (e * p + np.arange(p + 1)) % N_, (d / 2.0) * basis.weights)
        return w

    return np.outer(line(mesh.n_y, mesh.dy, L.N_y), line(mesh.n_x, mesh.dx, L.N_x))


def load_vector(mesh: MeshConfig, basis: Basis1D, source) -> np.ndarray:
    """operators.py:143-146."""
    X, Y = nodal_coordinates(mesh, basis)
    return _global_quadrature(mesh, basis) * source(X, Y)


def manufactured_rhs_poisson(mesh: MeshConfig, basis: Basis1D, source) -> np.ndarray:
    """operators.py:149-151."""
    return project_mean(load_vector(mesh, basis, source))


def poisson_benchmark(mesh: MeshConfig, basis: Basis1D):
    """u = sin(pi x) sin(pi y) test problem (operators.py:154-164): (f, u_samples)."""
    def u_exact(x, y):
        return np.sin(np.pi * x) * np.sin(np.pi * y)

    f = manufactured_rhs_poisson(mesh, basis, lambda x, y: 2.0 * np.pi ** 2 * u_exact(x, y))
    X, Y = nodal_coordinates(mesh, basis)
    return f, u_exact(X, Y)


def diffusivity_field(mesh: MeshConfig, basis: Basis1D, nu_hat: float, s: float = 0.2) -> np.ndarray:
    """nu = 1 + nu_hat sin(2 pi (x - s)) sin(2 pi (y - s)) (operators.py:167-173)."""
    if not 0.0 <= nu_hat < 1.0:
        raise ValueError(f"diffusivity amplitude must be in [0, 1), got {nu_hat}")
    X, Y = nodal_coordinates(mesh, basis)
    return 1.0 + nu_hat * np.sin(2 * np.pi * (X - s)) * np.sin(2 * np.pi * (Y - s))


def manufactured_rhs_diffusion(mesh: MeshConfig, basis: Basis1D, nu_hat: float, s: float = 0.2):
    """u = sin(2 pi x) sin(2 pi y) with variable nu (operators.py:176-199): (f, nu, u_samples)."""
    nu = diffusivity_field(mesh, basis, nu_hat, s)
    tp = 2.0 * np.pi

    def source(x, y):
        u = np.sin(tp * x) * np.sin(tp * y)
        ux = tp * np.cos(tp * x) * np.sin(tp * y)
        uy = tp * np.sin(tp * x) * np.cos(tp * y)
        nv = 1.0 + nu_hat * np.sin(tp * (x - s)) * np.sin(tp * (y - s))
        nx = tp * nu_hat * np.cos(tp * (x - s)) * np.sin(tp * (y - s))
        ny = tp * nu_hat * np.sin(tp * (x - s)) * np.cos(tp * (y - s))
        return -(nv * (-2.0 * tp ** 2 * u) + nx * ux + ny * uy)

    f = project_mean(load_vector(mesh, basis, source))
    X, Y = nodal_coordinates(mesh, basis)
    return f, nu, np.sin(tp * X) * np.sin(tp * Y)


# ---------------------------------------------------------------------------
# Device-side problem generation: the same fields as the
# host builders above, evaluated per node on the GPU (smg_problem_field), so a
# 151 M-DOF level never exists on the host.  Same expressions and order; the
# FP64 sin/cos differ from numpy's by <= 2 ulp.

def _device_field(kind: int, mesh: MeshConfig, basis: Basis1D, nu_hat: float = 0.0, s: float = 0.2):
    lay = layout_for(mesh, basis.p)
    out = torch.empty(lay.shape, dtype=torch.float64, device="cuda")
    nodes = np.ascontiguousarray(basis.nodes, dtype=np.float64)
    w = np.ascontiguousarray(basis.weights, dtype=np.float64)
    N.check(N.lib().smg_problem_field(kind, basis.p, mesh.n_x, mesh.n_y, mesh.dx, mesh.dy, N.hptr(nodes),
                                      N.hptr(w), float(nu_hat), float(s), N.ptr(out), N.stream()),
            "problem_field")
    return out


def diffusivity_field_device(mesh: MeshConfig, basis: Basis1D, nu_hat: float, s: float = 0.2) -> torch.Tensor:
    """diffusivity_field on the device (operators.py:167-173)."""
    if not 0.0 <= nu_hat < 1.0:
        raise ValueError(f"diffusivity amplitude must be in [0, 1), got {nu_hat}")
    return _device_field(0, mesh, basis, nu_hat, s)


def poisson_benchmark_device(mesh: MeshConfig, basis: Basis1D):
    """poisson_benchmark on the device (operators.py:154-164): (f, u_samples)."""
    return project_mean(_device_field(1, mesh, basis)), _device_field(3, mesh, basis)


def manufactured_rhs_diffusion_device(mesh: MeshConfig, basis: Basis1D, nu_hat: float, s: float = 0.2):
    """manufactured_rhs_diffusion on the device (operators.py:176-199): (f, nu, u_samples)."""
    nu = diffusivity_field_device(mesh, basis, nu_hat, s)
    return project_mean(_device_field(2, mesh, basis, nu_hat, s)), nu, _device_field(4, mesh, basis)
