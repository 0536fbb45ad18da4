"""the multiplicative Schwarz smoother on the device
(smg_mult_sweep) against the reference's own outputs (tests/golden/mult.npz,
oracle/make_golden.py --mult) and the CPU oracle."""

import math

import numpy as np
import pytest
import torch

from conftest import golden, maxrel
import paper_1512_02390_b200 as P
from oracle import smg_oracle as O

pytestmark = pytest.mark.gpu


def _op(nx, ny, p, nu_hat, lx, ly):
    mesh = P.MeshConfig(nx, ny, lx, ly)
    b = P.gll_basis(p)
    if nu_hat < 0:
        return mesh, b, P.PoissonOperator(b, mesh), None
    op = P.DiffusionOperator(b, mesh, P.diffusivity_field(mesh, b, nu_hat, 0.2))
    return mesh, b, op, op.element_mean_nu()


def test_mult_sweeps_vs_reference(cuda_device):
    """Forward then reverse sweep (schwarz.py:336-353) at 1e-12, incl. meshes
    whose 3x3 element footprint wraps onto itself (2x2, 3x5, 4x3)."""
    g = golden("mult")
    for i in range(6):
        nx, ny, p, n_o, nu_hat, lx, ly = g[f"ms{i}_case"]
        mesh, b, op, nu_bar = _op(int(nx), int(ny), int(p), nu_hat, lx, ly)
        lay = P.layout_for(mesh, int(p))
        sm = P.MultiplicativeSchwarz(b, lay, mesh.dx, mesh.dy, int(n_o), nu_bar=nu_bar)
        u = torch.from_numpy(g[f"ms{i}_u"].copy()).cuda()
        f = g[f"ms{i}_f"]
        out = sm.smooth(op, u, f, 1)
        assert out is u
        assert maxrel(u.cpu().numpy(), g[f"ms{i}_u1"]) < 1e-12, (i, maxrel(u.cpu().numpy(), g[f"ms{i}_u1"]))
        sm.smooth(op, u, f, 1)
        assert sm.counter.i == 2
        assert maxrel(u.cpu().numpy(), g[f"ms{i}_u2"]) < 1e-12, (i, maxrel(u.cpu().numpy(), g[f"ms{i}_u2"]))


def _rates(res):
    res = np.asarray(res)
    return np.log10(res[:-1] / res[1:])


def test_mult_vcycle_and_histories_vs_reference(cuda_device):
    g = golden("mult")
    for j in range(2):
        nx, p, nu_hat = g[f"mv{j}_case"]
        h = P.build_hierarchy(P.MeshConfig(int(nx), int(nx), 1.0, 1.0), int(p), P.OverlapRule("fixed", 1),
                              smoother="mult", nu_hat=None if nu_hat < 0 else nu_hat, coarse="cg")
        f = g[f"mv{j}_f"]
        h.reset_smoothers()
        u = torch.from_numpy(g[f"mv{j}_uin"].copy()).cuda()
        P.v_cycle(h, u, f)
        assert maxrel(u.cpu().numpy(), g[f"mv{j}_uout"]) < 1e-10
        for solver in ("mg", "mgcg"):
            _, rep = P.solve(h, f, P.SolveConfig(solver=solver, seed=0), u0=np.zeros_like(f))
            want = g[f"mv{j}_{solver}_res"]
            assert rep.converged and not rep.breakdown
            assert abs(len(rep.residuals) - len(want)) <= 1
            n = min(len(rep.residuals), len(want))
            assert np.max(np.abs(_rates(rep.residuals[:n]) - _rates(want[:n]))) < 1e-3


@pytest.mark.parametrize("shape", [(8, 8, 8, 1), (6, 10, 4, 2), (5, 4, 16, 1)])
def test_mult_sweep_vs_oracle(cuda_device, shape):
    nx, ny, p, n_o = shape
    mesh = P.MeshConfig(nx, ny, 1.0, 1.5)
    b = P.gll_basis(p)
    lay = P.layout_for(mesh, p)
    op = P.PoissonOperator(b, mesh)
    rng = np.random.default_rng(7)
    u0 = rng.standard_normal(lay.shape)
    f = rng.standard_normal(lay.shape)
    sm = P.MultiplicativeSchwarz(b, lay, mesh.dx, mesh.dy, n_o)
    u = torch.from_numpy(u0.copy()).cuda()
    sm.smooth(op, u, f, 2)
    ob = O.gll(p)
    osm = O.MultSweep(ob, nx, ny, mesh.dx, mesh.dy, n_o)
    want = osm.smooth(O.Poisson(ob, nx, ny, mesh.dx, mesh.dy), u0.copy(), f, 2)
    assert maxrel(u.cpu().numpy(), want) < 1e-12


def test_mult_deterministic(cuda_device):
    mesh = P.MeshConfig(6, 6, 1.0, 1.0)
    h = P.build_hierarchy(mesh, 8, P.OverlapRule("fixed", 1), smoother="mult")
    f = O.project_mean(np.random.default_rng(3).standard_normal(h.top.op.layout.shape))
    _, r1 = P.solve(h, f, P.SolveConfig(solver="mgcg", seed=1))
    _, r2 = P.solve(h, f, P.SolveConfig(solver="mgcg", seed=1))
    assert r1.residuals == r2.residuals
    assert r1.converged and math.isfinite(r1.rbar)
