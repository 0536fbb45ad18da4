"""Run-to-run bitwise reproducibility of the device path (a race detector).

Every libsmg kernel writes each output from one thread in a fixed summation
order, and the launches are chained with programmatic dependent launch, so a
repeated V-cycle / smoother / solve on the same inputs must be bitwise equal
(the reference requires identical histories for equal seeds,
test_krylov.py:73-81).  A missing griddepcontrol.wait or a shared-memory
hazard shows up here as a run-to-run difference (this is how a PDL race in
the multiplicative sweep kernel was found).  compute-sanitizer is not
available on this pool, so these repeated runs are the race check.
"""

import numpy as np
import pytest
import torch

import paper_1512_02390_b200 as P
from paper_1512_02390_b200.multigrid import _v_cycle

pytestmark = pytest.mark.gpu

REPS = 8


def _rhs(shape, seed=0):
    return P.project_mean(np.random.default_rng(seed).standard_normal(shape))


@pytest.mark.parametrize("case", [
    # (n, p, nu_hat, orders, smoother)
    (64, 16, None, None, "add"),           # C2
    (16, 24, 0.9, (1, 3, 6, 12, 24), "add"),  # reduced C5: diffusion, opd_kernel at p = 24
    (8, 32, None, None, "add"),            # opd_kernel (Poisson) at p = 32, DMMA Schwarz
    (4, 8, 0.5, None, "mult"),             # multiplicative smoother with diffusion
])
def test_vcycle_bitwise_repeatable(cuda_device, case):
    n, p, nu_hat, orders, smoother = case
    h = P.build_hierarchy(P.MeshConfig(n, n, 1.0, 1.0), p, P.OverlapRule("fixed", 1), nu_hat=nu_hat,
                          nu_shift=0.0, orders=orders, smoother=smoother,
                          coarse="cg" if smoother == "mult" else None)
    f = torch.from_numpy(_rhs(h.top.op.layout.shape)).cuda()
    u0 = torch.from_numpy(np.random.default_rng(1).standard_normal(h.top.op.layout.shape)).cuda()
    ref = None
    for _ in range(REPS):
        h.reset_smoothers()
        u = u0.clone()
        _v_cycle(h, u, f)
        torch.cuda.synchronize()
        if ref is None:
            ref = u.clone()
        else:
            assert torch.equal(u, ref), float((u - ref).abs().max())


def test_smoother_and_operator_bitwise_repeatable(cuda_device):
    for n, p, nu_hat in [(256, 16, None), (64, 24, 0.9), (32, 32, None)]:
        mesh = P.MeshConfig(n, n, 1.0, 1.0)
        lay = P.layout_for(mesh, p)
        b = P.gll_basis(p)
        rng = np.random.default_rng(2)
        r = torch.from_numpy(rng.standard_normal(lay.shape)).cuda()
        sm = P.AdditiveSchwarz(b, lay, mesh.dx, mesh.dy, 1, P.WeightKind.QUINTIC)
        op = (P.PoissonOperator(b, mesh) if nu_hat is None
              else P.DiffusionOperator(b, mesh, 1.0 + nu_hat * rng.random(lay.shape)))
        outs = []
        for _ in range(REPS):
            c = torch.zeros_like(r)
            sm.correct(r, c)
            outs.append((c, op.apply(r)))
        torch.cuda.synchronize()
        for c, a in outs[1:]:
            assert torch.equal(c, outs[0][0]), ("schwarz", n, p)
            assert torch.equal(a, outs[0][1]), ("operator", n, p)


def test_mgcg_history_bitwise_repeatable(cuda_device):
    h = P.build_hierarchy(P.MeshConfig(16, 16, 1.0, 1.0), 24, P.OverlapRule("fixed", 1), nu_hat=0.9, nu_shift=0.0,
                          orders=(1, 3, 6, 12, 24))
    f = _rhs(h.top.op.layout.shape)
    cfg = P.SolveConfig(solver="mgcg", max_cycles=30)
    _, rep1 = P.solve(h, f, cfg, u0=np.zeros_like(f))
    for _ in range(3):
        _, rep = P.solve(h, f, cfg, u0=np.zeros_like(f))
        assert rep.residuals == rep1.residuals
