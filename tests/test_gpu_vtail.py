"""GPU parity of the V-cycle tail (smg_vtail_*: the lower levels + coarse
pseudo-inverse as one cooperative launch) against the per-kernel path
(SMG_VTAIL=0, itself pinned to the reference in test_gpu_parity.py) and the
CPU oracle.  Both paths compute the same exact-pinv V-cycle, so they agree to
rounding (1e-12 relative); against the oracle's CG coarse solve the bar is
the 1e-8 of the other pinv tests."""

import numpy as np
import pytest
import torch

from conftest import maxrel
import paper_1512_02390_b200 as P
from oracle import smg_oracle as O

pytestmark = pytest.mark.gpu

CASES = [
    # n_x, n_y, l_x, l_y, p, rule, orders
    (8, 8, 1.0, 1.0, 8, "fixed:1", None),        # C1
    (64, 64, 1.0, 1.0, 16, "fixed:1", None),     # C2
    (6, 10, 1.0, 1.0, 8, "fixed:1", None),       # ragged tiles
    (16, 16, 1.0, 1.0, 8, "ceilp2", None),       # n_o = 2 at p = 4: tail = level 1 only
    (16, 8, 2.0, 1.0, 16, "ceilp8", None),       # dx != dy
    (3, 9, 1.0, 2.0, 8, "fixed:1", None),        # 3 x 9 elements, dx != dy
    (5, 7, 1.0, 1.0, 4, "fixed:1", None),        # tiny, odd mesh
]


def _hier(case, monkeypatch, tail):
    nx, ny, lx, ly, p, rule, orders = case
    monkeypatch.setenv("SMG_VTAIL", "1" if tail else "0")
    h = P.build_hierarchy(P.MeshConfig(nx, ny, lx, ly), p, P.OverlapRule.parse(rule), orders=orders)
    h._setup_tail()  # reads SMG_VTAIL now, not at the first V-cycle
    return h


def _fields(h, seed):
    shape = h.top.op.layout.shape
    rng = np.random.default_rng(seed)
    f = O.project_mean(rng.standard_normal(shape))
    u = rng.standard_normal(shape)
    return f, u


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}x{c[1]}p{c[4]}{c[5]}")
def test_vtail_matches_per_kernel_path(cuda_device, monkeypatch, case):
    ht = _hier(case, monkeypatch, True)
    hk = _hier(case, monkeypatch, False)
    f, u0 = _fields(ht, 3)
    ut = torch.from_numpy(u0).cuda()
    uk = ut.clone()
    P.v_cycle(ht, ut, f)
    assert ht.tail_levels >= 1, "tail not engaged"
    P.v_cycle(hk, uk, f)
    assert hk.tail_levels == 0
    assert maxrel(ut.cpu().numpy(), uk.cpu().numpy()) < 1e-12
    # zero start (the MGCG preconditioner form)
    zt = torch.zeros_like(ut)
    zk = torch.zeros_like(ut)
    P.v_cycle(ht, zt, f)
    P.v_cycle(hk, zk, f)
    assert maxrel(zt.cpu().numpy(), zk.cpu().numpy()) < 1e-12


@pytest.mark.parametrize("case", CASES[:3], ids=lambda c: f"{c[0]}x{c[1]}p{c[4]}")
def test_vtail_vs_oracle(cuda_device, monkeypatch, case):
    nx, ny, lx, ly, p, rule, orders = case
    h = _hier(case, monkeypatch, True)
    f, u0 = _fields(h, 5)
    u = torch.from_numpy(u0).cuda()
    P.v_cycle(h, u, f)
    oh = O.Hierarchy(nx, ny, lx, ly, p, rule=rule, coarse_tol=1e-14)
    want = O.v_cycle(oh, u0.copy(), f)
    assert maxrel(u.cpu().numpy(), want) < 1e-8


def test_vtail_deterministic_and_graph_capturable(cuda_device, monkeypatch):
    from paper_1512_02390_b200.multigrid import _v_cycle
    h = _hier(CASES[1], monkeypatch, True)
    f, u0 = _fields(h, 7)
    fd = torch.from_numpy(f).cuda()
    a = torch.from_numpy(u0).cuda()
    b = a.clone()
    _v_cycle(h, a, fd)
    _v_cycle(h, b, fd)
    assert torch.equal(a, b)
    # captured as a CUDA graph (the bench's form) it gives the same bits
    c = torch.from_numpy(u0).cuda()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        _v_cycle(h, c, fd)
    torch.cuda.current_stream().wait_stream(s)
    c.copy_(torch.from_numpy(u0))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        _v_cycle(h, c, fd)
    c.copy_(torch.from_numpy(u0))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(a, c)


def test_vtail_solver_histories(cuda_device, monkeypatch):
    """C1 MG/MGCG histories through the tail match the per-kernel path's."""
    f = O.project_mean(np.random.default_rng(0).standard_normal((64, 64)))
    reps = {}
    for tail in (True, False):
        h = _hier(CASES[0], monkeypatch, tail)
        for solver in ("mg", "mgcg"):
            _, rep = P.solve(h, f, P.SolveConfig(solver=solver, seed=0), u0=np.zeros_like(f))
            reps[(tail, solver)] = rep
    for solver in ("mg", "mgcg"):
        a, b = reps[(True, solver)], reps[(False, solver)]
        assert a.cycles == b.cycles
        np.testing.assert_allclose(a.residuals, b.residuals, rtol=0, atol=1e-12 * a.residuals[0])


def test_vtail_not_engaged_outside_its_scope(cuda_device, monkeypatch):
    """Orders that are not 2^l or overlap != 1 keep the per-kernel path."""
    h = _hier((12, 12, 1.0, 1.0, 12, "fixed:1", (1, 3, 6, 12)), monkeypatch, True)
    assert h.tail_levels == 0
    h = _hier((16, 16, 1.0, 1.0, 16, "ceilp2", None), monkeypatch, True)
    assert h.tail_levels == 1
