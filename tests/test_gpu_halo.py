"""libsmg's strip halos and collectives (smg_halo_*, NCCL) on one GPU: a
one-rank communicator wraps onto itself, so every exchange runs as NCCL self
send/recv through the same code as between GPUs.  Checked bitwise against the
TorchTransport semantics (its one-rank branch is plain tensor copies / adds in
the same fixed order), and the strip V-cycle -- eager and captured into one
CUDA graph with its NCCL halos -- against the single-domain V-cycle."""

import numpy as np
import pytest
import torch

from conftest import maxrel
import paper_1512_02390_b200 as P
from paper_1512_02390_b200 import _native as NV
from paper_1512_02390_b200.strips import GpuEngine, NcclHaloTransport, StripPlan, StripSolver, TorchTransport
from oracle import smg_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def halo(cuda_device):
    plan = StripPlan(8, 4, 1.0, 1.0, 1, 0)
    tr = NcclHaloTransport(plan)
    yield plan, tr
    tr.close()


def _torch_world1(plan):
    t = TorchTransport.__new__(TorchTransport)
    t.plan = plan
    return t


@pytest.mark.parametrize("p,below,above", [(4, 4, 1), (4, 1, 2), (4, 0, 3), (4, 2, 0), (8, 8, 8), (2, 2, 1)])
def test_exchange_matches_torch(halo, p, below, above):
    plan, tr = halo
    rng = np.random.default_rng(p * 100 + below * 10 + above)
    a = torch.from_numpy(rng.standard_normal((p * plan.local_ny, p * plan.n_x))).cuda()
    b = a.clone()
    tr.exchange(a, p, below, above)
    _torch_world1(plan).exchange(b, p, below, above)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.parametrize("n_y", [4, 1])
@pytest.mark.parametrize("p,below,above", [(4, 1, 2), (4, 3, 4), (2, 2, 2), (8, 2, 3), (8, 8, 8), (2, 0, 2)])
def test_exchange_add_matches_torch(cuda_device, n_y, p, below, above):
    """Including one-element-row strips where the two added ranges overlap
    (s p < below + above): the fixed order (from below first) must match."""
    plan = StripPlan(8, n_y, 1.0, 1.0, 1, 0)
    tr = NcclHaloTransport(plan)
    try:
        rng = np.random.default_rng(7 + p + below + above)
        a = torch.from_numpy(rng.standard_normal((p * plan.local_ny, p * plan.n_x))).cuda()
        b = a.clone()
        tr.exchange_add(a, p, below, above)
        _torch_world1(plan).exchange_add(b, p, below, above)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    finally:
        tr.close()


def test_collectives_world1(halo):
    plan, tr = halo
    x = torch.arange(5, dtype=torch.float64, device="cuda") + 0.5
    y = x.clone()
    tr.allreduce_(x[1:4])
    assert torch.equal(x, y)
    own = torch.randn(6, 10, dtype=torch.float64, device="cuda")
    full = torch.zeros(6, 10, dtype=torch.float64, device="cuda")
    tr.allgather_rows(own, full)
    torch.cuda.synchronize()
    assert torch.equal(own, full)
    with pytest.raises(ValueError):
        tr.allgather_rows(own, torch.zeros(7, 10, dtype=torch.float64, device="cuda"))


def test_bad_arguments(halo):
    plan, tr = halo
    lib = NV.lib()
    t = torch.zeros(12, 8, dtype=torch.float64, device="cuda")
    # ghost rows below lo and at/above hi must exist inside the array
    with pytest.raises(ValueError):
        NV.check(lib.smg_halo_exchange(tr.h, t.data_ptr(), 12, 8, 2, 10, 3, 1, NV.stream()))
    with pytest.raises(ValueError):
        NV.check(lib.smg_halo_exchange(tr.h, t.data_ptr(), 12, 8, 2, 10, 1, 3, NV.stream()))
    with pytest.raises(ValueError):
        NV.check(lib.smg_halo_exchange_add(tr.h, t.data_ptr(), 12, 8, 4, 8, 1, 1, None, NV.stream()))
    assert lib.smg_halo_nccl_version() >= 21800


@pytest.mark.parametrize("graph", [False, True])
def test_strip_vcycle_native_halo_world1(cuda_device, halo, graph):
    """A whole strip V-cycle on one rank with libsmg's NCCL halos: equal to the
    TorchTransport strip cycle bitwise, and to the single-domain V-cycle."""
    _, tr = halo
    n, p = 16, 8
    N = n * p
    f = O.project_mean(np.random.default_rng(5).standard_normal((N, N)))
    u0 = np.random.default_rng(6).random((N, N))
    plan = StripPlan(n, n, 1.0, 1.0, 1, 0)
    rows = plan.global_rows(p)
    outs = []
    for transport in (_torch_world1(plan), NcclHaloTransport(plan)):
        eng = GpuEngine(plan, p, P.OverlapRule("fixed", 1))
        sol = StripSolver(plan, eng, transport)
        fl = torch.from_numpy(f[rows].copy()).cuda()
        u = torch.from_numpy(u0[rows].copy()).cuda()
        for _ in range(3):
            if graph and isinstance(transport, NcclHaloTransport):
                sol.v_cycle_graph(u, fl)
            else:
                sol.v_cycle(u, fl)
        torch.cuda.synchronize()
        outs.append(u[plan.own(p)].cpu().numpy())
        sol.release_graph()
        if isinstance(transport, NcclHaloTransport):
            transport.close()
    assert np.array_equal(outs[0], outs[1])
    h = P.build_hierarchy(P.MeshConfig(n, n, 1.0, 1.0), p, P.OverlapRule("fixed", 1))
    want = torch.from_numpy(u0).cuda()
    for _ in range(3):
        P.v_cycle(h, want, f)
    assert maxrel(outs[1], want.cpu().numpy()) < 1e-11


def test_strip_mgcg_native_halo_world1(cuda_device):
    """MGCG on one strip rank with NCCL all-reduced device dots: the C1
    reference history."""
    from conftest import golden
    g = golden("krylov")
    f = O.project_mean(np.random.default_rng(0).standard_normal((64, 64)))
    plan = StripPlan(8, 8, 1.0, 1.0, 1, 0)
    tr = NcclHaloTransport(plan)
    try:
        eng = GpuEngine(plan, 8, P.OverlapRule("fixed", 1))
        sol = StripSolver(plan, eng, tr)
        rows = plan.global_rows(8)
        u, rep = sol.solve_mgcg(torch.from_numpy(f[rows].copy()).cuda(), torch.zeros(len(rows), 64,
                                                                                     dtype=torch.float64,
                                                                                     device="cuda"))
        want = g["c1_mgcg_0_res"]
        assert len(rep.residuals) == len(want)
        assert np.max(np.abs(np.log10(np.asarray(rep.residuals) / want))) < 1e-6
        assert maxrel(u[plan.own(8)].cpu().numpy(), g["c1_mgcg_0_u"]) < 1e-8
    finally:
        tr.close()
