"""The strip decomposition with the real sm_100a kernels: 2 and 4 ranks
emulated by threads on one GPU (ThreadTransport), against the single-domain
GPU path and the reference golden history."""

import numpy as np
import pytest
import torch

from conftest import golden, maxrel
import paper_1512_02390_b200 as P
from paper_1512_02390_b200.strips import GpuEngine, StripPlan, StripSolver, ThreadTransport, run_threads
from oracle import smg_oracle as O

pytestmark = pytest.mark.gpu


def _run(world, n, lx, ly, p, f, u0, solver=None, nu_hat=None, orders=None):
    def fn(rank, shared):
        plan = StripPlan(n, n, lx, ly, world, rank)
        eng = GpuEngine(plan, p, P.OverlapRule("fixed", 1), nu_hat=nu_hat, nu_shift=0.0, orders=orders)
        sol = StripSolver(plan, eng, ThreadTransport(plan, shared))
        rows = plan.global_rows(p)
        own = plan.own(p)
        fl = torch.from_numpy(f[rows].copy()).cuda()
        u = torch.from_numpy(u0[rows].copy()).cuda()
        if solver is None:
            sol.v_cycle(u, fl)
            return u[own].cpu().numpy(), None
        run = sol.solve_mg if solver == "mg" else sol.solve_mgcg
        u, rep = run(fl, u)
        return u[own].cpu().numpy(), rep.residuals
    return run_threads(world, fn)


@pytest.mark.parametrize("world", [2, 4])
def test_strip_vcycle_matches_single_gpu(cuda_device, world):
    n, p = 16, 8
    N = n * p
    f = O.project_mean(np.random.default_rng(0).standard_normal((N, N)))
    u0 = np.random.default_rng(1).random((N, N))
    out = _run(world, n, 1.0, 1.0, p, f, u0)
    got = np.concatenate([o[0] for o in out], 0)
    h = P.build_hierarchy(P.MeshConfig(n, n, 1.0, 1.0), p, P.OverlapRule("fixed", 1))
    want = P.v_cycle(h, torch.from_numpy(u0).cuda(), f).cpu().numpy()
    assert maxrel(got, want) < 1e-11


@pytest.mark.parametrize("world", [2, 4])
def test_strip_mgcg_c1_history(cuda_device, world):
    """BASELINE C1 (8x8, p=8) MGCG on 2/4 emulated ranks vs the reference history."""
    g = golden("krylov")
    f = O.project_mean(np.random.default_rng(0).standard_normal((64, 64)))
    out = _run(world, 8, 1.0, 1.0, 8, f, np.zeros((64, 64)), solver="mgcg")
    want = g["c1_mgcg_0_res"]
    for _, res in out:
        assert len(res) == len(want)
        assert np.max(np.abs(np.log10(np.asarray(res) / want))) < 1e-6
    got = np.concatenate([o[0] for o in out], 0)
    assert maxrel(got, g["c1_mgcg_0_u"]) < 1e-8


def test_strip_diffusion_mg(cuda_device):
    """Variable diffusion (nu sampled at global coordinates on each strip)."""
    n, p = 8, 8
    N = n * p
    f = O.project_mean(np.random.default_rng(2).standard_normal((N, N)))
    out = _run(2, n, 1.0, 1.0, p, f, np.zeros((N, N)), solver="mg", nu_hat=0.9)
    h = P.build_hierarchy(P.MeshConfig(n, n, 1.0, 1.0), p, P.OverlapRule("fixed", 1), nu_hat=0.9, nu_shift=0.0)
    _, rep = P.solve(h, f, P.SolveConfig(solver="mg"), u0=np.zeros_like(f))
    for _, res in out:
        assert len(res) == len(rep.residuals)
        assert np.max(np.abs(np.log10(np.asarray(res) / np.asarray(rep.residuals)))) < 1e-6


def test_strip_vcycle_graph_world1(cuda_device):
    """The strip V-cycle captured as a CUDA graph (StripSolver.v_cycle_graph)
    equals the eager strip V-cycle bitwise; world-1 TorchTransport (its halo
    copies are device ops, so the capture covers the whole cycle)."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1512_02390_b200.strips import TorchTransport
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        n, p = 16, 8
        N = n * p
        f = O.project_mean(np.random.default_rng(5).standard_normal((N, N)))
        u0 = np.random.default_rng(6).random((N, N))
        plan = StripPlan(n, n, 1.0, 1.0, 1, 0)
        rows = plan.global_rows(p)
        outs = []
        for graph in (False, True):
            eng = GpuEngine(plan, p, P.OverlapRule("fixed", 1))
            sol = StripSolver(plan, eng, TorchTransport(plan))
            fl = torch.from_numpy(f[rows].copy()).cuda()
            u = torch.from_numpy(u0[rows].copy()).cuda()
            for _ in range(3):
                if graph:
                    sol.v_cycle_graph(u, fl)
                else:
                    sol.v_cycle(u, fl)
            torch.cuda.synchronize()
            outs.append(u[plan.own(p)].cpu().numpy())
        assert np.array_equal(outs[0], outs[1])
        h = P.build_hierarchy(P.MeshConfig(n, n, 1.0, 1.0), p, P.OverlapRule("fixed", 1))
        want = torch.from_numpy(u0).cuda()
        for _ in range(3):
            P.v_cycle(h, want, f)
        assert maxrel(outs[1], want.cpu().numpy()) < 1e-11
    finally:
        dist.destroy_process_group()
