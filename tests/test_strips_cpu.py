"""World-size-2 (and 3) CPU tests of the strip decomposition (strips.py) over
torch.distributed/gloo, with the CPU oracle as the per-rank engine: the
assembled strip V-cycle and solver histories must match the global oracle."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import smg_oracle as O
from paper_1512_02390_b200.strips import G, StripPlan, StripSolver, TorchTransport


class OracleEngine:
    """Engine interface of StripSolver implemented with the numpy oracle on
    the rank's local periodic mesh (torch CPU tensors at the boundary); the
    ghost element rows' Schwarz windows are off (nu_bar = inf there), as in
    the GPU engine."""

    def __init__(self, plan, p, rule="fixed:1", nu_hat=None):
        self.plan = plan
        nx, nyl, lx, lyl = plan.local_mesh_args()
        self.h = O.Hierarchy(nx, nyl, lx, lyl, p, rule=rule, nu_hat=None)
        ghost = plan.ghost_mask()
        for l in range(1, len(self.h.levels)):
            lv = self.h.levels[l]
            nb = np.where(ghost, np.inf, 1.0)
            lv.sm = O.AdditiveSweep(lv.b, nx, nyl, lx / nx, lyl / nyl, lv.n_o, "w5", nu_bar=nb)
        self.hg = O.Hierarchy(plan.n_x, plan.n_y, plan.l_x, plan.l_y, 2, rule=rule)
        self.orders = [lv.p for lv in self.h.levels]
        self.n_o = [lv.n_o for lv in self.h.levels]
        self.n_pre = [lv.n_pre for lv in self.h.levels]
        self.n_post = [lv.n_post for lv in self.h.levels]
        self.us = [self.zeros(l) for l in range(len(self.orders))]
        self.fs = [self.zeros(l) for l in range(len(self.orders))]
        self._work = [self.zeros(l) for l in range(len(self.orders))]
        self.full0 = torch.zeros((plan.n_y, plan.n_x), dtype=torch.float64)

    def zeros(self, l):
        return torch.zeros(self.h.levels[l].op.shape, dtype=torch.float64)

    def work(self, l):
        return self._work[l]

    def clone(self, a):
        return a.clone()

    def copy(self, dst, src):
        dst.copy_(torch.as_tensor(src))

    def fill_zero(self, a):
        a.zero_()

    def residual(self, l, u, f, out):
        Au = self.h.levels[l].op.apply(u.numpy())
        out.copy_(torch.from_numpy(Au if f is None else f.numpy() - Au))

    def correct(self, l, r, u, zero):
        c = torch.from_numpy(self.h.levels[l].sm.correction(r.numpy()))
        if zero:
            u.copy_(c)
        else:
            u.add_(c)

    def restrict(self, l, fine, out):
        out.copy_(torch.from_numpy(O.restrict(self.h, l, fine.numpy())))

    def prolong_add(self, l, coarse, fine):
        fine.add_(torch.from_numpy(O.prolongate(self.h, l, coarse.numpy())))

    def coarse_local(self, f0, u0):
        full = O.coarse_solve(self.hg, f0.numpy())
        u0.copy_(torch.from_numpy(full[self.plan.global_rows(self.orders[0])]))

    # device-scalar BLAS-1 restated on host tensors (krylov.py:91-111)
    def scalars(self):
        return torch.zeros(8, dtype=torch.float64), torch.zeros(1, dtype=torch.int32)

    def dot(self, a, b, out):
        out[0] = float(torch.sum(a * b))

    def dot2(self, z, r, r_old, out):
        out[0] = float(torch.sum(z * (r if r_old is None else r - r_old)))
        out[1] = float(torch.sum(z * r))

    def cg_update(self, u, r, r_new, d, q, scal, flag):
        if not scal[1] > 0.0:
            flag[0] = 1
            return
        alpha = float(scal[0] / scal[1])
        u.add_(d, alpha=alpha)
        r_new.copy_(r - alpha * q)
        scal[2] = float(torch.sum(r_new * r_new))
        scal[6] = alpha

    def cg_beta_finish(self, scal):
        scal[5] = scal[3] / scal[0]
        scal[0] = scal[4]

    def cg_direction(self, d, z, scal):
        d.mul_(float(scal[5])).add_(z)

    def read(self, scal, flag):
        return [float(v) for v in scal], int(flag[0])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASE = dict(n_x=6, n_y=8, l_x=1.5, l_y=1.0, p=8)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = CASE
        plan = StripPlan(c["n_x"], c["n_y"], c["l_x"], c["l_y"], world, rank)
        eng = OracleEngine(plan, c["p"])
        sol = StripSolver(plan, eng, TorchTransport(plan))
        N = (c["p"] * c["n_y"], c["p"] * c["n_x"])
        f = O.project_mean(np.random.default_rng(3).standard_normal(N))
        u0 = np.random.default_rng(4).random(N)
        rows = plan.global_rows(c["p"])
        own = plan.own(c["p"])
        # one V-cycle from a nonzero start
        u = torch.from_numpy(u0[rows].copy())
        fl = torch.from_numpy(f[rows].copy())
        sol.v_cycle(u, fl)
        vc_own = u[own].numpy().copy()
        # MG and MGCG histories from zero
        _, rep_mg = sol.solve_mg(torch.from_numpy(f[rows].copy()), torch.zeros_like(u))
        u_cg, rep_cg = sol.solve_mgcg(torch.from_numpy(f[rows].copy()), torch.zeros_like(u))
        q.put((rank, vc_own, rep_mg.residuals, rep_cg.residuals, u_cg[own].numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_strip_decomposition_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    c = CASE
    h = O.Hierarchy(c["n_x"], c["n_y"], c["l_x"], c["l_y"], c["p"])
    N = (c["p"] * c["n_y"], c["p"] * c["n_x"])
    f = O.project_mean(np.random.default_rng(3).standard_normal(N))
    u0 = np.random.default_rng(4).random(N)
    want = O.v_cycle(h, u0.copy(), f)
    got = np.concatenate([t[1] for t in out], 0)
    assert np.abs(got - want).max() / np.abs(want).max() < 1e-11
    _, res_mg, _ = O.solve_mg(h, f, u0=np.zeros_like(f))
    _, res_cg, _, _ = O.solve_mgcg(h, f, u0=np.zeros_like(f))
    for t in out:  # every rank reports the same (allreduced) history
        assert len(t[2]) == len(res_mg) and np.allclose(t[2], res_mg, rtol=1e-9)
        assert len(t[3]) == len(res_cg) and np.allclose(t[3], res_cg, rtol=1e-8)


def test_strip_plan_geometry():
    pl = StripPlan(4, 8, 2.0, 2.0, 4, 1)
    assert G == 1 and pl.s == 2 and pl.ey0 == 2 and pl.local_ny == 2 + 2 * G
    rows = pl.global_rows(4)
    assert rows[0] == (2 - G) * 4 and len(rows) == 4 * pl.local_ny
    own = pl.own(4)
    assert list(rows[own]) == list(range(8, 16))
    m = pl.ghost_mask()
    assert m.shape == (4, 4) and m[0].all() and m[3].all() and not m[1:3].any()
    with pytest.raises(ValueError):
        StripPlan(4, 8, 2.0, 2.0, 8, 0).check_level(2, 1)   # one element row at p=2 < 2 n_o + 1
    with pytest.raises(ValueError):
        StripPlan(4, 6, 2.0, 2.0, 4, 0)
    assert StripPlan(4, 8, 2.0, 2.0, 4, 0).below() == 3


def test_make_transport_choice(monkeypatch):
    """SMG_HALO selects the strip transport; unknown values fail loudly."""
    from paper_1512_02390_b200.strips import StripPlan, TorchTransport, make_transport
    import socket
    import torch.distributed as dist
    plan = StripPlan(4, 4, 1.0, 1.0, 1, 0)
    monkeypatch.setenv("SMG_HALO", "mpi")
    with pytest.raises(ValueError):
        make_transport(plan)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        monkeypatch.setenv("SMG_HALO", "torch")
        assert isinstance(make_transport(plan), TorchTransport)
        # a two-rank plan over a non-NCCL group keeps torch.distributed's transport
        monkeypatch.setenv("SMG_HALO", "nccl")
        assert isinstance(make_transport(StripPlan(4, 4, 1.0, 1.0, 2, 0)), TorchTransport)
    finally:
        dist.destroy_process_group()
