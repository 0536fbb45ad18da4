"""GPU parity: the sm_100a path (through libsmg's C ABI) against the
reference's golden vectors and the CPU oracle.

Tolerances (north star): operator / smoother / transfer outputs <= 1e-12
relative (max|d| / max|ref|); iteration counts +-1; per-cycle log10
reductions and rbar within 1e-3.  The pinv coarse solver is exact where the
reference's CG stops at 1e-12, so V-cycle outputs with it are compared at
1e-9 and solver histories on iteration counts and rates.
"""

import math

import numpy as np
import pytest
import torch

from conftest import golden, maxrel
import paper_1512_02390_b200 as P
from paper_1512_02390_b200 import schwarz as S
from oracle import smg_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-12


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def test_fd_solve_blocks(cuda_device):
    g = golden("schwarz_setup")
    for i in range(int(g["n_fd"])):
        p, n_o, dx, dy = g[f"fd{i}_case"]
        fd = S.build_fast_diag(P.gll_basis(int(p)), dx, dy, int(n_o), S.WeightKind.QUINTIC)
        got = host(fd.solve(dev(g[f"fd{i}_r"])))
        assert maxrel(got, g[f"fd{i}_solve"]) < TOL, (i, maxrel(got, g[f"fd{i}_solve"]))


def test_operators_vs_reference(cuda_device):
    g = golden("operators")
    for i in range(int(g["n_op"])):
        nx, ny, lx, ly, p = g[f"op{i}_case"]
        mesh = P.MeshConfig(int(nx), int(ny), lx, ly)
        b = P.gll_basis(int(p))
        u = dev(g[f"op{i}_u"])
        A = P.PoissonOperator(b, mesh)
        assert maxrel(host(A.apply(u)), g[f"op{i}_Au"]) < TOL, ("poisson", i)
        B = P.DiffusionOperator(b, mesh, g[f"op{i}_nu"])
        assert maxrel(host(B.apply(u)), g[f"op{i}_Bu"]) < TOL, ("diffusion", i)
        np.testing.assert_allclose(B.element_mean_nu(), g[f"op{i}_nubar"], rtol=1e-15)
        f = dev(g[f"op{i}_Au"]) * 0.5
        r = host(P.residual(A, u, f))
        assert maxrel(r, 0.5 * g[f"op{i}_Au"] - g[f"op{i}_Au"]) < TOL


def test_operator_rejects_bad_shapes(cuda_device):
    A = P.PoissonOperator(P.gll_basis(4), P.MeshConfig(3, 2))
    with pytest.raises(ValueError):
        A.apply(torch.zeros(5, 5, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        P.DiffusionOperator(P.gll_basis(2), P.MeshConfig(2, 2), np.zeros((4, 4)))


def _sweep_case(g, i):
    nx, ny, lx, ly, p, n_o, nu_hat = g[f"sw{i}_case"]
    nx, ny, p, n_o = int(nx), int(ny), int(p), int(n_o)
    mesh = P.MeshConfig(nx, ny, lx, ly)
    b = P.gll_basis(p)
    lay = P.layout_for(mesh, p)
    if nu_hat < 0:
        op, nb = P.PoissonOperator(b, mesh), None
    else:
        op = P.DiffusionOperator(b, mesh, P.diffusivity_field(mesh, b, nu_hat, 0.2))
        nb = op.element_mean_nu()
    sm = P.AdditiveSchwarz(b, lay, mesh.dx, mesh.dy, n_o, S.WeightKind(str(g[f"sw{i}_kind"])), nu_bar=nb)
    return op, sm


def test_additive_sweeps_vs_reference(cuda_device):
    g = golden("sweeps")
    for i in range(int(g["n_sw"])):
        op, sm = _sweep_case(g, i)
        f = dev(g[f"sw{i}_f"])
        for n_it, key in ((1, "u1"), (2, "u2")):
            u = dev(g[f"sw{i}_u0"])
            out = sm.smooth(op, u, f, n_it)
            assert out is u
            assert maxrel(host(u), g[f"sw{i}_{key}"]) < TOL, (i, key, maxrel(host(u), g[f"sw{i}_{key}"]))


def test_sweep_alias_guard(cuda_device):
    mesh = P.MeshConfig(2, 2)
    b = P.gll_basis(2)
    with pytest.raises(ValueError):
        P.AdditiveSchwarz(b, P.layout_for(mesh, 2), mesh.dx, mesh.dy, 1, S.WeightKind.QUINTIC)


def test_transfers_vs_reference_and_adjoint(cuda_device):
    g = golden("multigrid")
    h = P.build_hierarchy(P.MeshConfig(4, 3, 2.0, 2.0), 32, P.OverlapRule("fixed", 1))
    for l in range(1, h.depth + 1):
        Pu = host(P.prolongate(h, l, dev(g[f"tr{l}_uc"])))
        assert maxrel(Pu, g[f"tr{l}_P"]) < TOL
        Rv = host(P.restrict_residual(h, l, dev(g[f"tr{l}_vf"])))
        assert maxrel(Rv, g[f"tr{l}_R"]) < TOL
        lhs = np.vdot(Pu, g[f"tr{l}_vf"])
        rhs = np.vdot(g[f"tr{l}_uc"], Rv)
        assert abs(lhs - rhs) <= 1e-13 * abs(lhs)
    with pytest.raises(ValueError):
        P.prolongate(h, 0, np.zeros((1, 1)))


@pytest.mark.parametrize("case", [(64, 64, 16, None, (1, 2, 4, 8, 16)), (12, 8, 8, None, (1, 2, 4, 8)),
                                  (16, 16, 24, 0.9, (1, 3, 6, 12, 24)), (6, 6, 32, None, (1, 2, 4, 8, 16, 32))])
def test_fused_residual_restrict_bitwise(cuda_device, case):
    """smg_residual_restrict (one fused launch where enabled: p_f <= 8 by default,
    SMG_RR_FUSED=2 for all) == residual launch + restriction launch, bitwise."""
    from paper_1512_02390_b200 import _native as NV
    nx, ny, p, nu_hat, orders = case
    h = P.build_hierarchy(P.MeshConfig(nx, ny, 1.0, 1.0), p, P.OverlapRule("fixed", 1), nu_hat=nu_hat,
                          orders=orders)
    lib = NV.lib()
    st = NV.stream()
    rng = np.random.default_rng(3)
    for l in range(h.depth, 0, -1):
        lv = h.levels[l]
        u = dev(rng.standard_normal(lv.op.layout.shape))
        f = dev(rng.standard_normal(lv.op.layout.shape))
        fc1 = torch.empty_like(h.levels[l - 1].f)
        fc2 = torch.empty_like(h.levels[l - 1].f)
        work = torch.empty_like(u)
        NV.check(lib.smg_residual_restrict(lv.transfer.handle.raw, lv.op._handle.raw, NV.ptr(u), NV.ptr(f),
                                           NV.ptr(fc1), NV.ptr(work), st), "rr")
        NV.check(lib.smg_op_residual(lv.op._handle.raw, NV.ptr(u), NV.ptr(f), NV.ptr(work), st), "res")
        NV.check(lib.smg_restrict(lv.transfer.handle.raw, NV.ptr(work), NV.ptr(fc2), st), "restrict")
        torch.cuda.synchronize()
        assert torch.equal(fc1, fc2), (case, l, float((fc1 - fc2).abs().max()))


def test_transfers_p24_chain(cuda_device):
    mesh = P.MeshConfig(3, 4, 1.0, 1.0)
    h = P.build_hierarchy(mesh, 24, P.OverlapRule("fixed", 1), orders=(1, 3, 6, 12, 24), nu_hat=0.9, nu_shift=0.0)
    oh = O.Hierarchy(3, 4, 1.0, 1.0, 24, nu_hat=0.9, nu_shift=0.0, orders=[1, 3, 6, 12, 24])
    rng = np.random.default_rng(3)
    for l in range(1, h.depth + 1):
        uc = rng.standard_normal(h.levels[l - 1].op.layout.shape)
        vf = rng.standard_normal(h.levels[l].op.layout.shape)
        assert maxrel(host(P.prolongate(h, l, uc)), O.prolongate(oh, l, uc)) < TOL
        assert maxrel(host(P.restrict_residual(h, l, vf)), O.restrict(oh, l, vf)) < TOL


def test_coarse_solvers(cuda_device):
    g = golden("multigrid")
    for i, (nx, ny, lx, ly, nu_hat) in enumerate([(4, 4, 2.0, 2.0, None), (8, 8, 1.0, 1.0, None),
                                                   (16, 8, 8.0, 1.0, None), (8, 8, 1.0, 1.0, 0.9)]):
        mesh = P.MeshConfig(nx, ny, lx, ly)
        want = g[f"cs{i}_u0"]
        h = P.build_hierarchy(mesh, 2, P.OverlapRule("fixed", 1), nu_hat=nu_hat, coarse="cg")
        got = host(P.coarse_solve(h, g[f"cs{i}_f0"]))
        assert maxrel(got, want) < 1e-10, ("cg", i, maxrel(got, want))
        assert h.coarse_cg_exhausted == 0
        if nu_hat is None:
            hp = P.build_hierarchy(mesh, 2, P.OverlapRule("fixed", 1))
            got = host(P.coarse_solve(hp, g[f"cs{i}_f0"]))
            # exact pseudo-inverse vs the reference's 1e-12-accurate CG
            assert maxrel(got, want) < 1e-9, ("pinv", i, maxrel(got, want))
            assert abs(got.mean()) < 1e-13 * np.abs(got).max()


@pytest.mark.parametrize("coarse", ["cg", "pinv"])
def test_v_cycle_vs_reference(cuda_device, coarse):
    g = golden("multigrid")
    for i in range(4):
        nx, ny, lx, ly, p, nu_hat, n_post = g[f"vc{i}_case"]
        if coarse == "pinv" and nu_hat >= 0:
            continue
        h = P.build_hierarchy(P.MeshConfig(int(nx), int(ny), lx, ly), int(p), P.OverlapRule.parse(str(g[f"vc{i}_rule"])),
                              nu_hat=None if nu_hat < 0 else nu_hat, n_post=int(n_post), coarse=coarse)
        tol = 1e-11 if coarse == "cg" else 1e-8
        u = dev(g[f"vc{i}_uin"])
        out = P.v_cycle(h, u, g[f"vc{i}_f"])
        assert out is u
        assert maxrel(host(u), g[f"vc{i}_uout"]) < tol, (i, maxrel(host(u), g[f"vc{i}_uout"]))
        z = torch.zeros_like(u)
        P.v_cycle(h, z, g[f"vc{i}_f"])
        assert maxrel(host(z), g[f"vc{i}_uzero"]) < tol


def _rates(res):
    res = np.asarray(res)
    return np.log10(res[:-1] / res[1:])


def _check_history(got, want, label):
    assert abs(len(got) - len(want)) <= 1, (label, len(got), len(want))
    n = min(len(got), len(want))
    assert np.max(np.abs(_rates(got[:n]) - _rates(want[:n]))) < 1e-3, label
    rb_got = math.log10(got[0] / got[-1]) / (len(got) - 1)
    rb_want = math.log10(want[0] / want[-1]) / (len(want) - 1)
    assert abs(rb_got - rb_want) < 1e-3, (label, rb_got, rb_want)


@pytest.mark.parametrize("coarse", ["cg", "pinv"])
def test_c1_solver_histories(cuda_device, coarse):
    """BASELINE configs[0]: 8x8, p=8, [0,1]^2, seeded N(0,1) mean-zero f, zero start."""
    g = golden("krylov")
    h = P.build_hierarchy(P.MeshConfig(8, 8, 1.0, 1.0), 8, P.OverlapRule("fixed", 1), coarse=coarse)
    for seed in (0, 1, 2):
        f = O.project_mean(np.random.default_rng(seed).standard_normal((64, 64)))
        for solver in ("mg", "mgcg"):
            u, rep = P.solve(h, f, P.SolveConfig(solver=solver, seed=seed), u0=np.zeros_like(f))
            want = g[f"c1_{solver}_{seed}_res"]
            assert rep.converged and not rep.breakdown
            _check_history(rep.residuals, want, (solver, seed))
            assert rep.cycles == len(rep.residuals) - 1
            if coarse == "cg":
                assert maxrel(host(u), g[f"c1_{solver}_{seed}_u"]) < 1e-9


def test_random_start_and_determinism(cuda_device):
    g = golden("krylov")
    mesh = P.MeshConfig(4, 4)
    h = P.build_hierarchy(mesh, 8, P.OverlapRule("fixed", 1), coarse="cg")
    f = g["rs_f"]
    for solver in ("mg", "mgcg"):
        cfg = P.SolveConfig(solver=solver, tol_reduction=1e8, max_cycles=40, seed=5)
        _, rep1 = P.solve(h, f, cfg)
        _, rep2 = P.solve(h, f, cfg)
        assert rep1.residuals == rep2.residuals  # bitwise (test_krylov.py:73-81)
        _check_history(rep1.residuals, g[f"rs_{solver}_res"], solver)


def test_c2_full_size_histories(cuda_device):
    """BASELINE configs[1]: 64x64, p=16 (1,048,576 DOF), seed 0."""
    g = golden("large_c2")
    mesh = P.MeshConfig(64, 64, 1.0, 1.0)
    f = O.project_mean(np.random.default_rng(0).standard_normal((1024, 1024)))
    for coarse in ("pinv", "cg"):
        h = P.build_hierarchy(mesh, 16, P.OverlapRule("fixed", 1), coarse=coarse)
        u = P.v_cycle(h, torch.zeros(1024, 1024, dtype=torch.float64, device="cuda"), f)
        assert maxrel(host(u)[::16, ::16], g["c2_vcycle_sample"]) < 1e-9
        r = float(torch.linalg.vector_norm(P.residual(h.top.op, u, f)))
        assert abs(r - float(g["c2_vcycle_resnorm"])) < 1e-9 * float(g["c2_vcycle_resnorm"])
        for solver in ("mg", "mgcg"):
            u, rep = P.solve(h, f, P.SolveConfig(solver=solver), u0=np.zeros_like(f))
            _check_history(rep.residuals, g[f"c2_{solver}_res"], (coarse, solver))


@pytest.mark.parametrize("p", [4, 8, 12, 16, 24, 32])
def test_smoother_microbench_parity(cuda_device, p):
    """The smoother-only microbenchmark config: 64x64 elements, n_o=1, random r,
    u=0: one correction vs the CPU oracle."""
    n = 64
    mesh = P.MeshConfig(n, n, 1.0, 1.0)
    b = P.gll_basis(p)
    lay = P.layout_for(mesh, p)
    sm = P.AdditiveSchwarz(b, lay, mesh.dx, mesh.dy, 1, S.WeightKind.QUINTIC)
    r = np.random.default_rng(1).standard_normal(lay.shape)
    u = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
    sm.correct(dev(r), u)
    osm = O.AdditiveSweep(O.gll(p), n, n, mesh.dx, mesh.dy, 1, "w5")
    assert maxrel(host(u), osm.correction(r)) < TOL


def test_dense_coloured_path_parity(cuda_device, monkeypatch):
    """The coloured dense-FD fallback (used when factors are not even/odd)."""
    monkeypatch.setenv("SMG_FD_DENSE", "1")
    g = golden("sweeps")
    for i in range(int(g["n_sw"])):
        op, sm = _sweep_case(g, i)
        u = dev(g[f"sw{i}_u0"])
        sm.smooth(op, u, dev(g[f"sw{i}_f"]), 2)
        assert maxrel(host(u), g[f"sw{i}_u2"]) < TOL


@pytest.mark.parametrize("n_o", [0, 1, 2, 3])
@pytest.mark.parametrize("shape", [(2, 2), (3, 5), (6, 4), (7, 3), (16, 8)])
def test_tiled_sweep_ragged_meshes(cuda_device, n_o, shape):
    """Tile/band protocol on meshes whose element counts force odd tilings,
    single-tile rows/columns and periodic self-neighbours."""
    p = 8
    nx, ny = shape
    if p + 1 + 2 * n_o > p * min(nx, ny):
        pytest.skip("window would alias")
    mesh = P.MeshConfig(nx, ny, 1.3, 0.7)
    b = P.gll_basis(p)
    lay = P.layout_for(mesh, p)
    sm = P.AdditiveSchwarz(b, lay, mesh.dx, mesh.dy, n_o, S.WeightKind.QUINTIC)
    r = np.random.default_rng(nx * 10 + ny).standard_normal(lay.shape)
    u0 = np.random.default_rng(5).standard_normal(lay.shape)
    u = dev(u0)
    sm.correct(dev(r), u)
    osm = O.AdditiveSweep(O.gll(p), nx, ny, mesh.dx, mesh.dy, n_o, "w5")
    want = u0 + osm.correction(r)
    assert maxrel(host(u), want) < TOL
    # bitwise reproducible run to run (counters reset, fixed band order)
    u2 = dev(u0)
    sm.correct(dev(r), u2)
    assert torch.equal(u, u2)


def test_c3_vcycle_full_size(cuda_device):
    """BASELINE configs[2]: 128x128, p=32 (16.8M DOF), one V-cycle from zero."""
    g = golden("xlarge_c3")
    mesh = P.MeshConfig(128, 128, 1.0, 1.0)
    h = P.build_hierarchy(mesh, 32, P.OverlapRule("fixed", 1))
    f = O.project_mean(np.random.default_rng(0).standard_normal((4096, 4096)))
    fd = torch.from_numpy(f).cuda()
    u = P.v_cycle(h, torch.zeros_like(fd), fd)
    assert maxrel(host(u)[::64, ::64], g["c3_vcycle_sample"]) < 1e-9
    assert abs(float(torch.linalg.vector_norm(u)) - float(g["c3_vcycle_norm"])) < 1e-9 * float(g["c3_vcycle_norm"])
    r1 = float(torch.linalg.vector_norm(P.residual(h.top.op, u, fd)))
    assert abs(r1 - g["c3_res"][1]) < 1e-7 * g["c3_res"][1]


def test_c4_mgcg_full_size(cuda_device):
    """BASELINE configs[3]: [0,8]x[0,1], 256x256 elements (AR 8), p=16, MGCG to 1e-10
    (the reference took 21 min on 8 CPU cores for the golden history)."""
    g = golden("xlarge_c4")
    mesh = P.MeshConfig(256, 256, 8.0, 1.0)
    h = P.build_hierarchy(mesh, 16, P.OverlapRule("fixed", 1))
    f = O.project_mean(np.random.default_rng(0).standard_normal((4096, 4096)))
    u, rep = P.solve(h, f, P.SolveConfig(solver="mgcg"), u0=np.zeros_like(f))
    assert rep.converged and not rep.breakdown and not bool(g["c4_breakdown"])
    _check_history(rep.residuals, g["c4_mgcg_res"], "c4")


def test_c5_reduced_mgcg(cuda_device):
    """BASELINE configs[4] geometry and hierarchy at reduced size: variable nu
    (nu_hat=0.9, shift 0 == 1 + 0.9 sin x sin y on [0,2pi]^2), 64x64 elements,
    p=24 with levels (1,3,6,12,24), MGCG to 1e-10, coarse solved by the
    reference's own CG (parity mode)."""
    g = golden("xlarge_c5r")
    mesh = P.MeshConfig(64, 64, 1.0, 1.0)
    h = P.build_hierarchy(mesh, 24, P.OverlapRule("fixed", 1), orders=(1, 3, 6, 12, 24), nu_hat=0.9,
                          nu_shift=0.0, coarse="cg")
    f = O.project_mean(np.random.default_rng(0).standard_normal((1536, 1536)))
    u, rep = P.solve(h, f, P.SolveConfig(solver="mgcg"), u0=np.zeros_like(f))
    assert rep.converged and not rep.breakdown
    _check_history(rep.residuals, g["c5r_mgcg_res"], "c5r")
    assert maxrel(host(u)[::24, ::24], g["c5r_mgcg_sample"]) < 1e-6


def test_diffusion_coarse_pcg_vs_reference(cuda_device):
    """Fast coarse mode for variable nu: preconditioned CG reaches the
    reference CG's answer to within its own 1e-12 tolerance (x condition)."""
    g = golden("multigrid")
    mesh = P.MeshConfig(8, 8, 1.0, 1.0)
    h = P.build_hierarchy(mesh, 2, P.OverlapRule("fixed", 1), nu_hat=0.9, coarse="pcg")
    got = host(P.coarse_solve(h, g["cs3_f0"]))
    assert maxrel(got, g["cs3_u0"]) < 1e-9
    assert h.coarse_iterations[-1] < 100


def test_c5_reduced_mgcg_fast_coarse(cuda_device):
    """Reduced C5 with the default (PCG) coarse solver: same history within tolerance."""
    g = golden("xlarge_c5r")
    mesh = P.MeshConfig(64, 64, 1.0, 1.0)
    h = P.build_hierarchy(mesh, 24, P.OverlapRule("fixed", 1), orders=(1, 3, 6, 12, 24), nu_hat=0.9,
                          nu_shift=0.0)
    assert h.coarse == "pcg"
    f = O.project_mean(np.random.default_rng(0).standard_normal((1536, 1536)))
    u, rep = P.solve(h, f, P.SolveConfig(solver="mgcg"), u0=np.zeros_like(f))
    assert rep.converged and not rep.breakdown
    _check_history(rep.residuals, g["c5r_mgcg_res"], "c5r-pcg")
    assert max(h.coarse_iterations) < 120
