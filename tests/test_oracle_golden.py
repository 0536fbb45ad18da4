"""Pin the CPU oracle (oracle/smg_oracle.py) against golden vectors produced
by the unmodified reference (oracle/make_golden.py)."""

import numpy as np
import pytest

from conftest import golden, maxrel
from oracle import smg_oracle as O


def test_basis_bitwise():
    g = golden("basis")
    for p in [1, 2, 3, 4, 5, 6, 8, 12, 16, 24, 32]:
        b = O.gll(p)
        np.testing.assert_array_equal(b.nodes, g[f"nodes_{p}"])
        np.testing.assert_array_equal(b.weights, g[f"weights_{p}"])
        np.testing.assert_array_equal(b.diff, g[f"diff_{p}"])
        np.testing.assert_array_equal(b.stiff, g[f"stiff_{p}"])
    for pc, pf in [(1, 2), (2, 4), (4, 8), (8, 16), (16, 32), (1, 3), (3, 6), (6, 12), (12, 24)]:
        np.testing.assert_array_equal(O.interp(O.gll(pc), O.gll(pf)), g[f"J_{pc}_{pf}"])


def test_weights_bitwise():
    g = golden("schwarz_setup")
    for kind in O.WEIGHT_KINDS:
        for p, n_o in [(2, 1), (4, 1), (8, 1), (8, 2), (16, 1), (16, 2), (24, 1), (24, 3), (32, 1), (32, 4)]:
            np.testing.assert_array_equal(O.weights_1d(kind, O.gll(p), n_o), g[f"w_{kind}_{p}_{n_o}"])


def test_fd_factors_bitwise_and_solve():
    g = golden("schwarz_setup")
    for i in range(int(g["n_fd"])):
        p, n_o, dx, dy = g[f"fd{i}_case"]
        p, n_o = int(p), int(n_o)
        b = O.gll(p)
        L, m = O.restricted_patch(b, dx, n_o)
        np.testing.assert_array_equal(L, g[f"fd{i}_L"])
        np.testing.assert_array_equal(m, g[f"fd{i}_m"])
        fd = O.fast_diag(b, dx, dy, n_o, "w5")
        # the cyclic Jacobi restatement reproduces the reference factors exactly
        np.testing.assert_array_equal(fd.Sx, g[f"fd{i}_Sx"])
        np.testing.assert_array_equal(fd.Sy, g[f"fd{i}_Sy"])
        np.testing.assert_array_equal(fd.lx, g[f"fd{i}_lx"])
        np.testing.assert_array_equal(fd.ly, g[f"fd{i}_ly"])
        np.testing.assert_array_equal(fd.W, g[f"fd{i}_W"])
        assert maxrel(fd.solve(g[f"fd{i}_r"]), g[f"fd{i}_solve"]) < 1e-14


def test_operators():
    g = golden("operators")
    for i in range(int(g["n_op"])):
        nx, ny, lx, ly, p = g[f"op{i}_case"]
        nx, ny, p = int(nx), int(ny), int(p)
        b = O.gll(p)
        u = g[f"op{i}_u"]
        A = O.Poisson(b, nx, ny, lx / nx, ly / ny)
        assert maxrel(A.apply(u), g[f"op{i}_Au"]) < 1e-14
        B = O.Diffusion(b, nx, ny, lx / nx, ly / ny, g[f"op{i}_nu"])
        assert maxrel(B.apply(u), g[f"op{i}_Bu"]) < 1e-14
        assert maxrel(B.element_mean_nu(), g[f"op{i}_nubar"]) < 1e-15
        np.testing.assert_allclose(O.diffusivity(b, nx, ny, lx / nx, ly / ny, 0.9, 0.0),
                                   g[f"op{i}_nufield"], rtol=0, atol=1e-15)


def test_sweeps():
    g = golden("sweeps")
    for i in range(int(g["n_sw"])):
        nx, ny, lx, ly, p, n_o, nu_hat = g[f"sw{i}_case"]
        nx, ny, p, n_o = int(nx), int(ny), int(p), int(n_o)
        kind = str(g[f"sw{i}_kind"])
        b = O.gll(p)
        dx, dy = lx / nx, ly / ny
        if nu_hat < 0:
            op, nb = O.Poisson(b, nx, ny, dx, dy), None
        else:
            op = O.Diffusion(b, nx, ny, dx, dy, O.diffusivity(b, nx, ny, dx, dy, nu_hat, 0.2))
            nb = op.element_mean_nu()
        sm = O.AdditiveSweep(b, nx, ny, dx, dy, n_o, kind, nb)
        assert maxrel(sm.smooth(op, g[f"sw{i}_u0"].copy(), g[f"sw{i}_f"], 1), g[f"sw{i}_u1"]) < 1e-13
        assert maxrel(sm.smooth(op, g[f"sw{i}_u0"].copy(), g[f"sw{i}_f"], 2), g[f"sw{i}_u2"]) < 1e-13


def test_transfers_coarse_vcycle():
    g = golden("multigrid")
    h = O.Hierarchy(4, 3, 2.0, 2.0, 32)
    for l in range(1, h.depth + 1):
        assert maxrel(O.prolongate(h, l, g[f"tr{l}_uc"]), g[f"tr{l}_P"]) < 1e-14
        assert maxrel(O.restrict(h, l, g[f"tr{l}_vf"]), g[f"tr{l}_R"]) < 1e-14
    for i, (nx, ny, lx, ly, nu_hat) in enumerate([(4, 4, 2.0, 2.0, None), (8, 8, 1.0, 1.0, None),
                                                   (16, 8, 8.0, 1.0, None), (8, 8, 1.0, 1.0, 0.9)]):
        h = O.Hierarchy(nx, ny, lx, ly, 2, nu_hat=nu_hat)
        assert maxrel(O.coarse_solve(h, g[f"cs{i}_f0"]), g[f"cs{i}_u0"]) < 1e-12
    for i in range(4):
        nx, ny, lx, ly, p, nu_hat, n_post = g[f"vc{i}_case"]
        h = O.Hierarchy(int(nx), int(ny), lx, ly, int(p), rule=str(g[f"vc{i}_rule"]),
                        nu_hat=None if nu_hat < 0 else nu_hat, n_post=int(n_post))
        assert maxrel(O.v_cycle(h, g[f"vc{i}_uin"].copy(), g[f"vc{i}_f"]), g[f"vc{i}_uout"]) < 1e-12
        assert maxrel(O.v_cycle(h, np.zeros_like(g[f"vc{i}_f"]), g[f"vc{i}_f"]), g[f"vc{i}_uzero"]) < 1e-12


def test_c1_histories():
    g = golden("krylov")
    h = O.Hierarchy(8, 8, 1.0, 1.0, 8)
    for seed in (0, 1, 2):
        f = O.project_mean(np.random.default_rng(seed).standard_normal((64, 64)))
        u, res, ok = O.solve_mg(h, f, seed=seed, u0=np.zeros_like(f))
        want = g[f"c1_mg_{seed}_res"]
        assert ok and len(res) == len(want)
        np.testing.assert_allclose(res, want, rtol=1e-9)
        u, res, ok, broke = O.solve_mgcg(h, f, seed=seed, u0=np.zeros_like(f))
        want = g[f"c1_mgcg_{seed}_res"]
        assert ok and not broke and len(res) == len(want)
        np.testing.assert_allclose(res, want, rtol=1e-9)
    # random-start path (krylov.py:36-39)
    h = O.Hierarchy(4, 4, 2.0, 2.0, 8)
    f = g["rs_f"]
    _, res, _ = O.solve_mg(h, f, tol=1e8, max_cycles=40, seed=5)
    np.testing.assert_allclose(res, g["rs_mg_res"], rtol=1e-9)
    _, res, _, _ = O.solve_mgcg(h, f, tol=1e8, max_cycles=40, seed=5)
    np.testing.assert_allclose(res, g["rs_mgcg_res"], rtol=1e-9)


def _mult_op(nx, ny, p, nu_hat, lx, ly):
    b = O.gll(p)
    dx, dy = lx / nx, ly / ny
    if nu_hat < 0:
        return b, O.Poisson(b, nx, ny, dx, dy), None
    op = O.Diffusion(b, nx, ny, dx, dy, O.diffusivity(b, nx, ny, dx, dy, nu_hat, 0.2))
    return b, op, op.element_mean_nu()


def test_multiplicative_sweeps_vs_reference():
    """schwarz.py:293-353 forward then reverse sweep."""
    g = golden("mult")
    for i in range(6):
        nx, ny, p, n_o, nu_hat, lx, ly = g[f"ms{i}_case"]
        nx, ny, p, n_o = int(nx), int(ny), int(p), int(n_o)
        b, op, nu_bar = _mult_op(nx, ny, p, nu_hat, lx, ly)
        sm = O.MultSweep(b, nx, ny, lx / nx, ly / ny, n_o, nu_bar)
        u = g[f"ms{i}_u"].copy()
        f = g[f"ms{i}_f"]
        sm.smooth(op, u, f, 1)
        assert maxrel(u, g[f"ms{i}_u1"]) < 1e-12, (i, maxrel(u, g[f"ms{i}_u1"]))
        sm.smooth(op, u, f, 1)
        assert maxrel(u, g[f"ms{i}_u2"]) < 1e-12, (i, maxrel(u, g[f"ms{i}_u2"]))


def test_multiplicative_vcycle_and_histories():
    g = golden("mult")
    for j in range(2):
        nx, p, nu_hat = g[f"mv{j}_case"]
        nx, p = int(nx), int(p)
        h = O.Hierarchy(nx, nx, 1.0, 1.0, p, smoother="mult", nu_hat=None if nu_hat < 0 else nu_hat)
        f = g[f"mv{j}_f"]
        h.reset_smoothers()
        out = O.v_cycle(h, g[f"mv{j}_uin"].copy(), f)
        assert maxrel(out, g[f"mv{j}_uout"]) < 1e-10
        _, res, ok = O.solve_mg(h, f, u0=np.zeros_like(f))
        want = g[f"mv{j}_mg_res"]
        assert ok and len(res) == len(want)
        np.testing.assert_allclose(res, want, rtol=1e-8)
        _, res, ok, brk = O.solve_mgcg(h, f, u0=np.zeros_like(f))
        want = g[f"mv{j}_mgcg_res"]
        assert ok and not brk and len(res) == len(want)
        np.testing.assert_allclose(res, want, rtol=1e-8)
