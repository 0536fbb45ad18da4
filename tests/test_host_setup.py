"""CPU tests of the product's host-side setup and API plumbing, pinned to the
reference's golden vectors (no GPU needed)."""

import math

import numpy as np
import pytest

from conftest import golden
import paper_1512_02390_b200 as P
from paper_1512_02390_b200 import schwarz as S
from paper_1512_02390_b200.metrics import cycle_cost, cycles_per_decade10


def test_basis_bitwise_vs_reference():
    g = golden("basis")
    for p in [1, 2, 3, 4, 5, 6, 8, 12, 16, 24, 32]:
        b = P.gll_basis(p)
        for k in ("nodes", "weights", "diff", "stiff"):
            np.testing.assert_array_equal(getattr(b, k), g[f"{k}_{p}"])
    for pc, pf in [(1, 2), (2, 4), (4, 8), (8, 16), (16, 32), (1, 3), (3, 6), (6, 12), (12, 24)]:
        np.testing.assert_array_equal(P.interp_matrix(P.gll_basis(pc), P.gll_basis(pf)).matrix, g[f"J_{pc}_{pf}"])
    with pytest.raises(ValueError):
        P.gll_basis(0)
    with pytest.raises(ValueError):
        P.interp_matrix(P.gll_basis(4), P.gll_basis(2))


def test_fd_factors_and_weights_bitwise_vs_reference():
    g = golden("schwarz_setup")
    for kind in S.WeightKind:
        for p, n_o in [(2, 1), (4, 1), (8, 1), (8, 2), (16, 1), (16, 2), (24, 1), (24, 3), (32, 1), (32, 4)]:
            b = P.gll_basis(p)
            w = S.build_weight_1d(kind, b, S.subdomain_geometry(b, n_o))
            np.testing.assert_array_equal(w, g[f"w_{kind.value}_{p}_{n_o}"])
    for i in range(int(g["n_fd"])):
        p, n_o, dx, dy = g[f"fd{i}_case"]
        b = P.gll_basis(int(p))
        L, m = S.restricted_1d(b, dx, int(n_o))
        np.testing.assert_array_equal(L, g[f"fd{i}_L"])
        np.testing.assert_array_equal(m, g[f"fd{i}_m"])
        fd = S.build_fast_diag(b, dx, dy, int(n_o), S.WeightKind.QUINTIC)
        np.testing.assert_array_equal(fd.S_x, g[f"fd{i}_Sx"])
        np.testing.assert_array_equal(fd.S_y, g[f"fd{i}_Sy"])
        np.testing.assert_array_equal(fd.lam_x, g[f"fd{i}_lx"])
        np.testing.assert_array_equal(fd.lam_y, g[f"fd{i}_ly"])
        np.testing.assert_array_equal(fd.weight, g[f"fd{i}_W"])


def test_weight_profiles_partition_of_unity():
    for kind in S.WeightKind:
        for p, n_o in [(4, 1), (8, 2), (16, 1)]:
            b = P.gll_basis(p)
            w = S.build_weight_1d(kind, b, S.subdomain_geometry(b, n_o))
            total = np.zeros(8 * p)
            np.add.at(total, (np.arange(8)[:, None] * p + np.arange(-n_o, p + n_o + 1)[None, :]) % (8 * p),
                      np.broadcast_to(w, (8, w.size)))
            np.testing.assert_allclose(total, 1.0, atol=1e-13)
    with pytest.raises(ValueError):
        S.weight_value(S.WeightKind.QUINTIC, 0.0, 0.0)
    with pytest.raises(ValueError):
        S.restricted_1d(P.gll_basis(4), 0.5, 4)


def test_jacobi_matches_lapack_and_zero():
    rng = np.random.default_rng(31)
    for n in (3, 6, 15):
        a = rng.standard_normal((n, n))
        a = a + a.T
        lam, v = S.jacobi_eigh(a)
        np.testing.assert_allclose(lam, np.linalg.eigvalsh(a), atol=1e-12 * np.abs(lam).max())
        np.testing.assert_allclose(v.T @ v, np.eye(n), atol=1e-12)
    lam, v = S.jacobi_eigh(np.zeros((4, 4)))
    assert np.all(lam == 0) and np.array_equal(v, np.eye(4))


def test_overlap_rule_and_configs():
    R = P.OverlapRule
    assert R("fixed", 2).layers(8) == 2 and R("floorp8").layers(4) == 0
    assert R("ceilp8").layers(16) == 2 and R("ceilp2").layers(8) == 4
    assert R("fixed", 5).layers(2) == 1
    assert R.parse("fixed:3") == R("fixed", 3)
    with pytest.raises(ValueError):
        R.parse("fixed")
    with pytest.raises(ValueError):
        R("quadratic").layers(8)
    P.SolveConfig()
    for bad in (dict(tol_reduction=1.0), dict(max_cycles=0), dict(solver="jacobi")):
        with pytest.raises(ValueError):
            P.SolveConfig(**bad)


def test_metrics_match_reference_formulas():
    rep = P.ConvergenceReport([1.0, 0.1, 0.01], True, 2, 0.0)
    assert rep.rbar == pytest.approx(1.0) and rep.n10 == 10
    rep = P.ConvergenceReport([1.0], True, 0, 0.0)
    assert math.isinf(rep.rbar) and rep.n10 == 0
    assert cycles_per_decade10(1.3) == 8
    w_cyc, w_op, ratio = cycle_cost(16, 64, 2, 1)
    assert w_op == 2.0 * 17 ** 3 * 64 and ratio == pytest.approx(w_cyc / w_op)


def test_mesh_validation_and_windows():
    with pytest.raises(ValueError):
        P.MeshConfig(1, 4)
    with pytest.raises(ValueError):
        P.MeshConfig(2, 2, l_x=0.0)
    m = P.MeshConfig(4, 2, 8.0, 2.0)
    assert m.dx == 2.0 and m.aspect_ratio == 2.0 and m.n_el == 8
    from paper_1512_02390_b200.mesh import FieldLayout, element_indices
    iy, ix = element_indices(FieldLayout(2, 3, 2), 2, 1)
    assert list(ix) == [4, 5, 0] and list(iy) == [2, 3, 0]
    with pytest.raises(IndexError):
        element_indices(FieldLayout(2, 3, 2), 3, 0)


def test_public_names_cover_reference_hot_path():
    names = ["Basis1D", "Interp1D", "gll_basis", "interp_matrix", "overlap_width", "SolveConfig", "solve",
             "solve_mg", "solve_mgcg", "Field", "FieldLayout", "MeshConfig", "gather_element",
             "scatter_add_element", "ConvergenceReport", "convergence_rate", "cycle_cost", "work_per_decades",
             "MultigridHierarchy", "OverlapRule", "build_hierarchy", "coarse_solve", "prolongate",
             "restrict_residual", "v_cycle", "DiffusionOperator", "PoissonOperator",
             "manufactured_rhs_diffusion", "manufactured_rhs_poisson", "residual", "AdditiveSchwarz",
             "FastDiagSolver", "MultiplicativeSchwarz", "WeightKind", "build_fast_diag", "restricted_1d",
             "weight_value"]
    for n in names:
        assert hasattr(P, n), n


def test_problem_builders_host():
    mesh = P.MeshConfig(3, 2, 3.0, 4.0)
    from paper_1512_02390_b200.operators import load_vector
    f = load_vector(mesh, P.gll_basis(4), lambda x, y: np.ones_like(x))
    np.testing.assert_allclose(f.sum(), 12.0, rtol=1e-13)
    g = golden("operators")
    for i in range(int(g["n_op"])):
        nx, ny, lx, ly, p = g[f"op{i}_case"]
        msh = P.MeshConfig(int(nx), int(ny), lx, ly)
        np.testing.assert_allclose(P.diffusivity_field(msh, P.gll_basis(int(p)), 0.9, 0.0), g[f"op{i}_nufield"],
                                   rtol=0, atol=1e-15)
