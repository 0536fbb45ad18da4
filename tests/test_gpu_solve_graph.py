"""Graph-captured solver cycles (krylov.py) against the eager launches:
identical residual histories (bitwise) for MG and MGCG."""

import numpy as np
import pytest

import paper_1512_02390_b200 as P
from oracle import smg_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("solver", ["mg", "mgcg"])
@pytest.mark.parametrize("case", [(8, 8, 8, 1.0), (16, 8, 16, 4.0)])
def test_solve_graph_bitwise(cuda_device, monkeypatch, solver, case):
    nx, ny, p, lx = case
    mesh = P.MeshConfig(nx, ny, lx, 1.0)
    f = O.project_mean(np.random.default_rng(nx + p).standard_normal((p * ny, p * nx)))
    out = {}
    for graph in ("1", "0"):
        monkeypatch.setenv("SMG_SOLVE_GRAPH", graph)
        h = P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1))
        u, rep = P.solve(h, f, P.SolveConfig(solver=solver), u0=np.zeros_like(f))
        out[graph] = (u.cpu().numpy(), rep.residuals, rep.cycles)
    assert out["1"][1] == out["0"][1] and out["1"][2] == out["0"][2]
    assert np.array_equal(out["1"][0], out["0"][0])
