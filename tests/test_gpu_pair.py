"""Paired-line Schwarz engine (csrc/smg_fdp.cuh) on the GPU: selected where it is
compiled, equal to the reference's sweep (golden fixtures, oracle) at 1e-12, equal to the
even/odd tiled engine to rounding, bitwise reproducible.  Reference: schwarz.py:215-222,
255-275; mesh.py:124-150."""
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _smoother(P, p, nx, ny, lx, ly, n_o, nu_bar=None, engine=None):
    old = os.environ.get("SMG_FD_ENGINE")
    if engine is None:
        os.environ.pop("SMG_FD_ENGINE", None)
    else:
        os.environ["SMG_FD_ENGINE"] = engine
    try:
        mesh = P.MeshConfig(nx, ny, lx, ly)
        lay = P.layout_for(mesh, p)
        return P.AdditiveSchwarz(P.gll_basis(p), lay, mesh.dx, mesh.dy, n_o, P.WeightKind.QUINTIC, nu_bar=nu_bar), lay
    finally:
        if old is None:
            os.environ.pop("SMG_FD_ENGINE", None)
        else:
            os.environ["SMG_FD_ENGINE"] = old


CASES = [  # p, n_x, n_y, l_x, l_y, n_o, diffusion
    (6, 8, 4, 1.0, 1.0, 1, True),
    (8, 4, 4, 1.0, 1.0, 1, False),      # every tile is a seam tile
    (8, 16, 12, 1.0, 3.0, 1, True),
    (12, 8, 8, 1.0, 1.0, 1, False),
    (12, 8, 4, 2.0, 1.0, 2, True),
    (16, 4, 4, 1.0, 1.0, 1, False),
    (16, 12, 8, 8.0, 1.0, 1, True),     # aspect ratio 8 (C4's geometry)
    (16, 8, 6, 1.0, 1.0, 1, False),     # only the 4x2 tile divides
    (16, 8, 8, 1.0, 1.0, 2, True),
    (24, 8, 4, 1.0, 1.0, 1, True),
    (24, 4, 4, 1.0, 1.0, 3, False),
    (32, 8, 4, 1.0, 1.0, 1, False),
    (32, 4, 4, 1.0, 1.0, 4, True),
]


@pytest.mark.parametrize("p,nx,ny,lx,ly,n_o,diff", CASES)
def test_pair_engine_matches_oracle_and_tiled_engine(p, nx, ny, lx, ly, n_o, diff):
    import paper_1512_02390_b200 as P
    from oracle import smg_oracle as O
    rng = np.random.default_rng(100 * p + n_o)
    nub = 0.25 + rng.random((ny, nx)) if diff else None
    sm, lay = _smoother(P, p, nx, ny, lx, ly, n_o, nub)
    eng, tx, ty = sm.kernel_info()
    assert eng == "pair", (eng, tx, ty)
    assert nx % tx == 0 and ny % ty == 0
    r = rng.standard_normal(lay.shape)
    u0 = rng.standard_normal(lay.shape)
    u = torch.from_numpy(u0).cuda()
    sm.correct(torch.from_numpy(r).cuda(), u)
    got = u.cpu().numpy() - u0
    ref = O.AdditiveSweep(O.gll(p), nx, ny, lx / nx, ly / ny, n_o, "w5", nu_bar=nub).correction(r)
    sc = np.abs(ref).max()
    assert np.abs(got - ref).max() / sc < 1e-12
    old, _ = _smoother(P, p, nx, ny, lx, ly, n_o, nub, engine="dfma")
    assert old.kernel_info()[0] == "tiled-dfma"
    u2 = torch.from_numpy(u0).cuda()
    old.correct(torch.from_numpy(r).cuda(), u2)
    assert np.abs(u2.cpu().numpy() - u0 - got).max() / sc < 1e-13
    # bitwise reproducible; u_is_zero writes instead of adding
    u3 = torch.from_numpy(u0).cuda()
    sm.correct(torch.from_numpy(r).cuda(), u3)
    assert torch.equal(u3, u)


def test_pair_engine_golden_sweeps():
    """The reference's own smooth() outputs (tests/golden/sweeps.npz) with the default engine
    selection; the paired-line kernel must be the one that ran wherever it is compiled and a
    tile divides the mesh."""
    from test_gpu_parity import TOL, _sweep_case, dev, golden, host, maxrel
    g = golden("sweeps")
    engines = []
    for i in range(int(g["n_sw"])):
        op, sm = _sweep_case(g, i)
        engines.append(sm.kernel_info()[0])
        u = dev(g[f"sw{i}_u0"])
        sm.smooth(op, u, dev(g[f"sw{i}_f"]), 2)
        assert maxrel(host(u), g[f"sw{i}_u2"]) < TOL, (i, engines[-1])
    assert "pair" in engines, engines
