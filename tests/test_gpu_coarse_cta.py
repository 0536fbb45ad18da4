"""The one-CTA coarse CG (smg_blas.cu ccg_cta_kernel, Poisson p = 1 meshes up
to 64 x 64): solution within 1e-10 of the reference's plain CG restatement
(multigrid.py:196-228, oracle.cg) with the same iteration count (+-1: the
stencil sums in another order than the reference's element loop), and the
same answer as the grid-wide path it replaces (SMG_CCG_CTA=0, subprocess)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import maxrel
from oracle import smg_oracle as O

pytestmark = pytest.mark.gpu

CASES = [(3, 3, 1.0, 1.0), (3, 5, 1.0, 1.0), (8, 8, 1.0, 1.0), (16, 12, 2.0, 0.5), (64, 64, 1.0, 1.0),
         (64, 48, 1.0, 3.0), (128, 32, 1.0, 1.0)]


def _f0(nx, ny):
    return np.random.default_rng(nx * 1000 + ny).standard_normal((ny, nx)) + 0.25


@pytest.mark.parametrize("case", CASES)
def test_cta_cg_vs_oracle(cuda_device, case):
    import paper_1512_02390_b200 as P
    nx, ny, lx, ly = case
    f0 = _f0(nx, ny)
    h = P.build_hierarchy(P.MeshConfig(nx, ny, lx, ly), 2, P.OverlapRule("fixed", 1), coarse="cg")
    got = P.coarse_solve(h, f0).cpu().numpy()
    ho = O.Hierarchy(nx, ny, lx, ly, 2)
    want = O.coarse_solve(ho, f0)
    assert maxrel(got, want) < 1e-10, maxrel(got, want)
    assert abs(h.coarse_iterations[-1] - ho.coarse_iters[-1]) <= 1, (h.coarse_iterations, ho.coarse_iters)
    assert abs(got.sum()) < 1e-12 * max(1.0, np.abs(got).sum())
    # deterministic: a second solve is bitwise equal
    assert np.array_equal(P.coarse_solve(h, f0).cpu().numpy(), got)


def test_cta_cg_matches_grid_path(cuda_device, tmp_path):
    import paper_1512_02390_b200 as P
    nx, ny = 64, 64
    f0 = _f0(nx, ny)
    h = P.build_hierarchy(P.MeshConfig(nx, ny, 1.0, 1.0), 2, P.OverlapRule("fixed", 1), coarse="cg")
    cta = P.coarse_solve(h, f0).cpu().numpy()
    np.save(tmp_path / "f0.npy", f0)
    code = (
        "import numpy as np, paper_1512_02390_b200 as P\n"
        f"f0 = np.load(r'{tmp_path / 'f0.npy'}')\n"
        "h = P.build_hierarchy(P.MeshConfig(64, 64, 1.0, 1.0), 2, P.OverlapRule('fixed', 1), coarse='cg')\n"
        f"np.save(r'{tmp_path / 'grid.npy'}', P.coarse_solve(h, f0).cpu().numpy())\n"
        "print(h.coarse_iterations[-1])\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, SMG_CCG_CTA="0"),
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    grid = np.load(tmp_path / "grid.npy")
    assert maxrel(cta, grid) < 1e-10
    assert abs(int(out.stdout.split()[-1]) - h.coarse_iterations[-1]) <= 1
