import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P
from oracle import smg_oracle as O
def run(nx, ny, p, n_o, nu_hat, lx, ly):
    mesh = P.MeshConfig(nx, ny, lx, ly); b = P.gll_basis(p); lay = P.layout_for(mesh, p)
    ob = O.gll(p)
    if nu_hat is None:
        op = P.PoissonOperator(b, mesh); nb = None; oop = O.Poisson(ob, nx, ny, mesh.dx, mesh.dy)
    else:
        nu = P.diffusivity_field(mesh, b, nu_hat, 0.2)
        op = P.DiffusionOperator(b, mesh, nu); nb = op.element_mean_nu()
        oop = O.Diffusion(ob, nx, ny, mesh.dx, mesh.dy, nu)
    rng = np.random.default_rng(1); u0 = rng.standard_normal(lay.shape); f = rng.standard_normal(lay.shape)
    sm = P.MultiplicativeSchwarz(b, lay, mesh.dx, mesh.dy, n_o, nu_bar=nb)
    u = torch.from_numpy(u0.copy()).cuda(); sm.smooth(op, u, f, 1)
    osm = O.MultSweep(ob, nx, ny, mesh.dx, mesh.dy, n_o, None if nb is None else oop.element_mean_nu())
    want = osm.smooth(oop, u0.copy(), f, 1)
    got = u.cpu().numpy()
    print((nx, ny, p, n_o, nu_hat, lx, ly), np.abs(got - want).max() / np.abs(want).max())
for c in [(6,4,8,1,0.9,2.0,1.0),(6,4,8,1,None,2.0,1.0),(4,4,8,1,0.9,1.0,1.0),(6,4,8,1,0.9,1.0,1.0),(4,6,8,1,0.9,1.0,1.0),(4,4,4,1,0.5,1.0,1.0),(5,5,4,1,0.5,1.0,1.0)]:
    run(*c)
