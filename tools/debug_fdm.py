import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P
from oracle import smg_oracle as O
for n, p in [(64, 16), (16, 16), (8, 16)]:
    mesh = P.MeshConfig(n, n, 1.0, 1.0); lay = P.layout_for(mesh, p)
    os.environ["SMG_FD_ENGINE"] = "dmma"
    sm = P.AdditiveSchwarz(P.gll_basis(p), lay, mesh.dx, mesh.dy, 1, P.WeightKind.QUINTIC)
    r = np.random.default_rng(1).standard_normal(lay.shape)
    u = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
    sm.correct(torch.from_numpy(r).cuda(), u)
    want = O.AdditiveSweep(O.gll(p), n, n, mesh.dx, mesh.dy, 1, "w5").correction(r)
    err = np.abs(u.cpu().numpy() - want)
    bad = np.argwhere(err > 1e-9 * np.abs(want).max())
    print(n, p, "maxrel", err.max() / np.abs(want).max(), "nbad", len(bad))
    if len(bad):
        ys, xs = bad[:, 0], bad[:, 1]
        print("  rows", np.unique(ys // p)[:20], "cols", np.unique(xs // p)[:20])
        print("  local rows", np.unique(ys % p), "local cols", np.unique(xs % p)[:20])
