import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_1512_02390_b200 as P
n, p = int(sys.argv[1]), int(sys.argv[2])
mesh = P.MeshConfig(n, n, 1.0, 1.0)
lay = P.layout_for(mesh, p)
sm = P.AdditiveSchwarz(P.gll_basis(p), lay, mesh.dx, mesh.dy, 1, P.WeightKind.QUINTIC)
r = torch.randn(lay.shape, dtype=torch.float64, device="cuda")
u = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
sm.correct(r, u)
torch.cuda.synchronize()
print("ok", n, p, float(u.abs().sum()))
