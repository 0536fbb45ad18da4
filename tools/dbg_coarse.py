import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1512_02390_b200 as P
pre = sys.argv[1] if len(sys.argv) > 1 else ""
if "op" in pre:
    mesh = P.MeshConfig(8, 8, 1.0, 1.0)
    op = P.PoissonOperator(P.gll_basis(4), mesh)
    u = torch.randn(op.layout.shape, dtype=torch.float64, device="cuda")
    out = torch.empty_like(u); op.residual_into(u, u, out); torch.cuda.synchronize(); print("op ok")
for nx, ny in [(8, 8), (4, 4), (16, 8), (64, 64)]:
    mesh = P.MeshConfig(nx, ny, 1.0, 1.0)
    hp = P.build_hierarchy(mesh, 2, P.OverlapRule("fixed", 1))
    f = np.random.default_rng(0).standard_normal((ny, nx)); f -= f.mean()
    try:
        got = P.coarse_solve(hp, f); torch.cuda.synchronize()
        print(nx, ny, "ok", float(got.abs().max()))
    except Exception as e:
        print(nx, ny, "ERR", repr(e)[:200]); break
