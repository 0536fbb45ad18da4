"""Small driver for ncu captures: runs each hot kernel a few times on one config.

    python tools/prof_kernels.py --n 256 --p 16 [--what fd,op,restrict,prolong]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as NV  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--p", type=int, default=16)
ap.add_argument("--n_o", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--what", default="fd,op,restrict,prolong,diff")
a = ap.parse_args()
what = a.what.split(",")
mesh = P.MeshConfig(a.n, a.n, 1.0, 1.0)
lay = P.layout_for(mesh, a.p)
b = P.gll_basis(a.p)
r = torch.randn(lay.shape, dtype=torch.float64, device="cuda")
u = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
out = torch.empty_like(u)
if "fd" in what:
    sm = P.AdditiveSchwarz(b, lay, mesh.dx, mesh.dy, a.n_o, P.WeightKind.QUINTIC)
    for _ in range(a.reps):
        sm.correct(r, u)
if "op" in what:
    op = P.PoissonOperator(b, mesh)
    for _ in range(a.reps):
        op.residual_into(u, r, out)
if "diff" in what:
    nu = 1.0 + 0.5 * torch.rand(lay.shape, dtype=torch.float64)
    dop = P.DiffusionOperator(b, mesh, nu.numpy())
    for _ in range(a.reps):
        dop.residual_into(u, r, out)
if "restrict" in what or "prolong" in what:
    h = P.build_hierarchy(mesh, a.p, P.OverlapRule("fixed", 1))
    for _ in range(a.reps):
        if "restrict" in what:
            P.restrict_residual(h, h.depth, r)
        if "prolong" in what:
            P.prolongate(h, h.depth, h.levels[-2].u)
torch.cuda.synchronize()
print("done", NV.lib().smg_launch_count())
