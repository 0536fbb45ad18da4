"""Halo-free tensor-core operator kernel (opdh_kernel + fixup, SMG_OPDH=1) against the fused
kernel (SMG_OPDH=0 is read once per process: compare through the ring-less entry point) and
the oracle: residual and apply, diffusion p = 24 and Poisson p = 32.  GPU."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as N  # noqa: E402
from oracle import smg_oracle as O  # noqa: E402

worst = 0.0
for kind, p, nx, ny, lx, ly in [("diffusion", 12, 4, 3, 1.0, 1.0), ("diffusion", 12, 16, 8, 1.0, 3.0), ("diffusion", 24, 4, 3, 1.0, 1.0), ("diffusion", 24, 8, 8, 2.0, 1.0),
                                ("poisson", 32, 3, 4, 1.0, 1.3), ("poisson", 32, 8, 8, 1.0, 1.0)]:
    mesh = P.MeshConfig(nx, ny, lx, ly)
    b = P.gll_basis(p)
    rng = np.random.default_rng(5)
    lay = P.layout_for(mesh, p)
    u = rng.standard_normal(lay.shape)
    f = rng.standard_normal(lay.shape)
    if kind == "poisson":
        op = P.PoissonOperator(b, mesh)
        want = O.Poisson(O.gll(p), nx, ny, mesh.dx, mesh.dy).apply(u)
    else:
        nu = 1 + 0.5 * rng.random(lay.shape)
        op = P.DiffusionOperator(b, mesh, nu)
        want = O.Diffusion(O.gll(p), nx, ny, mesh.dx, mesh.dy, nu).apply(u)
    assert op.ring is not None, "no ring: the halo-free kernel is not engaged"
    ud, fd = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
    got = op.apply(ud).cpu().numpy()
    r = torch.empty_like(ud)
    op.residual_into(ud, fd, r)
    old = torch.empty_like(ud)
    N.check(N.lib().smg_op_residual(op._handle.raw, N.ptr(ud), N.ptr(fd), N.ptr(old), N.stream()), "residual")   # ring-less kernels
    sc = np.abs(want).max()
    e1 = np.abs(got - want).max() / sc
    e2 = np.abs(r.cpu().numpy() - (f - want)).max() / sc
    e3 = (r - old).abs().max().item() / sc
    worst = max(worst, e1, e2, e3)
    print(f"{kind} p={p} {nx}x{ny}: apply vs oracle {e1:.2e}  residual vs oracle {e2:.2e}  vs fused kernel {e3:.2e}", flush=True)
print("worst", worst)
sys.exit(0 if worst < 1e-12 else 1)
