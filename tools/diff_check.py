"""Diffusion operator (op_kernel, fused residual+restriction) vs the oracle at
several orders / tilings; prints max-relative errors.  GPU."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from oracle import smg_oracle as O  # noqa: E402

for n, p in [(4, 8), (8, 4), (4, 3), (8, 8), (2, 24), (4, 12), (4, 6), (16, 2)]:
    mesh = P.MeshConfig(n, n, 1.0, 1.0)
    lay = P.layout_for(mesh, p)
    rng = np.random.default_rng(0)
    u = rng.standard_normal(lay.shape)
    nu = 1 + 0.5 * rng.random(lay.shape)
    B = P.DiffusionOperator(P.gll_basis(p), mesh, nu)
    got = B.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    want = O.Diffusion(O.gll(p), n, n, 1.0 / n, 1.0 / n, nu).apply(u)
    print(f"n={n} p={p}: maxrel {np.abs(got - want).max() / np.abs(want).max():.2e}", flush=True)

# Poisson (opd_kernel at p = 32, op/opw kernels elsewhere) vs the oracle
for n, p in [(2, 32), (4, 32), (3, 32), (4, 16), (4, 8)]:
    mesh = P.MeshConfig(n, n + 1, 1.0, 1.3)
    lay = P.layout_for(mesh, p)
    u = np.random.default_rng(1).standard_normal(lay.shape)
    A = P.PoissonOperator(P.gll_basis(p), mesh)
    got = A.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    want = O.Poisson(O.gll(p), n, n + 1, 1.0 / n, 1.3 / (n + 1)).apply(u)
    print(f"poisson {n}x{n + 1} p={p}: maxrel {np.abs(got - want).max() / np.abs(want).max():.2e}", flush=True)

# fused residual + restriction (rr_kernel) vs residual + restriction launches
from paper_1512_02390_b200 import _native as NV  # noqa: E402
lib = NV.lib()
st = NV.stream()
for nx, p, orders in [(4, 8, (1, 2, 4, 8)), (8, 8, (1, 2, 4, 8)), (16, 24, (1, 3, 6, 12, 24)), (8, 4, (1, 2, 4))]:
    h = P.build_hierarchy(P.MeshConfig(nx, nx, 1.0, 1.0), p, P.OverlapRule("fixed", 1), nu_hat=0.5, orders=orders)
    rng = np.random.default_rng(3)
    for l in range(h.depth, 0, -1):
        lv = h.levels[l]
        u = torch.from_numpy(rng.standard_normal(lv.op.layout.shape)).cuda()
        f = torch.from_numpy(rng.standard_normal(lv.op.layout.shape)).cuda()
        fc1 = torch.empty_like(h.levels[l - 1].f)
        fc2 = torch.empty_like(h.levels[l - 1].f)
        work = torch.empty_like(u)
        NV.check(lib.smg_residual_restrict(lv.transfer.handle.raw, lv.op._handle.raw, NV.ptr(u), NV.ptr(f),
                                           NV.ptr(fc1), NV.ptr(work), st), "rr")
        NV.check(lib.smg_op_residual(lv.op._handle.raw, NV.ptr(u), NV.ptr(f), NV.ptr(work), st), "res")
        NV.check(lib.smg_restrict(lv.transfer.handle.raw, NV.ptr(work), NV.ptr(fc2), st), "restrict")
        torch.cuda.synchronize()
        print(f"rr n={nx} p_f={lv.basis.p}: max |fused - two-launch| {float((fc1 - fc2).abs().max()):.2e}", flush=True)
