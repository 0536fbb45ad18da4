"""Time one operator residual r = f - A u (CUDA events, L2 flushed, median of
21) for (n, p, kind) cases: HBM roofline fraction at the algorithmic bytes
(24 B/DOF Poisson: u, f, r; 32 B/DOF diffusion: + nu).

    python tools/time_op.py [n:p:kind ...]     kind = poisson | diffusion
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402

HBM = 6548.5e9
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
cases = [a.split(":") for a in sys.argv[1:]] or [["512", "24", "diffusion"], ["128", "32", "poisson"],
                                                  ["64", "16", "poisson"], ["256", "16", "poisson"]]
for n, p, kind in cases:
    n, p = int(n), int(p)
    mesh = P.MeshConfig(n, n, 1.0, 1.0)
    b = P.gll_basis(p)
    if kind == "poisson":
        op, nb = P.PoissonOperator(b, mesh), 24.0
    else:
        op, nb = P.DiffusionOperator(b, mesh, P.diffusivity_field_device(mesh, b, 0.9, 0.0)), 32.0
    sh = op.layout.shape
    u = torch.randn(sh, dtype=torch.float64, device="cuda")
    f = torch.randn(sh, dtype=torch.float64, device="cuda")
    r = torch.empty_like(u)
    op.residual_into(u, f, r)
    ts = []
    for _ in range(21):
        flush.fill_(1.0)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        op.residual_into(u, f, r)
        e.record()
        ts.append((a, e))
    torch.cuda.synchronize()
    t = sorted(x.elapsed_time(y) for x, y in ts)[10] * 1e-3
    ndof = sh[0] * sh[1]
    print(f"{os.environ.get('TAG', '')} {kind:9s} n={n:3d} p={p:2d}: {t * 1e6:9.1f} us  {ndof / t / 1e9:6.2f} GDOF/s  "
          f"{nb * ndof / t / 1e9:7.0f} GB/s  frac {nb * ndof / t / HBM:.3f}", flush=True)
