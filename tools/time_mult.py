"""Multiplicative sweep time on the device vs the reference-algorithm oracle
on the host (one sweep; 16x16 and 64x64 elements, p = 8 / 16)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from oracle import smg_oracle as O  # noqa: E402

for n, p in [(16, 8), (64, 16)]:
    mesh = P.MeshConfig(n, n, 1.0, 1.0)
    b = P.gll_basis(p)
    lay = P.layout_for(mesh, p)
    op = P.PoissonOperator(b, mesh)
    sm = P.MultiplicativeSchwarz(b, lay, mesh.dx, mesh.dy, 1)
    f = torch.randn(lay.shape, dtype=torch.float64, device="cuda")
    u = torch.zeros_like(f)
    sm.smooth(op, u, f, 1)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sm.smooth(op, u, f, 2)
    e.record()
    torch.cuda.synchronize()
    t_gpu = a.elapsed_time(e) / 2e3
    ob = O.gll(p)
    osm = O.MultSweep(ob, n, n, mesh.dx, mesh.dy, 1)
    oop = O.Poisson(ob, n, n, mesh.dx, mesh.dy)
    ff = f.cpu().numpy()
    uu = np.zeros_like(ff)
    t0 = time.perf_counter()
    if n <= 16:
        osm.smooth(oop, uu, ff, 1)
        t_cpu = time.perf_counter() - t0
    else:
        # a bounded sample: the first 256 subdomains, scaled
        r = ff - oop.apply(uu)
        order = [(x, y) for y in range(n) for x in range(n)][:256]
        for ex, ey in order:
            win = np.ix_(osm.wy[ey], osm.wx[ex])
            du = osm.fd.solve(r[win])
            uu[win] += du
            osm._local_update(oop, r, du, ex, ey)
        t_cpu = (time.perf_counter() - t0) * (n * n / 256)
    print(f"{n}x{n} p={p}: GPU {1e3 * t_gpu:.2f} ms/sweep ({1e6 * t_gpu / (n * n):.2f} us/subdomain), "
          f"CPU oracle {1e3 * t_cpu:.1f} ms/sweep, x{t_cpu / t_gpu:.0f}")
