"""Time one Schwarz correction (CUDA events, L2 flushed before each launch,
median of 21) over (n, p) and contraction engines, with the roofline fraction
max(24 B/DOF / HBM, even/odd flops / FP64 peak) / t.

    SMG_FDT_LC=1|2 ENGINES=dfma,dmma_eo python tools/time_fd_sweep.py [n:p ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402

HBM = 6548.5e9
P64 = 37.15e12
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
cfgs = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or \
    [(256, 8), (256, 12), (256, 16), (256, 24), (256, 32), (128, 32), (64, 16)]
engines = os.environ.get("ENGINES", "dfma").split(",")
tag = os.environ.get("TAG", "lc" + os.environ.get("SMG_FDT_LC", "2"))
NO = int(os.environ.get("NO", "1"))   # overlap layers


def eo_flops_per_dof(p, n_o=1):
    m = p + 1 + 2 * n_o
    he, ho = (m + 1) // 2, m // 2
    return (8 * m * (he * he + ho * ho) + m * m) / (p * p)


for n, p in cfgs:
    mesh = P.MeshConfig(n, n, 1.0, 1.0)
    lay = P.layout_for(mesh, p)
    r = torch.randn(lay.shape, dtype=torch.float64, device="cuda")
    u = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
    t_roof = max(24.0 * lay.size / HBM, eo_flops_per_dof(p, NO) * lay.size / P64) * 1e6
    for eng in engines:
        os.environ["SMG_FD_ENGINE"] = eng
        sm = P.AdditiveSchwarz(P.gll_basis(p), lay, mesh.dx, mesh.dy, NO, P.WeightKind.QUINTIC)
        for _ in range(3):
            sm.correct(r, u)
        ts = []
        for _ in range(21):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sm.correct(r, u)
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        t = sorted(x.elapsed_time(y) for x, y in ts)[10] * 1e3
        print(f"{tag} {eng:8s} {sm.kernel_info()} n_o={NO} n={n:3d} p={p:2d}: {t:8.1f} us  {lay.size / t / 1e3:7.2f} GDOF/s  "
              f"roof {t_roof:7.1f} us  frac {t_roof / t:.3f}", flush=True)
