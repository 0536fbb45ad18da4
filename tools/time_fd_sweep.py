"""Time one Schwarz correction at 256x256 elements over p (CUDA events, L2 flushed before each launch).

Used to compare library builds: SMG_LIB=<alternative libsmg*.so> python tools/time_fd_sweep.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402

flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
lib = os.path.basename(os.environ.get("SMG_LIB", "libsmg.so"))
for n, p in [(256, 8), (256, 12), (256, 16), (256, 24), (256, 32), (64, 16)]:
    mesh = P.MeshConfig(n, n, 1.0, 1.0)
    lay = P.layout_for(mesh, p)
    sm = P.AdditiveSchwarz(P.gll_basis(p), lay, mesh.dx, mesh.dy, 1, P.WeightKind.QUINTIC)
    r = torch.randn(lay.shape, dtype=torch.float64, device="cuda")
    u = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
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
    print(f"{lib} n={n} p={p}: {t:8.1f} us  {lay.size / t / 1e3:7.2f} GDOF/s", flush=True)
