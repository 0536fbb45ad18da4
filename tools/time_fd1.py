"""Time one Schwarz correction for (n, p) from argv (CUDA events, L2 flushed)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402

flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
n, p = int(sys.argv[1]), int(sys.argv[2])
mesh = P.MeshConfig(n, n, 1.0, 1.0)
lay = P.layout_for(mesh, p)
sm = P.AdditiveSchwarz(P.gll_basis(p), lay, mesh.dx, mesh.dy, 1, P.WeightKind.QUINTIC)
r = torch.randn(lay.shape, dtype=torch.float64, device="cuda")
u = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
sm.correct(r, u)
ts = []
for _ in range(10):
    flush.fill_(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sm.correct(r, u)
    b.record()
    ts.append((a, b))
torch.cuda.synchronize()
t = sorted(x.elapsed_time(y) for x, y in ts)[5] * 1e3
print(f"{os.environ.get('TAG', '')} n={n} p={p}: {t:8.1f} us  {lay.size / t / 1e3:7.2f} GDOF/s")
