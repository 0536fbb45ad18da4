"""Run a few eager C2 V-cycles (for ncu launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200.multigrid import _v_cycle  # noqa: E402

n, p = int(os.environ.get("N", "64")), int(os.environ.get("PP", "16"))
mesh = P.MeshConfig(n, n, 1.0, 1.0)
h = P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1))
f = torch.randn(h.top.op.layout.shape, dtype=torch.float64, device="cuda")
f -= f.mean()
u = torch.zeros_like(f)
for _ in range(int(os.environ.get("REPS", "3"))):
    _v_cycle(h, u, f)
torch.cuda.synchronize()
print("ok")
