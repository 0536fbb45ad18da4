"""C2 V-cycle time (graph replay, L2 flushed, CUDA events) -- quick tuning probe."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200.multigrid import _v_cycle  # noqa: E402

n, p = int(os.environ.get("N", "64")), int(os.environ.get("PP", "16"))
h = P.build_hierarchy(P.MeshConfig(n, n, 1.0, 1.0), p, P.OverlapRule("fixed", 1))
f = torch.randn(h.top.op.layout.shape, dtype=torch.float64, device="cuda")
f -= f.mean()
u = torch.zeros_like(f)
_v_cycle(h, u, f)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    _v_cycle(h, u, f)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    _v_cycle(h, u, f)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ts = []
for i in range(60):
    flush.fill_(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    ts.append((a, b))
torch.cuda.synchronize()
t = sorted(x.elapsed_time(y) for x, y in ts[10:])
print(f"{os.environ.get('TAG', '')} vcycle median {1e3 * t[len(t) // 2]:.1f} us  min {1e3 * t[0]:.1f}")
