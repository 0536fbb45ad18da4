"""One fused residual + restriction call (smg_residual_restrict_ws) at the top level of a Poisson
hierarchy, for ncu.  python tools/prof_rr.py [n] [p]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as N  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p = int(sys.argv[2]) if len(sys.argv) > 2 else 16
h = P.build_hierarchy(P.MeshConfig(n, n, 1.0, 1.0), p, P.OverlapRule("fixed", 1))
lv = h.top
u = torch.randn(lv.op.layout.shape, dtype=torch.float64, device="cuda")
f = torch.randn(lv.op.layout.shape, dtype=torch.float64, device="cuda")
fc = torch.empty(h.levels[-2].op.layout.shape, dtype=torch.float64, device="cuda")
for _ in range(3):
    N.check(N.lib().smg_residual_restrict_ws(lv.transfer.handle.raw, lv.op._handle.raw, N.ptr(u), N.ptr(f), N.ptr(fc),
                                             N.ptr(lv.work), lv.transfer.ws_ptr(), lv.op.ring_ptr(), N.stream()), "rr")
torch.cuda.synchronize()
print("ok")
