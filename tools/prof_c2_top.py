"""Run each C2 top-level kernel call once (residual, Schwarz correction, residual restricted
in place, stand-alone restriction, prolongation) -- the launches bench.py times -- for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as NV  # noqa: E402

mesh = P.MeshConfig(64, 64, 1.0, 1.0)
h = P.build_hierarchy(mesh, 16, P.OverlapRule("fixed", 1))
lib = NV.lib()
top = h.top
shape = top.op.layout.shape
st = NV.stream()
r = torch.randn(shape, dtype=torch.float64, device="cuda")
u = torch.randn(shape, dtype=torch.float64, device="cuda")
out = torch.empty_like(r)
fc = h.levels[-2].f
uc = torch.randn(fc.shape, dtype=torch.float64, device="cuda")
for _ in range(int(os.environ.get("REPS", "1"))):
    NV.check(lib.smg_op_residual(top.op._handle.raw, NV.ptr(u), NV.ptr(r), NV.ptr(out), st))
    NV.check(lib.smg_schwarz_correct(top.smoother._h.raw, NV.ptr(r), NV.ptr(out), NV.ptr(top.smoother.ring), st))
    NV.check(lib.smg_residual_restrict_ws(top.transfer.handle.raw, top.op._handle.raw, NV.ptr(u), NV.ptr(r), NV.ptr(fc),
                                          NV.ptr(out), top.transfer.ws_ptr(), top.op.ring_ptr(), st))
    NV.check(lib.smg_restrict(top.transfer.handle.raw, NV.ptr(r), NV.ptr(fc), st))
    NV.check(lib.smg_prolongate(top.transfer.handle.raw, NV.ptr(uc), NV.ptr(out), 1, st))
torch.cuda.synchronize()
print("ok")
