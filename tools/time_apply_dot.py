"""q = A p with p.q (smg_op_apply_dot) at C5's top level (512^2 elements, p = 24, variable nu): us per call.
SMG_OPDH_DOT=0 selects apply + separate dot pass.  GPU."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as N  # noqa: E402

n = int(os.environ.get("N", "512"))
p = int(os.environ.get("P", "24"))
mesh = P.MeshConfig(n, n, 1.0, 1.0)
b = P.gll_basis(p)
lay = P.layout_for(mesh, p)
g = torch.Generator(device="cuda").manual_seed(1)
nu = 1.0 + 0.5 * torch.rand(lay.shape, dtype=torch.float64, device="cuda", generator=g)
op = P.DiffusionOperator(b, mesh, nu)
u = torch.randn(lay.shape, dtype=torch.float64, device="cuda", generator=g)
q = torch.empty_like(u)
d = torch.zeros(1, dtype=torch.float64, device="cuda")
lib = N.lib()


def call():
    N.check(lib.smg_op_apply_dot(op._handle.raw, N.ptr(u), N.ptr(q), N.ptr(d), N.ptr(op.partials), op.ring_ptr(),
                                 N.stream()), "apply_dot")


for _ in range(3):
    call()
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
a.record()
for _ in range(reps):
    call()
e.record()
torch.cuda.synchronize()
want = float((u * op.apply(u)).sum().item())
print(f"apply_dot {n}^2 p={p}: {1e3 * a.elapsed_time(e) / reps:.1f} us per call; p.q {d.item():.15e} vs {want:.15e}")
