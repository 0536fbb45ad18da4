"""Per-phase cycle breakdown of the tiled Schwarz kernel (thread 0 of every
CTA, clock64 at each phase boundary, SMG_FDT_PHASES=1).  Cycles per tile per
CTA; with R CTAs resident per SM the SM finishes a tile every total/R cycles.

    python tools/fdt_phases.py [n:p ...]
"""
import ctypes as C
import os
import sys

os.environ["SMG_FDT_PHASES"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as NV  # noqa: E402

NAMES = ["tiles", "wait_r", "stage1", "stage2", "stage3", "stage4", "fold", "wait_u", "gather+ring", "issue"]
cfgs = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(256, 16), (256, 24), (256, 32)]
lib = NV.lib()
buf = (C.c_ulonglong * 10)()
for n, p in cfgs:
    mesh = P.MeshConfig(n, n, 1.0, 1.0)
    lay = P.layout_for(mesh, p)
    sm = P.AdditiveSchwarz(P.gll_basis(p), lay, mesh.dx, mesh.dy, 1, P.WeightKind.QUINTIC)
    r = torch.randn(lay.shape, dtype=torch.float64, device="cuda")
    u = torch.randn(lay.shape, dtype=torch.float64, device="cuda")
    sm.correct(r, u)
    torch.cuda.synchronize()
    lib.smg_debug_fdt_phases(buf, 10)
    reps = 5
    for _ in range(reps):
        sm.correct(r, u)
    torch.cuda.synchronize()
    assert lib.smg_debug_fdt_phases(buf, 10) == 0
    tiles = buf[0]
    tot = sum(buf[1:10])
    print(f"n={n} p={p} ({os.environ.get('SMG_FD_ENGINE', 'default')}): {tiles // reps} tiles per call, "
          f"{tot / tiles:.0f} cycles per tile per CTA")
    for k in range(1, 10):
        print(f"   {NAMES[k]:12s} {buf[k] / tiles:8.0f}  {100.0 * buf[k] / tot:5.1f}%")
