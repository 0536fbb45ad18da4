"""Time the p = 1 coarse plain CG (parity mode) on the C1/C2 coarse meshes:
CUDA events around P.coarse_solve's device work, SMG_CCG_CTA selects the path."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402

for nx in (8, 32, 64):
    h = P.build_hierarchy(P.MeshConfig(nx, nx, 1.0, 1.0), 2, P.OverlapRule("fixed", 1), coarse="cg")
    f0 = torch.from_numpy(np.random.default_rng(nx).standard_normal((nx, nx))).cuda()
    for _ in range(3):
        P.coarse_solve(h, f0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 20
    for _ in range(n):
        P.coarse_solve(h, f0)
    b.record()
    torch.cuda.synchronize()
    print(f"cta={os.environ.get('SMG_CCG_CTA', '1')} {nx}x{nx}: {a.elapsed_time(b) / n * 1e3:.1f} us/solve, "
          f"{h.coarse_iterations[-1]} iterations")
