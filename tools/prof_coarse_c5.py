"""One coarse PCG solve of C5's p = 1 level (512^2, nu_hat = 0.9) for an ncu launch list."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402

n = int(os.environ.get("N", "512"))
h = P.build_hierarchy(P.MeshConfig(n, n, 1.0, 1.0), 3, P.OverlapRule("fixed", 1), orders=(1, 3), nu_hat=0.9, nu_shift=0.0)
f = np.random.default_rng(0).standard_normal((n, n))
f -= f.mean()
for _ in range(int(os.environ.get("REPS", "2"))):
    P.coarse_solve(h, f)
torch.cuda.synchronize()
print("ok")
