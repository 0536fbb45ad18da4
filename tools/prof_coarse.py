import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1512_02390_b200 as P
h = P.build_hierarchy(P.MeshConfig(64, 64, 1.0, 1.0), 2, P.OverlapRule("fixed", 1))
f = np.random.default_rng(0).standard_normal((64, 64)); f -= f.mean()
for _ in range(3):
    P.coarse_solve(h, f)
torch.cuda.synchronize(); print("ok")
