"""Paired-line Schwarz engine (SMG_FD_ENGINE=pair) against the default tiled
engine and the oracle: max-relative differences of one correction.  GPU.

    python tools/pair_check.py [p ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from oracle import smg_oracle as O  # noqa: E402

ps = [int(a) for a in sys.argv[1:]] or [16]
worst = 0.0
for p in ps:
    for (nx, ny, lx, ly, no, nu) in [(4, 4, 1.0, 1.0, 1, False), (8, 4, 1.0, 1.0, 1, False), (12, 8, 1.0, 2.0, 1, True),
                                     (16, 16, 8.0, 1.0, 1, False), (8, 8, 1.0, 1.0, 2, True)]:
        mesh = P.MeshConfig(nx, ny, lx, ly)
        lay = P.layout_for(mesh, p)
        rng = np.random.default_rng(7)
        r = rng.standard_normal(lay.shape)
        u0 = rng.standard_normal(lay.shape)
        nub = 0.5 + rng.random((ny, nx)) if nu else None
        outs = {}
        for eng in ("dfma", "pair"):
            os.environ["SMG_FD_ENGINE"] = eng
            sm = P.AdditiveSchwarz(P.gll_basis(p), lay, mesh.dx, mesh.dy, no, P.WeightKind.QUINTIC, nu_bar=nub)
            u = torch.from_numpy(u0).cuda()
            sm.correct(torch.from_numpy(r).cuda(), u)
            torch.cuda.synchronize()
            outs[eng] = u.cpu().numpy() - u0
        ref = O.AdditiveSweep(O.gll(p), nx, ny, mesh.dx, mesh.dy, no, "w5", nu_bar=nub).correction(r)
        sc = np.abs(ref).max()
        e1 = np.abs(outs["pair"] - outs["dfma"]).max() / sc
        e2 = np.abs(outs["pair"] - ref).max() / sc
        worst = max(worst, e1, e2)
        print(f"p={p} {nx}x{ny} n_o={no} nu={nu}: pair vs dfma {e1:.2e}  pair vs oracle {e2:.2e}", flush=True)
print("worst", worst)
sys.exit(0 if worst < 1e-11 else 1)
