import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_1512_02390_b200 as P
import test_gpu_parity as T
if len(sys.argv) > 1:
    T.test_operators_vs_reference(None)
    print("ops done", flush=True)
g = T.golden("multigrid")
for i, (nx, ny, lx, ly) in enumerate([(4, 4, 2.0, 2.0), (8, 8, 1.0, 1.0), (16, 8, 8.0, 1.0)]):
    mesh = P.MeshConfig(nx, ny, lx, ly)
    hp = P.build_hierarchy(mesh, 2, P.OverlapRule("fixed", 1))
    f0 = g[f"cs{i}_f0"]
    print(i, f0.shape, f0.dtype, f0.flags['C_CONTIGUOUS'], flush=True)
    try:
        got = P.coarse_solve(hp, f0); torch.cuda.synchronize()
        print(i, "ok", float(got.abs().max()), flush=True)
    except Exception as e:
        print(i, "ERR", repr(e)[:200], flush=True); break
