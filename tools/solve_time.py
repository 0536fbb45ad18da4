import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1512_02390_b200 as P
from paper_1512_02390_b200 import _native as N
for name, n, p, lx, solver in [("c3", 128, 32, 1.0, "mg"), ("c2", 64, 16, 1.0, "mg"), ("c4", 256, 16, 8.0, "mgcg")]:
    mesh = P.MeshConfig(n, n, lx, 1.0)
    h = P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1))
    f = P.project_mean(np.random.default_rng(0).standard_normal(h.top.op.layout.shape))
    fd = torch.from_numpy(np.asarray(f)).cuda() if not isinstance(f, torch.Tensor) else f
    cfg = P.SolveConfig(solver=solver)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        u, rep_ = P.solve(h, fd, cfg, u0=torch.zeros_like(fd))
        torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"{name}: {rep_.cycles} cycles, {1e3*(t1-t0):.2f} ms, {1e6*(t1-t0)/rep_.cycles:.0f} us per cycle", flush=True)
    # residual with norm vs without
    op = h.top.op
    u = torch.randn_like(fd); r = torch.empty_like(fd); nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
    for fn, tag in ((lambda: op.residual_into(u, fd, r, norm2=nrm), "residual+norm"), (lambda: op.residual_into(u, fd, r), "residual")):
        for _ in range(3): fn()
        torch.cuda.synchronize(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): fn()
        b.record(); torch.cuda.synchronize()
        print(f"   {tag}: {a.elapsed_time(b)*100:.1f} us")
