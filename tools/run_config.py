"""Run one BASELINE config end to end on the GPU and print cycles, rates and timings.

    python tools/run_config.py c5 [--solver mgcg] [--cycles N]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200.multigrid import _v_cycle  # noqa: E402

CONFIGS = {
    "c1": dict(n=8, l=(1.0, 1.0), p=8, orders=None, nu_hat=None, solver="mg"),
    "c2": dict(n=64, l=(1.0, 1.0), p=16, orders=None, nu_hat=None, solver="mg"),
    "c3": dict(n=128, l=(1.0, 1.0), p=32, orders=None, nu_hat=None, solver="mg"),
    "c4": dict(n=256, l=(8.0, 1.0), p=16, orders=None, nu_hat=None, solver="mgcg"),
    "c5": dict(n=512, l=(1.0, 1.0), p=24, orders=(1, 3, 6, 12, 24), nu_hat=0.9, solver="mgcg"),
}

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--solver", default=None)
ap.add_argument("--cycles", type=int, default=200)
a = ap.parse_args()
c = CONFIGS[a.config]
t0 = time.perf_counter()
mesh = P.MeshConfig(c["n"], c["n"], *c["l"])
h = P.build_hierarchy(mesh, c["p"], P.OverlapRule("fixed", 1), orders=c["orders"], nu_hat=c["nu_hat"], nu_shift=0.0)
t_build = time.perf_counter() - t0
shape = h.top.op.layout.shape
f = P.project_mean(np.random.default_rng(0).standard_normal(shape))
fd = torch.from_numpy(f).cuda()
# one timed V-cycle from zero (after a warm-up)
u = torch.zeros_like(fd)
_v_cycle(h, u, fd)
torch.cuda.synchronize()
a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a0.record()
_v_cycle(h, u, fd)
b0.record()
torch.cuda.synchronize()
t_vc = a0.elapsed_time(b0) / 1e3
solver = a.solver or c["solver"]
t1 = time.perf_counter()
u, rep = P.solve(h, f, P.SolveConfig(solver=solver, max_cycles=a.cycles), u0=np.zeros_like(f))
torch.cuda.synchronize()
t_solve = time.perf_counter() - t1
# again: the first solve captured the cycle graphs (krylov.py), the second replays them
t1 = time.perf_counter()
u, rep = P.solve(h, f, P.SolveConfig(solver=solver, max_cycles=a.cycles), u0=np.zeros_like(f))
torch.cuda.synchronize()
t_solve2 = time.perf_counter() - t1
res = np.asarray(rep.residuals)
out = {"config": a.config, "dofs": int(np.prod(shape)), "solver": solver, "cycles": rep.cycles,
       "converged": rep.converged, "rbar": rep.rbar, "rates": np.round(np.log10(res[:-1] / res[1:]), 4).tolist(),
       "build_s": round(t_build, 2), "vcycle_ms": round(1e3 * t_vc, 3), "vcycle_gdofs": np.prod(shape) / t_vc / 1e9,
       "solve_s_first": round(t_solve, 3), "solve_s": round(t_solve2, 3), "coarse": h.coarse,
       "coarse_iters_max": max(h.coarse_iterations) if h.coarse_iterations else None,
       "mem_gb": torch.cuda.max_memory_allocated() / 1e9}
print(json.dumps(out))
