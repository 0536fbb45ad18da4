"""Warm per-component timing of the C2 V-cycle (each component repeated, CUDA events)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as N  # noqa: E402

n = int(os.environ.get("N", "64"))
p = int(os.environ.get("PP", "16"))
mesh = P.MeshConfig(n, n, 1.0, 1.0)
h = P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1))
lib = N.lib()


def timeit(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


rows = []
tot = 0.0
for l in range(h.depth, 0, -1):
    lv = h.levels[l]
    lv.u.normal_()
    lv.f.normal_()
    st = N.stream()
    t_res = timeit(lambda: N.check(lib.smg_op_residual(lv.op._handle.raw, N.ptr(lv.u), N.ptr(lv.f), N.ptr(lv.work), st)))
    t_fd = timeit(lambda: N.check(lib.smg_schwarz_correct(lv.smoother._h.raw, N.ptr(lv.work), N.ptr(lv.u), N.ptr(lv.smoother.ring), st)))
    fc = h.levels[l - 1].f
    t_rs = timeit(lambda: N.check(lib.smg_restrict(lv.transfer.handle.raw, N.ptr(lv.work), N.ptr(fc), st)))
    uc = h.levels[l - 1].u
    t_pr = timeit(lambda: N.check(lib.smg_prolongate(lv.transfer.handle.raw, N.ptr(uc), N.ptr(lv.u), 1, st)))
    t_rr = timeit(lambda: N.check(lib.smg_residual_restrict(lv.transfer.handle.raw, lv.op._handle.raw, N.ptr(lv.u),
                                                           N.ptr(lv.f), N.ptr(fc), N.ptr(lv.work), st)))
    n_res = 2 if l == h.depth else 1
    rows.append((lv.basis.p, t_res, t_fd, t_rs, t_pr, t_rr))
    tot += n_res * t_res + t_fd + t_rs + t_pr
f0, u0 = h.levels[0].f, h.levels[0].u
t_c = timeit(lambda: N.check(lib.smg_coarse_pinv(h._pinv.handle.raw, N.ptr(f0), N.ptr(u0), N.ptr(h._pinv.ws), N.stream())))
tot += t_c
print(f"{'p':>3} {'residual':>9} {'schwarz':>9} {'restrict':>9} {'prolong':>9} {'res+restr':>9}   (us, warm, back-to-back)")
for r in rows:
    print(f"{r[0]:3d} {r[1]:9.2f} {r[2]:9.2f} {r[3]:9.2f} {r[4]:9.2f} {r[5]:9.2f}")
print(f"coarse pinv {t_c:.2f} us;  sum of components (top residual x2) = {tot:.1f} us")
