"""Warm per-component timing of one BASELINE config's V-cycle (C2..C5): per
level the residual, Schwarz correction, restriction, prolongation and fused
residual+restriction, the coarse solve, and the whole V-cycle (CUDA events).

    python tools/vcycle_breakdown_cfg.py c5
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as N  # noqa: E402
from paper_1512_02390_b200.multigrid import _coarse_into, _v_cycle  # noqa: E402

CONFIGS = {
    "c2": dict(n=64, l=(1.0, 1.0), p=16, orders=None, nu_hat=None),
    "c3": dict(n=128, l=(1.0, 1.0), p=32, orders=None, nu_hat=None),
    "c4": dict(n=256, l=(8.0, 1.0), p=16, orders=None, nu_hat=None),
    "c5": dict(n=512, l=(1.0, 1.0), p=24, orders=(1, 3, 6, 12, 24), nu_hat=0.9),
}
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
mesh = P.MeshConfig(c["n"], c["n"], *c["l"])
h = P.build_hierarchy(mesh, c["p"], P.OverlapRule("fixed", 1), orders=c["orders"], nu_hat=c["nu_hat"], nu_shift=0.0)
lib = N.lib()


def timeit(fn, reps=20):
    for _ in range(3):
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
st = N.stream()
for l in range(h.depth, 0, -1):
    lv = h.levels[l]
    lv.u.normal_()
    lv.f.normal_()
    fc = h.levels[l - 1].f
    uc = h.levels[l - 1].u
    t_res = timeit(lambda: N.check(lib.smg_op_residual_ws(lv.op._handle.raw, N.ptr(lv.u), N.ptr(lv.f), N.ptr(lv.work), lv.op.ring_ptr(), st)))
    t_fd = timeit(lambda: N.check(lib.smg_schwarz_correct(lv.smoother._h.raw, N.ptr(lv.work), N.ptr(lv.u), N.ptr(lv.smoother.ring), st)))
    t_rs = timeit(lambda: N.check(lib.smg_restrict_ws(lv.transfer.handle.raw, N.ptr(lv.work), N.ptr(fc), lv.transfer.ws_ptr(), st)))
    t_pr = timeit(lambda: N.check(lib.smg_prolongate(lv.transfer.handle.raw, N.ptr(uc), N.ptr(lv.u), 1, st)))
    t_rr = timeit(lambda: N.check(lib.smg_residual_restrict_ws(lv.transfer.handle.raw, lv.op._handle.raw, N.ptr(lv.u),
                                                              N.ptr(lv.f), N.ptr(fc), N.ptr(lv.work),
                                                              lv.transfer.ws_ptr(), lv.op.ring_ptr(), st)))
    rows.append((lv.basis.p, lv.op.layout.size, t_res, t_fd, t_rs, t_pr, t_rr))
    tot += t_res + t_fd + t_rr + t_pr
f0, u0 = h.levels[0].f, h.levels[0].u
f0.normal_()
f0 -= f0.mean()
t_c = timeit(lambda: _coarse_into(h, f0, u0))
tot += t_c
f = torch.from_numpy(P.project_mean(np.random.default_rng(0).standard_normal(h.top.op.layout.shape))).cuda()
u = torch.zeros_like(f)
t_v = timeit(lambda: _v_cycle(h, u, f), reps=5)
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'c5'}: coarse={h.coarse}, levels {[lv.basis.p for lv in h.levels]}")
print(f"{'p':>3} {'DOFs':>11} {'residual':>9} {'schwarz':>9} {'restrict':>9} {'prolong':>9} {'res+restr':>9}   (us, warm)")
for r in rows:
    print(f"{r[0]:3d} {r[1]:11d} {r[2]:9.1f} {r[3]:9.1f} {r[4]:9.1f} {r[5]:9.1f} {r[6]:9.1f}")
print(f"coarse solve {t_c:.1f} us (iterations {h.coarse_iterations[-1] if h.coarse_iterations else '-'})")
print(f"sum of components (smooth = residual + schwarz) = {tot:.1f} us;  V-cycle {t_v:.1f} us")
