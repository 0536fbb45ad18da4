"""Where an MGCG iteration's time goes (C4 by default): the whole solve
(wall, host syncs included) against the V-cycle alone and the BLAS-1 /
operator kernels between V-cycles, each timed with CUDA events (L2 not
flushed: the solver runs them back to back)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as N  # noqa: E402
from paper_1512_02390_b200.multigrid import _v_cycle  # noqa: E402

cfg = os.environ.get("CFG", "c4")
if cfg == "c4":
    mesh, p, kw = P.MeshConfig(256, 256, 8.0, 1.0), 16, {}
elif cfg == "c2":
    mesh, p, kw = P.MeshConfig(64, 64, 1.0, 1.0), 16, {}
else:
    mesh, p, kw = P.MeshConfig(512, 512, 1.0, 1.0), 24, dict(orders=(1, 3, 6, 12, 24), nu_hat=0.9, nu_shift=0.0)
h = P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1), **kw)
shape = h.top.op.layout.shape
f = np.random.default_rng(0).standard_normal(shape)
f -= f.mean()
fd = torch.from_numpy(f).cuda()
u0 = torch.zeros_like(fd)
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    u, rep = P.solve(h, fd, P.SolveConfig(solver="mgcg"), u0=u0)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
print(f"{cfg}: MGCG {rep.cycles} cycles, {wall * 1e3:.1f} ms wall, {wall / max(rep.cycles, 1) * 1e6:.0f} us per cycle")


def ev(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


lib = N.lib()
st = N.stream()
n = fd.numel()
z = torch.zeros_like(fd)
q = torch.empty_like(fd)
r2 = torch.empty_like(fd)
s = torch.zeros(8, dtype=torch.float64, device="cuda")
s[0] = 1.0
s[1] = 1.0
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
ws = h.reduce_ws
pv = torch.randn_like(fd)
uu = torch.zeros_like(fd)
t_v = ev(lambda: _v_cycle(h, z, fd, u_zero=True))
t_op = ev(lambda: h.top.op.residual_into(pv, None, q))
t_dot = ev(lambda: N.check(lib.smg_dot(N.ptr(pv), N.ptr(q), n, N.ptr(s[1:2]), N.ptr(ws), st)))
t_upd = ev(lambda: N.check(lib.smg_cg_update2(N.ptr(uu), N.ptr(fd), N.ptr(r2), N.ptr(pv), N.ptr(q), n, N.ptr(s),
                                              N.ptr(flag), N.ptr(ws), st)))
t_beta = ev(lambda: N.check(lib.smg_dot2(N.ptr(z), N.ptr(r2), N.ptr(fd), n, N.ptr(s[3:5]), N.ptr(ws), st)))
t_dir = ev(lambda: N.check(lib.smg_cg_direction(N.ptr(pv), N.ptr(z), n, N.ptr(s), st)))
HBM = 6548.5e9
for name, t, nb in [("v_cycle", t_v, 0), ("op apply", t_op, 16), ("dot p.q", t_dot, 16), ("cg_update2", t_upd, 48),
                    ("dot2 (beta)", t_beta, 24), ("direction", t_dir, 24)]:
    bw = f"  {nb * n / (t * 1e-6) / 1e9:7.0f} GB/s ({nb * n / (t * 1e-6) / HBM:.0%} of HBM)" if nb else ""
    print(f"  {name:12s} {t:8.1f} us{bw}")
tot = t_v + t_op + t_dot + t_upd + t_beta + t_dir
print(f"  sum of kernels {tot:.1f} us per cycle; host/launch gap {wall / max(rep.cycles, 1) * 1e6 - tot:.0f} us")
