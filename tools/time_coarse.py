"""Per-launch timing of the coarse-level pieces at C5's p = 1 level (512^2):
pseudo-inverse (FFT), p = 1 diffusion residual, one dot, and one whole
coarse PCG solve.  CUDA events, warm.  GPU."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as N  # noqa: E402
from paper_1512_02390_b200.multigrid import _coarse_into  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
mesh = P.MeshConfig(n, n, 1.0, 1.0)
h = P.build_hierarchy(mesh, 3, P.OverlapRule("fixed", 1), orders=(1, 3), nu_hat=0.9, nu_shift=0.0)
lib = N.lib()
st = N.stream()
f0, u0 = h.levels[0].f, h.levels[0].u
f0.normal_()
f0 -= f0.mean()
w = torch.empty_like(f0)


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


t_p = timeit(lambda: N.check(lib.smg_coarse_pinv(h._pinv.handle.raw, N.ptr(f0), N.ptr(u0), N.ptr(h._pinv.ws), st)))
t_r = timeit(lambda: N.check(lib.smg_op_residual(h.levels[0].op._handle.raw, N.ptr(u0), N.ptr(f0), N.ptr(w), st)))
t_s = timeit(lambda: _coarse_into(h, f0, u0), reps=10)
print(f"n={n}: pinv {t_p:.1f} us, p=1 residual {t_r:.1f} us, PCG solve {t_s:.1f} us "
      f"({h.coarse_iterations[-1]} iterations, {t_s / max(1, h.coarse_iterations[-1]):.1f} us each)")
