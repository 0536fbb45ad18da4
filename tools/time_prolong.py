"""Time the top-level prolongation u_f += P u_c (CUDA events, L2 flushed, median of 21) with
the tiled / warp kernels (SMG_PRW=0) and the warp-per-fine-element kernel (SMG_PRW=2), and
check the two against each other.    python tools/time_prolong.py [n:p ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
HBM = 6548.5e9
cfgs = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(128, 32), (256, 24), (256, 16), (64, 16)]
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as N  # noqa: E402

flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for n, p in cfgs:
    mesh = P.MeshConfig(n, n, 1.0, 1.0)
    orders = None if p & (p - 1) == 0 else tuple(sorted({1} | {p // (2 ** k) for k in range(6) if p % (2 ** k) == 0}))
    outs = {}
    for mode in ("0", "2"):
        os.environ["SMG_PRW"] = mode
        h = P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1), orders=orders) if orders else \
            P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1))
        lv = h.top
        torch.manual_seed(0)
        uc = torch.randn(h.levels[-2].op.layout.shape, dtype=torch.float64, device="cuda")
        u0 = torch.randn(lv.op.layout.shape, dtype=torch.float64, device="cuda")
        uf = u0.clone()
        call = lambda: N.check(N.lib().smg_prolongate(lv.transfer.handle.raw, N.ptr(uc), N.ptr(uf), 1, N.stream()), "p")  # noqa: E731
        call()
        outs[mode] = (uf - u0).clone()
        ts = []
        for _ in range(21):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        t = sorted(x.elapsed_time(y) for x, y in ts)[10] * 1e3
        byt = 8.0 * lv.op.layout.size * 2.25
        print(f"SMG_PRW={mode} n={n} p={p}: {t:8.1f} us  roof {byt / HBM * 1e6:6.1f} us  frac {byt / HBM * 1e6 / t:.3f}", flush=True)
        del h
    d = (outs["2"] - outs["0"]).abs().max().item() / outs["0"].abs().max().item()
    print(f"   warp-per-fine-element vs tiled: max rel {d:.2e}")
