"""Time the top-level restriction (CUDA events, L2 flushed, median of 21) with and without
the halo-free kernel (SMG_RW=0|1|2), and check the two against each other.

    python tools/time_restrict.py [n:p ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
HBM = 6548.5e9
cfgs = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(128, 32), (256, 24), (256, 16), (64, 16)]
import paper_1512_02390_b200 as P  # noqa: E402

flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for n, p in cfgs:
    mesh = P.MeshConfig(n, n, 1.0, 1.0)
    orders = None if p & (p - 1) == 0 else tuple(sorted({1} | {p // (2 ** k) for k in range(6) if p % (2 ** k) == 0}))
    outs = {}
    for mode in ("0", "1", "2"):
        os.environ["SMG_RW"] = mode
        h = P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1), orders=orders) if orders else \
            P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1))
        lay = h.top.op.layout
        torch.manual_seed(0)
        r = torch.randn(lay.shape, dtype=torch.float64, device="cuda")
        for _ in range(3):
            out = P.restrict_residual(h, h.depth, r)
        ts = []
        for _ in range(21):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = P.restrict_residual(h, h.depth, r)
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        t = sorted(x.elapsed_time(y) for x, y in ts)[10] * 1e3
        outs[mode] = out.clone()
        byt = 8.0 * lay.size * 1.25
        ws = h.top.transfer.ws
        print(f"SMG_RW={mode} n={n} p={p}: {t:8.1f} us (incl. the output allocation)  roof {byt / HBM * 1e6:6.1f} us  "
              f"frac {byt / HBM * 1e6 / t:.3f}  ring {'-' if ws is None else ws.numel()}", flush=True)
        del h
    d = (outs["2"] - outs["0"]).abs().max().item() / outs["0"].abs().max().item()
    print(f"   halo-free vs tiled: max rel {d:.2e}")
