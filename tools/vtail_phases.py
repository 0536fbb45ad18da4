"""Per-phase durations of the V-cycle tail kernel (globaltimer, CTA 0) at C2."""
import ctypes as C
import os
import sys

os.environ["SMG_VTAIL_PROF"] = "1"
os.environ.setdefault("SMG_VTAIL", "1")
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02390_b200 as P  # noqa: E402
from paper_1512_02390_b200 import _native as N  # noqa: E402
from paper_1512_02390_b200.multigrid import _v_cycle  # noqa: E402

n, p = int(os.environ.get("N", "64")), int(os.environ.get("PP", "16"))
h = P.build_hierarchy(P.MeshConfig(n, n, 1.0, 1.0), p, P.OverlapRule("fixed", 1))
f = torch.randn(h.top.op.layout.shape, dtype=torch.float64, device="cuda")
u = torch.zeros_like(f)
for _ in range(5):
    _v_cycle(h, u, f)
torch.cuda.synchronize()
K = h.tail_levels
names = ["start"]
for l in range(K, 0, -1):
    names += [f"A{l}(p={h.levels[l].basis.p})", f"BC{l}"]
names += ["D(pinv1)", "EF(pinv2+prolong)"]
acc = {nm: [] for nm in names[1:]}
for _ in range(20):
    _v_cycle(h, u, f)
    torch.cuda.synchronize()
    buf = (C.c_int64 * len(names))()
    N.check(N.lib().smg_vtail_profile(h._tail.raw, buf, len(names)))
    for i in range(1, len(names)):
        acc[names[i]].append((buf[i] - buf[i - 1]) / 1e3)
sub = {}
for _ in range(5):
    _v_cycle(h, u, f)
    torch.cuda.synchronize()
    buf = (C.c_int64 * 30)()
    N.check(N.lib().smg_vtail_profile(h._tail.raw, buf, 30))
    base = buf[len(names) - 2]
    for i in list(range(16, 18)) + list(range(22, 22 + 2 * K)):
        sub.setdefault(i, []).append((buf[i] - base) / 1e3)
bc = {}
for _ in range(5):
    _v_cycle(h, u, f)
    torch.cuda.synchronize()
    buf = (C.c_int64 * 64)()
    N.check(N.lib().smg_vtail_profile(h._tail.raw, buf, 64))
    for lv in range(3):
        b0 = 40 + 8 * lv
        bc.setdefault(lv, []).append([round((buf[b0 + i] - buf[b0]) / 1e3, 2) for i in range(7)])
for lv, v in bc.items():
    print("BC sub-marks p=", [8, 4, 2][lv], v[2], "(tables, f, gather, residual, xpass, ypass, end)")
print("EF sub-marks (us after the D barrier):", {k: round(sorted(v)[2], 2) for k, v in sub.items()})
tot = 0
for nm, v in acc.items():
    v.sort()
    tot += v[len(v) // 2]
    print(f"{nm:22s} {v[len(v) // 2]:8.2f} us")
print(f"tail total (median phases) {tot:.2f} us, K={K}")
