"""Cooperative coarse PCG (pcg_coop_kernel) against the launch-per-step loop (SMG_PCG_COOP=0, read once
per process: run in a child) on p = 1 diffusion problems of 128^2, 256^2 and 512^2 nodes, also a
non-square one.  GPU.  python tools/pcg_coop_check.py"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CASES = [(128, 128, 0.9), (256, 256, 0.5), (512, 512, 0.9), (256, 128, 0.7)]


def solve_all():
    import paper_1512_02390_b200 as P
    out = []
    for nx, ny, nh in CASES:
        h = P.build_hierarchy(P.MeshConfig(nx, ny, 1.0, 1.0), 3, P.OverlapRule("fixed", 1), orders=(1, 3), nu_hat=nh,
                              nu_shift=0.0)
        f = np.random.default_rng(nx + ny).standard_normal((ny, nx))
        f -= f.mean()
        u = P.coarse_solve(h, f)
        u = u.cpu().numpy() if hasattr(u, "cpu") else np.asarray(u)
        out.append((u, int(h.coarse_iterations[-1])))
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1:
        res = solve_all()
        np.savez(sys.argv[1], **{f"u{i}": r[0] for i, r in enumerate(res)}, it=np.array([r[1] for r in res]))
        sys.exit(0)
    tmp = "/tmp/pcg_ref.npz"
    env = dict(os.environ, SMG_PCG_COOP="0")
    subprocess.run([sys.executable, __file__, tmp], check=True, env=env)
    ref = np.load(tmp)
    got = solve_all()
    worst = 0.0
    for i, ((nx, ny, nh), (u, it)) in enumerate(zip(CASES, got)):
        d = np.abs(u - ref[f"u{i}"]).max() / np.abs(ref[f"u{i}"]).max()
        worst = max(worst, d)
        print(f"{nx}x{ny} nu_hat {nh}: iterations {it} (loop {int(ref['it'][i])}), max rel diff {d:.2e}")
        assert it == int(ref["it"][i])
    print("worst", worst)
    sys.exit(0 if worst < 1e-9 else 1)
