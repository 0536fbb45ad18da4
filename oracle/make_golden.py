"""Generate the golden fixtures in ``tests/golden/`` by running the UNMODIFIED
reference package (``/root/reference/pkg/src/schwarzmg``) in this container.

TEST INFRASTRUCTURE ONLY.  The GPU box has no ``/root/reference``; the
committed ``.npz`` files are what travels.  Re-run with

    python oracle/make_golden.py            # small fixtures (~1 min)
    python oracle/make_golden.py --large    # + BASELINE-size histories (slow)

Every fixture is produced by a reference call (named in the key comments), on
seeded inputs, so the oracle restatement in ``oracle/smg_oracle.py`` and the
CUDA path can both be checked against the reference's own numbers.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import schwarzmg  # noqa: F401
    from schwarzmg import basis, krylov, mesh, multigrid, operators, schwarz
    return basis, krylov, mesh, multigrid, operators, schwarz


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


# FD-factor cases: (p, n_o, dx, dy).  Includes every BASELINE top level at
# fixed:1 and ceilp8, and the smoother-microbenchmark orders.
FD_CASES = [
    (2, 1, 0.25, 0.25), (4, 1, 0.5, 0.5), (4, 1, 1.0, 0.25), (8, 2, 0.25, 0.25),
    (8, 1, 1 / 8, 1 / 8), (4, 1, 1 / 64, 1 / 64), (8, 1, 1 / 64, 1 / 64),
    (12, 1, 1 / 64, 1 / 64), (16, 1, 1 / 64, 1 / 64), (24, 1, 1 / 64, 1 / 64),
    (32, 1, 1 / 64, 1 / 64), (16, 2, 1 / 64, 1 / 64), (32, 1, 1 / 128, 1 / 128),
    (32, 4, 1 / 128, 1 / 128), (16, 1, 1 / 32, 1 / 256), (16, 2, 1 / 32, 1 / 256),
    (24, 1, 1 / 512, 1 / 512), (24, 3, 1 / 512, 1 / 512), (12, 1, 1 / 512, 1 / 512),
    (6, 1, 1 / 512, 1 / 512), (3, 1, 1 / 512, 1 / 512), (2, 1, 1 / 64, 1 / 64),
]


def small():
    basis, krylov, mesh, multigrid, operators, schwarz = _ref()
    rng = np.random.default_rng(20240601)

    # -- basis.py: gll_basis, interp_matrix
    out = {}
    for p in [1, 2, 3, 4, 5, 6, 8, 12, 16, 24, 32]:
        b = basis.gll_basis(p)
        out[f"nodes_{p}"] = b.nodes
        out[f"weights_{p}"] = b.weights
        out[f"diff_{p}"] = b.diff
        out[f"stiff_{p}"] = b.stiff
    for pc, pf in [(1, 2), (2, 4), (4, 8), (8, 16), (16, 32), (1, 3), (3, 6), (6, 12), (12, 24)]:
        out[f"J_{pc}_{pf}"] = basis.interp_matrix(basis.gll_basis(pc), basis.gll_basis(pf)).matrix
    save("basis", **out)

    # -- schwarz.py: weights, restricted_1d, jacobi-based FD factors
    out = {}
    for kind in schwarz.WeightKind:
        for p, n_o in [(2, 1), (4, 1), (8, 1), (8, 2), (16, 1), (16, 2), (24, 1), (24, 3), (32, 1), (32, 4)]:
            b = basis.gll_basis(p)
            g = schwarz.subdomain_geometry(b, n_o)
            out[f"w_{kind.value}_{p}_{n_o}"] = schwarz.build_weight_1d(kind, b, g)
    for i, (p, n_o, dx, dy) in enumerate(FD_CASES):
        b = basis.gll_basis(p)
        L, m = schwarz.restricted_1d(b, dx, n_o)
        fd = schwarz.build_fast_diag(b, dx, dy, n_o, schwarz.WeightKind.QUINTIC)
        out[f"fd{i}_case"] = np.array([p, n_o, dx, dy])
        out[f"fd{i}_L"] = L
        out[f"fd{i}_m"] = m
        out[f"fd{i}_Sx"] = fd.S_x
        out[f"fd{i}_Sy"] = fd.S_y
        out[f"fd{i}_lx"] = fd.lam_x
        out[f"fd{i}_ly"] = fd.lam_y
        out[f"fd{i}_W"] = fd.weight
        r = rng.standard_normal((3, 2, fd.S_x.shape[0], fd.S_x.shape[0]))
        out[f"fd{i}_r"] = r
        out[f"fd{i}_solve"] = fd.solve(r)
    out["n_fd"] = np.array(len(FD_CASES))
    save("schwarz_setup", **out)

    # -- operators.py: Poisson / diffusion apply, element_mean_nu
    out = {}
    cases = [(2, 2, 2.0, 2.0, 1), (3, 2, 3.0, 2.0, 2), (3, 2, 3.0, 2.0, 3), (5, 4, 1.0, 1.0, 4),
             (4, 6, 8.0, 1.0, 8), (3, 3, 1.0, 1.0, 16), (2, 3, 1.0, 1.0, 32), (4, 3, 2.0, 1.0, 12),
             (3, 4, 1.0, 1.0, 24), (4, 4, 1.0, 1.0, 6)]
    for i, (nx, ny, lx, ly, p) in enumerate(cases):
        msh = mesh.MeshConfig(nx, ny, lx, ly)
        b = basis.gll_basis(p)
        N = (p * ny, p * nx)
        u = rng.standard_normal(N)
        nu = 1.0 + 0.5 * rng.random(N)
        out[f"op{i}_case"] = np.array([nx, ny, lx, ly, p])
        out[f"op{i}_u"] = u
        out[f"op{i}_nu"] = nu
        out[f"op{i}_Au"] = operators.PoissonOperator(b, msh).apply(u)
        dop = operators.DiffusionOperator(b, msh, nu)
        out[f"op{i}_Bu"] = dop.apply(u)
        out[f"op{i}_nubar"] = dop.element_mean_nu()
        out[f"op{i}_nufield"] = operators.diffusivity_field(msh, b, 0.9, 0.0)
    out["n_op"] = np.array(len(cases))
    save("operators", **out)

    # -- schwarz.py: AdditiveSchwarz.smooth (Poisson and diffusion)
    out = {}
    sweeps = [(4, 4, 2.0, 2.0, 4, 1, "w5", None), (6, 5, 2.0, 2.0, 4, 1, "wa", None),
              (5, 6, 3.0, 1.0, 8, 2, "w5", None), (4, 4, 1.0, 1.0, 16, 1, "w5", None),
              (3, 3, 1.0, 1.0, 32, 1, "w3", None), (4, 3, 1.0, 1.0, 8, 1, "w5", 0.5),
              (4, 4, 1.0, 1.0, 12, 1, "w7", None), (3, 4, 1.0, 1.0, 24, 3, "w5", 0.9),
              (8, 8, 2.0, 2.0, 2, 0, "w1", None), (4, 4, 1.0, 1.0, 16, 4, "wt", None)]
    for i, (nx, ny, lx, ly, p, n_o, kind, nu_hat) in enumerate(sweeps):
        msh = mesh.MeshConfig(nx, ny, lx, ly)
        b = basis.gll_basis(p)
        lay = mesh.layout_for(msh, p)
        if nu_hat is None:
            op = operators.PoissonOperator(b, msh)
            nb = None
        else:
            op = operators.DiffusionOperator(b, msh, operators.diffusivity_field(msh, b, nu_hat, 0.2))
            nb = op.element_mean_nu()
        sm = schwarz.AdditiveSchwarz(b, lay, msh.dx, msh.dy, n_o, schwarz.WeightKind(kind), nu_bar=nb)
        u0 = rng.random((lay.N_y, lay.N_x))
        f = rng.standard_normal((lay.N_y, lay.N_x))
        out[f"sw{i}_case"] = np.array([nx, ny, lx, ly, p, n_o, -1.0 if nu_hat is None else nu_hat])
        out[f"sw{i}_kind"] = np.array(kind)
        out[f"sw{i}_u0"] = u0
        out[f"sw{i}_f"] = f
        out[f"sw{i}_u1"] = sm.smooth(op, u0.copy(), f, 1)
        out[f"sw{i}_u2"] = sm.smooth(op, u0.copy(), f, 2)
    out["n_sw"] = np.array(len(sweeps))
    save("sweeps", **out)

    # -- multigrid.py: transfers, coarse solve, v_cycle
    out = {}
    msh = mesh.MeshConfig(4, 3, 2.0, 2.0)
    h = multigrid.build_hierarchy(msh, 32, multigrid.OverlapRule("fixed", 1))
    for l in range(1, h.depth + 1):
        lo, hi = h.levels[l - 1].op.layout, h.levels[l].op.layout
        uc = rng.standard_normal((lo.N_y, lo.N_x))
        vf = rng.standard_normal((hi.N_y, hi.N_x))
        out[f"tr{l}_uc"] = uc
        out[f"tr{l}_vf"] = vf
        out[f"tr{l}_P"] = multigrid.prolongate(h, l, uc)
        out[f"tr{l}_R"] = multigrid.restrict_residual(h, l, vf)
    for i, (nx, ny, lx, ly, nu_hat) in enumerate([(4, 4, 2.0, 2.0, None), (8, 8, 1.0, 1.0, None),
                                                   (16, 8, 8.0, 1.0, None), (8, 8, 1.0, 1.0, 0.9)]):
        msh = mesh.MeshConfig(nx, ny, lx, ly)
        h = multigrid.build_hierarchy(msh, 2, multigrid.OverlapRule("fixed", 1), nu_hat=nu_hat)
        f0 = rng.standard_normal((ny, nx))
        out[f"cs{i}_f0"] = f0
        out[f"cs{i}_u0"] = multigrid.coarse_solve(h, f0)
    for i, (nx, ny, lx, ly, p, rule, nu_hat, n_post) in enumerate([
            (8, 8, 1.0, 1.0, 8, "fixed:1", None, 0), (4, 4, 2.0, 2.0, 16, "ceilp8", None, 0),
            (6, 4, 8.0, 1.0, 8, "fixed:1", None, 1), (4, 4, 1.0, 1.0, 8, "ceilp8", 0.5, 1)]):
        msh = mesh.MeshConfig(nx, ny, lx, ly)
        h = multigrid.build_hierarchy(msh, p, multigrid.OverlapRule.parse(rule), nu_hat=nu_hat,
                                      n_post=n_post)
        lay = h.top.op.layout
        f = operators.project_mean(np.random.default_rng(i).standard_normal((lay.N_y, lay.N_x)))
        u = rng.random((lay.N_y, lay.N_x))
        out[f"vc{i}_case"] = np.array([nx, ny, lx, ly, p, -1.0 if nu_hat is None else nu_hat, n_post])
        out[f"vc{i}_rule"] = np.array(rule)
        out[f"vc{i}_f"] = f
        out[f"vc{i}_uin"] = u
        out[f"vc{i}_uout"] = multigrid.v_cycle(h, u.copy(), f)
        out[f"vc{i}_uzero"] = multigrid.v_cycle(h, np.zeros_like(f), f)
    save("multigrid", **out)

    # -- krylov.py: C1 (BASELINE configs[0]) histories, seeds 0,1,2, both solvers
    out = {}
    msh = mesh.MeshConfig(8, 8, 1.0, 1.0)
    h = multigrid.build_hierarchy(msh, 8, multigrid.OverlapRule("fixed", 1))
    lay = h.top.op.layout
    for seed in (0, 1, 2):
        f = operators.project_mean(np.random.default_rng(seed).standard_normal((lay.N_y, lay.N_x)))
        for solver in ("mg", "mgcg"):
            cfg = krylov.SolveConfig(solver=solver, tol_reduction=1e10, max_cycles=200, seed=seed)
            u, rep = krylov.solve(h, f, cfg, u0=np.zeros_like(f))
            out[f"c1_{solver}_{seed}_res"] = np.array(rep.residuals)
            out[f"c1_{solver}_{seed}_u"] = u
            out[f"c1_{solver}_{seed}_rbar"] = np.array(rep.rbar)
    # the reference's own random-start (krylov.py:36-39) path, seed 5, AR 1, p=8, 4x4
    msh = mesh.MeshConfig(4, 4)
    h = multigrid.build_hierarchy(msh, 8, multigrid.OverlapRule("fixed", 1))
    f, _ = operators.poisson_benchmark(msh, h.top.basis)
    for solver in ("mg", "mgcg"):
        u, rep = krylov.solve(h, f, krylov.SolveConfig(solver=solver, tol_reduction=1e8,
                                                       max_cycles=40, seed=5))
        out[f"rs_{solver}_res"] = np.array(rep.residuals)
        out["rs_f"] = f
    save("krylov", **out)


def large():
    """BASELINE-size runs of the reference (slow; sampled outputs only)."""
    basis, krylov, mesh, multigrid, operators, schwarz = _ref()
    out = {}
    # C2: 64x64, p=16, MG solve (13 cycles in the survey), seed 0
    t = time.time()
    msh = mesh.MeshConfig(64, 64, 1.0, 1.0)
    h = multigrid.build_hierarchy(msh, 16, multigrid.OverlapRule("fixed", 1))
    lay = h.top.op.layout
    f = operators.project_mean(np.random.default_rng(0).standard_normal((lay.N_y, lay.N_x)))
    u1 = multigrid.v_cycle(h, np.zeros_like(f), f)
    out["c2_vcycle_sample"] = u1[::16, ::16].copy()
    out["c2_vcycle_norm"] = np.array(np.linalg.norm(u1))
    out["c2_vcycle_resnorm"] = np.array(np.linalg.norm(f - h.top.op.apply(u1)))
    for solver in ("mg", "mgcg"):
        u, rep = krylov.solve(h, f, krylov.SolveConfig(solver=solver, tol_reduction=1e10), u0=np.zeros_like(f))
        out[f"c2_{solver}_res"] = np.array(rep.residuals)
        out[f"c2_{solver}_sample"] = u[::16, ::16].copy()
    print(f"C2 done in {time.time() - t:.1f}s")
    save("large_c2", **out)


def _hand_hierarchy(multigrid, basis, mesh, operators, schwarz, msh, orders, nu_hat, nu_shift=0.0):
    """Hand-assembled reference hierarchy for non-power-of-two p (build_hierarchy
    rejects p=24, multigrid.py:139-140) from the reference's own Level,
    MultigridHierarchy, AdditiveSchwarz, interp_matrix, _global_prolongation."""
    levels = []
    for l, p_l in enumerate(orders):
        b = basis.gll_basis(p_l)
        lay = mesh.layout_for(msh, p_l)
        if nu_hat is None:
            op, nb = operators.PoissonOperator(b, msh), None
        else:
            op = operators.DiffusionOperator(b, msh, operators.diffusivity_field(msh, b, nu_hat, nu_shift))
            nb = op.element_mean_nu()
        if l == 0:
            lv = multigrid.Level(l, b, op, None, 0, 0, 0)
        else:
            sm = schwarz.AdditiveSchwarz(b, lay, msh.dx, msh.dy, 1, schwarz.WeightKind.QUINTIC, nu_bar=nb)
            lv = multigrid.Level(l, b, op, sm, 1, 0, 1)
            j = basis.interp_matrix(levels[-1].basis, b).matrix
            lv.px = multigrid._global_prolongation(j, orders[l - 1], p_l, msh.n_x)
            lv.py = multigrid._global_prolongation(j, orders[l - 1], p_l, msh.n_y)
        lv.u = lay.zeros()
        lv.f = lay.zeros()
        levels.append(lv)
    return multigrid.MultigridHierarchy(msh, levels)


def xlarge():
    """C3 one V-cycle, C5-like reduced MGCG (64^2, p=24), C4 full MGCG (~20 min)."""
    basis, krylov, mesh, multigrid, operators, schwarz = _ref()
    out = {}
    t = time.time()
    msh = mesh.MeshConfig(128, 128, 1.0, 1.0)
    h = multigrid.build_hierarchy(msh, 32, multigrid.OverlapRule("fixed", 1))
    lay = h.top.op.layout
    f = operators.project_mean(np.random.default_rng(0).standard_normal((lay.N_y, lay.N_x)))
    r0 = np.linalg.norm(f)
    u1 = multigrid.v_cycle(h, np.zeros_like(f), f)
    out["c3_vcycle_sample"] = u1[::64, ::64].copy()
    out["c3_vcycle_norm"] = np.array(np.linalg.norm(u1))
    out["c3_res"] = np.array([r0, np.linalg.norm(f - h.top.op.apply(u1))])
    print(f"C3 done in {time.time() - t:.1f}s")
    save("xlarge_c3", **out)
    out = {}
    t = time.time()
    msh = mesh.MeshConfig(64, 64, 1.0, 1.0)
    h = _hand_hierarchy(multigrid, basis, mesh, operators, schwarz, msh, [1, 3, 6, 12, 24], 0.9, 0.0)
    lay = h.top.op.layout
    f = operators.project_mean(np.random.default_rng(0).standard_normal((lay.N_y, lay.N_x)))
    u, rep = krylov.solve(h, f, krylov.SolveConfig(solver="mgcg", tol_reduction=1e10), u0=np.zeros_like(f))
    out["c5r_mgcg_res"] = np.array(rep.residuals)
    out["c5r_mgcg_sample"] = u[::24, ::24].copy()
    print(f"C5-reduced done in {time.time() - t:.1f}s")
    save("xlarge_c5r", **out)
    out = {}
    t = time.time()
    msh = mesh.MeshConfig(256, 256, 8.0, 1.0)
    h = multigrid.build_hierarchy(msh, 16, multigrid.OverlapRule("fixed", 1))
    lay = h.top.op.layout
    f = operators.project_mean(np.random.default_rng(0).standard_normal((lay.N_y, lay.N_x)))
    u, rep = krylov.solve(h, f, krylov.SolveConfig(solver="mgcg", tol_reduction=1e10), u0=np.zeros_like(f))
    out["c4_mgcg_res"] = np.array(rep.residuals)
    out["c4_mgcg_sample"] = u[::64, ::64].copy()
    out["c4_breakdown"] = np.array(rep.breakdown)
    print(f"C4 done in {time.time() - t:.1f}s")
    save("xlarge_c4", **out)


def harness():
    """variable/post-smoothed cycles and the reference's
    run_single / CSV harness (presets.py:90-111, :159-204) on small specs."""
    import json
    basis, krylov, mesh, multigrid, operators, schwarz = _ref()
    from schwarzmg import presets
    out = {}
    # f1: variable V-cycle (2^(L-l) smoothing steps, n_pre = n_post = 1), Poisson and diffusion
    for i, (nx, ny, p, nu_hat) in enumerate([(4, 4, 8, None), (4, 4, 8, 0.9), (6, 4, 16, 0.5)]):
        msh = mesh.MeshConfig(nx, ny, 1.0, 1.0)
        h = multigrid.build_hierarchy(msh, p, multigrid.OverlapRule("fixed", 1), n_pre=1, n_post=1,
                                      variable=True, nu_hat=nu_hat)
        lay = h.top.op.layout
        f = operators.project_mean(np.random.default_rng(10 + i).standard_normal((lay.N_y, lay.N_x)))
        u = np.random.default_rng(20 + i).random((lay.N_y, lay.N_x))
        out[f"var{i}_case"] = np.array([nx, ny, p, -1.0 if nu_hat is None else nu_hat])
        out[f"var{i}_f"] = f
        out[f"var{i}_uin"] = u
        out[f"var{i}_uout"] = multigrid.v_cycle(h, u.copy(), f)
    # f2: run_single records for small specs (the CSV schema's numbers)
    specs = [presets.RunSpec(p=8, n_x=4, n_y=4),
             presets.RunSpec(solver="mgcg", p=8, n_x=4, n_y=4, ar=2.0, overlap_rule="ceilp8"),
             presets.RunSpec(p=4, n_x=8, n_y=8, weight="w3"),
             presets.RunSpec(solver="mgcg", p=8, n_x=4, n_y=4, n_pre=1, n_post=1, nu_hat=0.5),
             presets.RunSpec(solver="mgcg", p=8, n_x=4, n_y=4, ar=2.0, overlap_rule="ceilp2", n_pre=1,
                             n_post=1, cycle="var", nu_hat=0.9)]
    recs = []
    for k, sp in enumerate(specs):
        for seed in (0, 1):
            r = presets.run_single(sp, seed)
            recs.append(r)
    out["rs_specs"] = np.array(json.dumps([presets.asdict(sp) for sp in specs]))
    out["rs_records"] = np.array(presets.records_to_json(recs))
    out["rs_csv"] = np.array(presets.records_to_csv(recs))
    grids = {name: [presets.asdict(sp) for sp in presets.preset_grid(name, full=full)]
             for name in presets.PRESET_NAMES for full in (False,)}
    grids.update({name + ":full": [presets.asdict(sp) for sp in presets.preset_grid(name, full=True)]
                  for name in ("table4",)})
    out["grids"] = np.array(json.dumps(grids))
    refs = {name: [presets.reference_rbar(name, sp) for sp in presets.preset_grid(name)]
            for name in presets.PRESET_NAMES}
    out["grid_refs"] = np.array(json.dumps(refs))
    save("harness", **out)
    # the published mean rates the reference's presets compare against
    # (presets.py TABLE2_RBAR..TABLE5), as data for the B200 harness
    pub = {"table2": {str(k): list(v) for k, v in presets.TABLE2_RBAR.items()},
           "table3": {str(k): list(v) for k, v in presets.TABLE3_RBAR.items()},
           "table4": {f"{k[0]},{k[1]}": {m: list(x) for m, x in v.items()} for k, v in presets.TABLE4.items()},
           "table5": {f"{k[0]},{k[1]}": {m: list(x) for m, x in v.items()} for k, v in presets.TABLE5.items()},
           "columns": list(presets._WEIGHT_COLUMNS)}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1512_02390_b200", "data",
                        "published_rates.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as fh:
        json.dump(pub, fh, indent=1)
    print(f"wrote {path}")



def mult():
    """the multiplicative smoother (schwarz.py:293-353) --
    single sweeps (forward, then reverse) and a multiplicative V-cycle and
    MG / MGCG histories, all from the reference."""
    basis, krylov, mesh, multigrid, operators, schwarz = _ref()
    out = {}
    cases = [(4, 4, 4, 1, None, 1.0, 1.0), (3, 5, 8, 2, None, 1.0, 2.0), (2, 2, 4, 1, None, 1.0, 1.0),
             (4, 4, 4, 1, 0.5, 1.0, 1.0), (4, 3, 3, 1, None, 1.0, 1.0), (6, 4, 8, 1, 0.9, 2.0, 1.0)]
    for i, (nx, ny, p, n_o, nu_hat, lx, ly) in enumerate(cases):
        msh = mesh.MeshConfig(nx, ny, lx, ly)
        b = basis.gll_basis(p)
        lay = mesh.layout_for(msh, p)
        if nu_hat is None:
            op = operators.PoissonOperator(b, msh)
            nu_bar = None
        else:
            op = operators.DiffusionOperator(b, msh, operators.diffusivity_field(msh, b, nu_hat, 0.2))
            nu_bar = op.element_mean_nu()
        cnt = schwarz.SweepCounter()
        sm = schwarz.MultiplicativeSchwarz(b, lay, msh.dx, msh.dy, n_o, nu_bar=nu_bar, counter=cnt)
        rng = np.random.default_rng(300 + i)
        u = rng.standard_normal((lay.N_y, lay.N_x))
        f = rng.standard_normal((lay.N_y, lay.N_x))
        out[f"ms{i}_case"] = np.array([nx, ny, p, n_o, -1.0 if nu_hat is None else nu_hat, lx, ly])
        out[f"ms{i}_u"] = u.copy()
        out[f"ms{i}_f"] = f
        u1 = sm.smooth(op, u.copy(), f, 1)          # forward sweep
        out[f"ms{i}_u1"] = u1.copy()
        out[f"ms{i}_u2"] = sm.smooth(op, u1, f, 1)  # reverse sweep
    # multiplicative V-cycle and solver histories (C1-like, smaller mesh)
    for j, (nx, p, nu_hat) in enumerate([(4, 8, None), (4, 8, 0.5)]):
        msh = mesh.MeshConfig(nx, nx, 1.0, 1.0)
        h = multigrid.build_hierarchy(msh, p, multigrid.OverlapRule("fixed", 1), smoother="mult", nu_hat=nu_hat)
        lay = h.top.op.layout
        f = operators.project_mean(np.random.default_rng(400 + j).standard_normal((lay.N_y, lay.N_x)))
        u = np.random.default_rng(500 + j).standard_normal((lay.N_y, lay.N_x))
        out[f"mv{j}_case"] = np.array([nx, p, -1.0 if nu_hat is None else nu_hat])
        out[f"mv{j}_f"] = f
        out[f"mv{j}_uin"] = u.copy()
        h.reset_smoothers()
        out[f"mv{j}_uout"] = multigrid.v_cycle(h, u.copy(), f)
        for solver in ("mg", "mgcg"):
            _, rep = krylov.solve(h, f, krylov.SolveConfig(solver=solver, seed=0), u0=np.zeros_like(f))
            out[f"mv{j}_{solver}_res"] = np.array(rep.residuals)
    save("mult", **out)


def c5full():
    """BASELINE configs[4] (C5) at full size: 512x512 elements, p=24, levels
    (1,3,6,12,24), nu_hat=0.9, nu_shift=0 (== [0,2pi]^2, nu = 1+0.9 sin x sin y),
    seeded mean-zero Gaussian f, zero start, MGCG to 1e10 (krylov.py:70-115).
    About 2-4 h and ~18 GB RSS in this container; run once in the background."""
    basis, krylov, mesh, multigrid, operators, schwarz = _ref()
    out = {}
    t = time.time()
    msh = mesh.MeshConfig(512, 512, 1.0, 1.0)
    h = _hand_hierarchy(multigrid, basis, mesh, operators, schwarz, msh, [1, 3, 6, 12, 24], 0.9, 0.0)
    lay = h.top.op.layout
    f = operators.project_mean(np.random.default_rng(0).standard_normal((lay.N_y, lay.N_x)))
    print(f"C5 build {time.time() - t:.1f}s", flush=True)
    u, rep = krylov.solve(h, f, krylov.SolveConfig(solver="mgcg", tol_reduction=1e10), u0=np.zeros_like(f))
    out["c5_mgcg_res"] = np.array(rep.residuals)
    out["c5_mgcg_sample"] = u[::192, ::192].copy()
    out["c5_mgcg_norm"] = np.array(np.linalg.norm(u))
    out["c5_breakdown"] = np.array(rep.breakdown)
    out["c5_wall"] = np.array(time.time() - t)
    print(f"C5 full done in {time.time() - t:.1f}s, {rep.cycles} cycles", flush=True)
    save("xlarge_c5", **out)


def c3full():
    """BASELINE configs[2] (C3): 128x128, p=32, fixed:1, full MG history to 1e10
    (krylov.py:49-67) from a zero start, seed 0."""
    basis, krylov, mesh, multigrid, operators, schwarz = _ref()
    out = {}
    t = time.time()
    msh = mesh.MeshConfig(128, 128, 1.0, 1.0)
    h = multigrid.build_hierarchy(msh, 32, multigrid.OverlapRule("fixed", 1))
    lay = h.top.op.layout
    f = operators.project_mean(np.random.default_rng(0).standard_normal((lay.N_y, lay.N_x)))
    u, rep = krylov.solve(h, f, krylov.SolveConfig(solver="mg", tol_reduction=1e10), u0=np.zeros_like(f))
    out["c3_mg_res"] = np.array(rep.residuals)
    out["c3_mg_sample"] = u[::64, ::64].copy()
    print(f"C3 full MG done in {time.time() - t:.1f}s, {rep.cycles} cycles", flush=True)
    save("xlarge_c3_mg", **out)


def ceilp8():
    """The paper's recommended overlap rule ceil(p/8) (multigrid.py:28-54) at the
    BASELINE top orders: additive sweeps at p=16/24/32 (n_o=2/3/4, m=21/31/41,
    schwarz.py:255-275), Poisson and diffusion, ragged meshes; one ceilp8
    V-cycle at p=32 (multigrid.py:231-251); coarse solves of p=1 meshes above
    64^2 (multigrid.py:196-228: plain CG to 1e-12), Poisson and diffusion.
    Inputs are regenerated from per-case seeds by the tests (ceilp8_inputs)
    instead of stored, to keep the fixture small."""
    basis, krylov, mesh, multigrid, operators, schwarz = _ref()
    out = {}
    for i, (nx, ny, lx, ly, p, n_o, nu_hat) in enumerate(CEILP8_SWEEPS):
        msh = mesh.MeshConfig(nx, ny, lx, ly)
        b = basis.gll_basis(p)
        lay = mesh.layout_for(msh, p)
        if nu_hat is None:
            op, nb = operators.PoissonOperator(b, msh), None
        else:
            op = operators.DiffusionOperator(b, msh, operators.diffusivity_field(msh, b, nu_hat, 0.2))
            nb = op.element_mean_nu()
        sm = schwarz.AdditiveSchwarz(b, lay, msh.dx, msh.dy, n_o, schwarz.WeightKind.QUINTIC, nu_bar=nb)
        u0, f = ceilp8_inputs(800 + i, (lay.N_y, lay.N_x))
        out[f"sw{i}_u1"] = sm.smooth(op, u0.copy(), f, 1)
        out[f"sw{i}_in_sample"] = np.array([u0[0, 0], f[-1, -1]])
    for i, (nx, ny, p) in enumerate(CEILP8_VCYCLES):
        msh = mesh.MeshConfig(nx, ny, 1.0, 1.0)
        h = multigrid.build_hierarchy(msh, p, multigrid.OverlapRule.parse("ceilp8"))
        lay = h.top.op.layout
        u, f = ceilp8_inputs(900 + i, (lay.N_y, lay.N_x))
        f = operators.project_mean(f)
        out[f"vc{i}_uout"] = multigrid.v_cycle(h, u.copy(), f)
    for i, (nx, ny, lx, ly, nu_hat) in enumerate(CEILP8_COARSE):
        msh = mesh.MeshConfig(nx, ny, lx, ly)
        h = multigrid.build_hierarchy(msh, 2, multigrid.OverlapRule("fixed", 1), nu_hat=nu_hat, nu_shift=0.0)
        _, f0 = ceilp8_inputs(950 + i, (ny, nx))
        out[f"cs{i}_u0"] = multigrid.coarse_solve(h, f0)
    save("ceilp8", **out)


# (n_x, n_y, l_x, l_y, p, n_o = ceil(p/8), nu_hat or None)
CEILP8_SWEEPS = [(6, 5, 1.0, 1.0, 16, 2, None), (5, 4, 1.0, 1.0, 24, 3, None), (5, 6, 2.0, 1.0, 32, 4, None),
                 (4, 4, 1.0, 1.0, 24, 3, 0.9), (4, 5, 1.0, 1.0, 32, 4, 0.5), (9, 7, 1.0, 1.0, 16, 2, None)]
CEILP8_VCYCLES = [(8, 8, 32)]
# p = 1 coarse meshes above 64^2 (n_x, n_y, l_x, l_y, nu_hat or None; nu_shift 0)
CEILP8_COARSE = [(128, 128, 1.0, 1.0, None), (128, 128, 1.0, 1.0, 0.9), (256, 128, 2.0, 1.0, 0.9)]


def ceilp8_inputs(seed, shape):
    """(u0 in [0,1), f ~ N(0,1)) for one ceilp8 fixture case."""
    rng = np.random.default_rng(seed)
    return rng.random(shape), rng.standard_normal(shape)

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true")
    ap.add_argument("--only-large", action="store_true")
    ap.add_argument("--xlarge", action="store_true")
    ap.add_argument("--harness", action="store_true", help="only the f1/f2 harness fixtures")
    ap.add_argument("--mult", action="store_true", help="only the f3 multiplicative fixtures")
    ap.add_argument("--c5full", action="store_true", help="only the full-size C5 MGCG history (hours)")
    ap.add_argument("--c3full", action="store_true", help="only the full C3 MG history")
    ap.add_argument("--ceilp8", action="store_true", help="only the ceil(p/8) sweeps / V-cycles / coarse solves")
    a = ap.parse_args()
    if a.c5full:
        c5full()
        sys.exit(0)
    if a.c3full:
        c3full()
        sys.exit(0)
    if a.ceilp8:
        ceilp8()
        sys.exit(0)
    if a.mult:
        mult()
        sys.exit(0)
    if a.harness:
        harness()
        sys.exit(0)
    if not (a.only_large or a.xlarge):
        small()
        harness()
        mult()
    if a.large or a.only_large:
        large()
    if a.xlarge:
        xlarge()
