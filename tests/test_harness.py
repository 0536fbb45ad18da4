"""variable / post-smoothed cycles and the
run_single / preset / CSV harness, against fixtures produced by the
unmodified reference (oracle/make_golden.py --harness)."""
import io
import json
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from conftest import golden, maxrel  # noqa: E402
from oracle import smg_oracle as O  # noqa: E402
from paper_1512_02390_b200 import cli, presets  # noqa: E402


def _records(g):
    return [presets.RunRecord(**d) for d in json.loads(str(g["rs_records"]))]


def test_csv_text_matches_reference():
    g = golden("harness")
    assert presets.records_to_csv(_records(g)) == str(g["rs_csv"])


def test_csv_round_trip():
    g = golden("harness")
    recs = presets.read_csv(io.StringIO(str(g["rs_csv"])))
    assert presets.records_to_csv(recs) == str(g["rs_csv"])
    assert json.loads(presets.records_to_json(recs))[0]["solver"] == "mg"


def test_preset_grids_and_published_rates():
    g = golden("harness")
    grids = json.loads(str(g["grids"]))
    refs = json.loads(str(g["grid_refs"]))
    for name in presets.PRESET_NAMES:
        mine = presets.preset_grid(name)
        assert [presets.asdict(s) for s in mine] == grids[name], name
        assert [presets.reference_rbar(name, s) for s in mine] == refs[name], name
    assert [presets.asdict(s) for s in presets.preset_grid("table4", full=True)] == grids["table4:full"]
    with pytest.raises(ValueError):
        presets.preset_grid("nope")
    assert presets.rbar_tolerance(0.5) == 0.15 and presets.rbar_tolerance(2.0) == pytest.approx(0.3)


def test_cli_parser():
    p = cli.build_parser()
    a = p.parse_args(["solve", "--p", "8", "--nel", "4,6", "--solver", "mgcg", "--nu-hat", "0.5"])
    assert a.nel == (4, 6) and a.solver == "mgcg" and a.nu_hat == 0.5 and a.tol == 1e10
    assert p.parse_args(["solve", "--p", "4", "--nel", "5"]).nel == (5, 5)
    with pytest.raises(SystemExit) as e:
        p.parse_args(["solve", "--solver", "bogus", "--p", "4"])
    assert e.value.code == 1


def test_oracle_variable_cycles():
    g = golden("harness")
    for i in range(3):
        nx, ny, p, nu_hat = g[f"var{i}_case"]
        h = O.Hierarchy(int(nx), int(ny), 1.0, 1.0, int(p), n_pre=1, n_post=1, variable=True,
                        nu_hat=None if nu_hat < 0 else nu_hat)
        got = O.v_cycle(h, g[f"var{i}_uin"].copy(), g[f"var{i}_f"])
        assert maxrel(got, g[f"var{i}_uout"]) < 1e-10, (i, maxrel(got, g[f"var{i}_uout"]))


@pytest.mark.gpu
def test_gpu_variable_cycles(cuda_device):
    import paper_1512_02390_b200 as P
    g = golden("harness")
    for i in range(3):
        nx, ny, p, nu_hat = g[f"var{i}_case"]
        for coarse in ("cg", None):
            h = P.build_hierarchy(P.MeshConfig(int(nx), int(ny), 1.0, 1.0), int(p), P.OverlapRule("fixed", 1),
                                  n_pre=1, n_post=1, variable=True, nu_hat=None if nu_hat < 0 else nu_hat,
                                  coarse=coarse)
            out = P.v_cycle(h, g[f"var{i}_uin"], g[f"var{i}_f"]).cpu().numpy()
            tol = 1e-10 if coarse == "cg" else 1e-7
            assert maxrel(out, g[f"var{i}_uout"]) < tol, (i, coarse, maxrel(out, g[f"var{i}_uout"]))


@pytest.mark.gpu
def test_gpu_run_single_matches_reference_records(cuda_device):
    g = golden("harness")
    specs = [presets.RunSpec(**d) for d in json.loads(str(g["rs_specs"]))]
    want = _records(g)
    k = 0
    for sp in specs:
        for seed in (0, 1):
            got, ref = presets.run_single(sp, seed), want[k]
            k += 1
            assert abs(got.cycles - ref.cycles) <= 1, (sp, seed, got.cycles, ref.cycles)
            assert abs(got.rbar - ref.rbar) < 1e-3, (sp, seed, got.rbar, ref.rbar)
            assert got.converged == ref.converged and got.n10 == ref.n10
            assert abs(got.omega1 - ref.omega1) < 1e-2 * ref.omega1
            for f in ("solver", "smoother", "weight", "p", "n_x", "n_y", "ar", "overlap_rule", "n_pre",
                      "n_post", "cycle_type", "nu_hat", "shift_s", "seed"):
                assert getattr(got, f) == getattr(ref, f), f


@pytest.mark.gpu
def test_gpu_cli_solve(cuda_device, capsys):
    rc = cli.main(["solve", "--p", "8", "--nel", "4"])
    out = capsys.readouterr().out.splitlines()
    assert rc == 0 and out[0] == ",".join(presets.CSV_FIELDS) and out[1].startswith("mg,add,w5,8,4,4,1,fixed:1")


@pytest.mark.gpu
def test_gpu_problem_generation_matches_host(cuda_device):
    """device-generated fields == the host builders."""
    import paper_1512_02390_b200 as P
    for nx, ny, lx, ly, p, nu_hat in [(4, 4, 1.0, 1.0, 8, 0.9), (6, 4, 2.0, 1.0, 16, 0.5), (8, 8, 8.0, 1.0, 3, 0.0),
                                      (3, 5, 1.0, 2.0, 24, 0.3)]:
        mesh = P.MeshConfig(nx, ny, lx, ly)
        b = P.gll_basis(p)
        f_h, u_h = P.poisson_benchmark(mesh, b)
        f_d, u_d = P.poisson_benchmark_device(mesh, b)
        assert np.abs(f_d.cpu().numpy() - f_h).max() <= 1e-13 * np.abs(f_h).max()
        assert np.abs(u_d.cpu().numpy() - u_h).max() <= 1e-14
        f_h, nu_h, u_h = P.manufactured_rhs_diffusion(mesh, b, nu_hat)
        f_d, nu_d, u_d = P.manufactured_rhs_diffusion_device(mesh, b, nu_hat)
        assert np.abs(f_d.cpu().numpy() - f_h).max() <= 1e-13 * np.abs(f_h).max()
        assert np.abs(nu_d.cpu().numpy() - nu_h).max() <= 1e-14
        assert np.abs(u_d.cpu().numpy() - u_h).max() <= 1e-14
        op_h = P.DiffusionOperator(b, mesh, nu_h)
        op_d = P.DiffusionOperator(b, mesh, nu_d)
        assert np.abs(op_d.element_mean_nu() - op_h.element_mean_nu()).max() <= 1e-14
        assert op_d.nu.shape == nu_h.shape
