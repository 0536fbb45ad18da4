"""Execute the reference-side ctypes stub of INTEGRATION.md §2 against the
UNMODIFIED reference (pip-installed into baseline/_ref; skipped when absent):
reference objects -> libsmg's C ABI -> the same smoothed iterate as the
reference's own AdditiveSchwarz.smooth (schwarz.py:268-275)."""

import os
import re
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _stub_source():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("## 2."):text.index("## 3.")]
    return re.search(r"```python\n(.*?)```", sec, re.S).group(1)


def test_stub_is_python():
    compile(_stub_source(), "INTEGRATION.md#2", "exec")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "schwarzmg")), reason="reference not installed in baseline/_ref")
def test_stub_matches_reference_smooth(cuda_device, monkeypatch):
    import torch
    monkeypatch.setenv("SMG_LIB", os.path.join(ROOT, "paper_1512_02390_b200", "libsmg.so"))
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from schwarzmg import basis, mesh, operators, schwarz
    ns = {}
    exec(_stub_source(), ns)
    rng = np.random.default_rng(7)
    for nx, ny, p, n_o in [(6, 5, 8, 1), (4, 4, 16, 2), (3, 4, 32, 1)]:
        msh = mesh.MeshConfig(nx, ny, 1.0, 1.0)
        b = basis.gll_basis(p)
        lay = mesh.layout_for(msh, p)
        op = operators.PoissonOperator(b, msh)
        sm = schwarz.AdditiveSchwarz(b, lay, msh.dx, msh.dy, n_o, schwarz.WeightKind.QUINTIC)
        u0 = rng.random((lay.N_y, lay.N_x))
        f = rng.standard_normal((lay.N_y, lay.N_x))
        want = sm.smooth(op, u0.copy(), f, 2)
        b200 = ns["B200Smoother"](sm, op)
        u = torch.from_numpy(u0.copy()).cuda()
        b200.smooth(u, torch.from_numpy(f).cuda(), 2)
        torch.cuda.synchronize()
        got = u.cpu().numpy()
        b200.close()
        assert np.abs(got - want).max() / np.abs(want).max() < 1e-12, (nx, ny, p, n_o)
