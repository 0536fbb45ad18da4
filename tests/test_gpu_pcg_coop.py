"""Cooperative coarse PCG (csrc/smg_fft.cu pcg_coop_kernel: the whole iteration loop in one kernel)
against the launch-per-step loop it replaces (SMG_PCG_COOP=0 is read once per process, so the
reference runs in a child process): same iteration counts, solutions equal to rounding
(reference multigrid.py:196-228 with the D^-1/2 A_P^+ D^-1/2 preconditioner of DESIGN 3.2)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_coop_matches_loop(tmp_path):
    tool = os.path.join(ROOT, "tools", "pcg_coop_check.py")
    out = subprocess.run([sys.executable, tool], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = [l for l in out.stdout.splitlines() if "iterations" in l]
    assert len(lines) == 4   # 128^2, 256^2, 512^2 and 256 x 128 nodes
    assert float(out.stdout.strip().splitlines()[-1].split()[-1]) < 1e-9
