"""CPU checks of the drop-in boundary: libsmg.so loads and exports exactly the
C ABI declared in include/smg.h (no compute without a GPU)."""

import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "smg.h")
LIB = os.path.join(ROOT, "paper_1512_02390_b200", "libsmg.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(smg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ["smg_schwarz_correct", "smg_op_residual", "smg_prolongate", "smg_restrict",
              "smg_coarse_pinv", "smg_coarse_cg", "smg_cg_update", "smg_dot"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build libsmg.so first (__graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (smg_[a-z0-9_]+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, f"declared but not exported: {missing}"


def test_ctypes_binding_covers_header():
    from paper_1512_02390_b200 import _native as N
    assert set(declared_symbols()) <= set(N.SIGNATURES), set(declared_symbols()) - set(N.SIGNATURES)
    lib = N.load(require_device=False)
    assert lib.smg_version() == 1
    assert lib.smg_reduce_ws_doubles() > 0


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_1512_02390_b200 import _native as N
    with pytest.raises(RuntimeError):
        N.load(require_device=True)
    lib = N.load(require_device=False)
    assert lib.smg_device_ok() == 0
