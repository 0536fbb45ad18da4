"""The one-launch ascending chain (smg_prolongate_chain) against the
per-level prolongations it replaces: bitwise on the top level, and whole
V-cycles bitwise with and without it (multigrid.py:247-248, n_post = 0)."""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_1512_02390_b200 as P
from paper_1512_02390_b200 import _native as NV

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", [(8, 8, 16), (12, 6, 8), (5, 7, 16), (4, 3, 4), (64, 64, 16)])
def test_chain_bitwise_vs_levels(cuda_device, case):
    nx, ny, p = case
    h = P.build_hierarchy(P.MeshConfig(nx, ny, 1.0, 1.0), p, P.OverlapRule("fixed", 1))
    K = h.depth
    rng = np.random.default_rng(nx * 100 + ny)
    fields = [torch.from_numpy(rng.standard_normal(lv.op.layout.shape)).cuda() for lv in h.levels]
    lib = NV.lib()
    st = NV.stream()
    # per level: u_l += P u_{l-1}', level by level
    ref = [f.clone() for f in fields]
    for l in range(1, K + 1):
        NV.check(lib.smg_prolongate(h.levels[l].transfer.handle.raw, NV.ptr(ref[l - 1]), NV.ptr(ref[l]), 1, st))
    got = [f.clone() for f in fields]
    tr = (C.c_void_p * K)(*[h.levels[l].transfer.handle.raw.value for l in range(1, K + 1)])
    us = (C.c_void_p * K)(*[got[l].data_ptr() for l in range(1, K + 1)])
    NV.check(lib.smg_prolongate_chain(tr, K, NV.ptr(got[0]), us, st), "chain")
    torch.cuda.synchronize()
    assert torch.equal(got[K], ref[K]), float((got[K] - ref[K]).abs().max())
    for l in range(1, K):   # intermediate levels are read, not written
        assert torch.equal(got[l], fields[l])


def test_chain_rejects_other_chains(cuda_device):
    h = P.build_hierarchy(P.MeshConfig(4, 4, 1.0, 1.0), 24, P.OverlapRule("fixed", 1), orders=(1, 3, 6, 12, 24))
    lib = NV.lib()
    u = [torch.zeros(lv.op.layout.shape, dtype=torch.float64, device="cuda") for lv in h.levels]
    tr = (C.c_void_p * 2)(*[h.levels[l].transfer.handle.raw.value for l in (1, 2)])
    us = (C.c_void_p * 2)(*[u[l].data_ptr() for l in (1, 2)])
    assert lib.smg_prolongate_chain(tr, 2, NV.ptr(u[0]), us, NV.stream()) == NV.SMG_EUNSUPPORTED


@pytest.mark.parametrize("p,nx", [(16, 64), (8, 8), (32, 6)])
def test_vcycle_with_chain_bitwise(cuda_device, monkeypatch, p, nx):
    mesh = P.MeshConfig(nx, nx, 1.0, 1.0)
    rng = np.random.default_rng(p)
    N = p * nx
    f = rng.standard_normal((N, N))
    f -= f.mean()
    u0 = torch.from_numpy(rng.standard_normal((N, N))).cuda()
    outs = []
    for chain in ("1", "0"):   # SMG_CHAIN=1 opts into the one-launch chain
        monkeypatch.setenv("SMG_CHAIN", chain)
        h = P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1))
        u = u0.clone()
        P.v_cycle(h, u, f)
        P.v_cycle(h, u, f)
        outs.append(u)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
