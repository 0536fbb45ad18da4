"""Halo-free kernels with caller-owned ring workspaces (include/smg.h): the tensor-core
operator kernel (smg_op_residual_ws; csrc/smg_opd.cu opdh_kernel + opdh_fixup) and the
warp-per-fine-element restriction (smg_restrict_ws; csrc/smg_rw.cu) against the oracle and
against the ring-less entry points.  Reference: operators.py:30-103, multigrid.py:188-193."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,p,nx,ny,lx,ly", [("diffusion", 12, 5, 3, 1.0, 1.0), ("diffusion", 12, 16, 8, 1.0, 4.0),
                                                ("diffusion", 24, 4, 3, 1.0, 1.0), ("diffusion", 24, 6, 8, 2.0, 1.0),
                                                ("poisson", 32, 3, 4, 1.0, 1.3), ("poisson", 32, 6, 6, 8.0, 1.0)])
def test_operator_ring_path(kind, p, nx, ny, lx, ly):
    import paper_1512_02390_b200 as P
    from oracle import smg_oracle as O
    from paper_1512_02390_b200 import _native as N
    mesh = P.MeshConfig(nx, ny, lx, ly)
    b = P.gll_basis(p)
    rng = np.random.default_rng(17)
    lay = P.layout_for(mesh, p)
    u, f = rng.standard_normal(lay.shape), rng.standard_normal(lay.shape)
    if kind == "poisson":
        op = P.PoissonOperator(b, mesh)
        want = O.Poisson(O.gll(p), nx, ny, mesh.dx, mesh.dy).apply(u)
    else:
        nu = 0.2 + rng.random(lay.shape)
        op = P.DiffusionOperator(b, mesh, nu)
        want = O.Diffusion(O.gll(p), nx, ny, mesh.dx, mesh.dy, nu).apply(u)
    assert op.ring is not None and op.ring.numel() == int(N.lib().smg_op_ring_doubles(op._handle.raw)) == nx * ny * 2 * p
    ud, fd = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
    sc = np.abs(want).max()
    assert np.abs(op.apply(ud).cpu().numpy() - want).max() / sc < 1e-12
    r = torch.empty_like(ud)
    op.residual_into(ud, fd, r)
    assert np.abs(r.cpu().numpy() - (f - want)).max() / sc < 1e-12
    # the ring-less entry point (fused kernel with halo) and a NULL ring agree with it to rounding
    old, nul = torch.empty_like(ud), torch.empty_like(ud)
    N.check(N.lib().smg_op_residual(op._handle.raw, N.ptr(ud), N.ptr(fd), N.ptr(old), N.stream()), "residual")
    N.check(N.lib().smg_op_residual_ws(op._handle.raw, N.ptr(ud), N.ptr(fd), N.ptr(nul), None, N.stream()), "residual")
    assert torch.equal(old, nul)
    assert (r - old).abs().max().item() / sc < 1e-13
    # bitwise reproducible
    r2 = torch.empty_like(ud)
    op.residual_into(ud, fd, r2)
    assert torch.equal(r, r2)


@pytest.mark.parametrize("p,orders,nx,ny", [(32, None, 4, 3), (24, (1, 3, 6, 12, 24), 5, 4), (16, None, 128, 128)])
def test_restriction_ring_path(p, orders, nx, ny):
    import paper_1512_02390_b200 as P
    from paper_1512_02390_b200 import _native as N
    mesh = P.MeshConfig(nx, ny, 1.0, 1.0)
    h = P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1), orders=orders) if orders else \
        P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1))
    tr = h.top.transfer
    pc = h.levels[-2].basis.p
    assert tr.ws is not None and tr.ws.numel() == nx * ny * (2 * pc + 1)
    torch.manual_seed(3)
    r = torch.randn(h.top.op.layout.shape, dtype=torch.float64, device="cuda")
    got = P.restrict_residual(h, h.depth, r)
    old = torch.empty_like(got)
    N.check(N.lib().smg_restrict(tr.handle.raw, N.ptr(r), N.ptr(old), N.stream()), "restrict")
    assert (got - old).abs().max().item() / old.abs().max().item() < 1e-13
    # adjointness with the prolongation (multigrid.py:180-193): <P^T r, c> = <r, P c>
    c = torch.randn(old.shape, dtype=torch.float64, device="cuda")
    pcf = P.prolongate(h, h.depth, c)
    lhs, rhs = (got * c).sum().item(), (r * pcf).sum().item()
    assert abs(lhs - rhs) < 1e-11 * max(abs(lhs), abs(rhs), 1.0)
    assert torch.equal(P.restrict_residual(h, h.depth, r), got)


@pytest.mark.parametrize("kind,p,nx,ny", [("poisson", 16, 8, 6), ("poisson", 8, 4, 4), ("poisson", 32, 4, 3),
                                          ("poisson", 4, 8, 8), ("diffusion", 24, 4, 4), ("diffusion", 24, 40, 30),
                                          ("diffusion", 6, 8, 8)])
def test_apply_dot(kind, p, nx, ny):
    """smg_op_apply_dot: q = A p and p . q (fused in the warp-per-element kernel at p = 8, 16 and
    in the persistent tensor-core diffusion kernel at p = 24 -- 40 x 30 elements: several per CTA;
    apply + dot pass elsewhere) against apply() and a float64 dot; uninitialised workspace."""
    import paper_1512_02390_b200 as P
    from paper_1512_02390_b200 import _native as N
    mesh = P.MeshConfig(nx, ny, 1.0, 2.0)
    b = P.gll_basis(p)
    rng = np.random.default_rng(3)
    lay = P.layout_for(mesh, p)
    op = P.PoissonOperator(b, mesh) if kind == "poisson" else P.DiffusionOperator(b, mesh, 0.3 + rng.random(lay.shape))
    u = torch.from_numpy(rng.standard_normal(lay.shape)).cuda()
    want_q = op.apply(u)
    want = float((u * want_q).sum().item())
    q = torch.empty_like(u)
    d = torch.full((1,), float("nan"), dtype=torch.float64, device="cuda")
    op.partials.fill_(float("nan"))   # the call must not depend on the workspace contents
    for _ in range(2):
        N.check(N.lib().smg_op_apply_dot(op._handle.raw, N.ptr(u), N.ptr(q), N.ptr(d), N.ptr(op.partials),
                                         op.ring_ptr(), N.stream()), "apply_dot")
        assert torch.equal(q, want_q)
        assert abs(d.item() - want) <= 1e-12 * float((u.abs() * want_q.abs()).sum().item())


@pytest.mark.parametrize("p", [16, 8, 4])
@pytest.mark.parametrize("nx,ny,lx,ly", [(6, 4, 1.0, 1.0), (4, 4, 1.0, 1.0), (64, 64, 1.0, 1.0), (8, 10, 2.0, 1.0),
                                         (128, 128, 1.0, 1.0)])
def test_fused_residual_restriction_p16(nx, ny, lx, ly, p):
    """smg_residual_restrict_ws at p_f = 16, 8, 4 (Poisson): the warp-per-element residual kernel restricts
    its element in place (r is never stored) + restrict_fixup, against residual then restriction
    (multigrid.py:247-248), twice into a dirty workspace; bitwise reproducible."""
    import paper_1512_02390_b200 as P
    from paper_1512_02390_b200 import _native as N
    mesh = P.MeshConfig(nx, ny, lx, ly)
    h = P.build_hierarchy(mesh, p, P.OverlapRule("fixed", 1))
    lv = h.top
    tr = lv.transfer
    assert tr.ws is not None and tr.ws.numel() == nx * ny * (p + 1), "no ring: the fused path is not engaged"
    torch.manual_seed(11)
    u = torch.randn(lv.op.layout.shape, dtype=torch.float64, device="cuda")
    f = torch.randn(lv.op.layout.shape, dtype=torch.float64, device="cuda")
    r = torch.empty_like(u)
    N.check(N.lib().smg_op_residual(lv.op._handle.raw, N.ptr(u), N.ptr(f), N.ptr(r), N.stream()), "residual")
    want = torch.empty(h.levels[-2].op.layout.shape, dtype=torch.float64, device="cuda")
    N.check(N.lib().smg_restrict(tr.handle.raw, N.ptr(r), N.ptr(want), N.stream()), "restrict")
    tr.ws.fill_(float("nan"))
    work = torch.full_like(u, float("nan"))
    got = [torch.full_like(want, float("nan")) for _ in range(2)]
    for g in got:
        N.check(N.lib().smg_residual_restrict_ws(tr.handle.raw, lv.op._handle.raw, N.ptr(u), N.ptr(f), N.ptr(g),
                                                 N.ptr(work), tr.ws_ptr(), lv.op.ring_ptr(), N.stream()), "rr")
    assert torch.equal(got[0], got[1])
    assert (got[0] - want).abs().max().item() <= 1e-13 * want.abs().max().item()
