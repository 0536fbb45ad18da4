"""Element-row strip decomposition of the V-cycle and the outer solvers
across ranks (one process per GPU).

Rank g owns element rows [g s, (g+1) s) (s = n_y / world) and keeps ONE ghost
element row on each side.  Its local arrays are the (p (s + 2), N_x) row window
of the global (N_y, N_x) field; every per-level operator, smoother and
transfer runs UNCHANGED on the local mesh ``MeshConfig(n_x, s + 2, l_x,
dy (s + 2))`` treated as periodic.  Outputs on owned rows are exact because

* ``r = f - A u`` on owned node rows reads u on the ghost element row below
  (p node rows) and on the first node row above -- the forward halo of u;
* the Schwarz correction is computed only for OWNED elements: the ghost
  elements' windows are switched off through the smoother's per-element
  scale 1/nu_bar = 0 (nu_bar = inf on the ghost rows; exact, bitwise the
  unscaled arithmetic elsewhere since 1/1.0 = 1.0).  An owned window reads r
  on n_o rows below the strip and n_o + 1 rows above it (the forward halo of
  r), and its correction lands on n_o ghost rows below and n_o + 1 above:
  those rows start from zero and are sent back to the neighbour that owns
  them, which adds them to its owned rows (the reverse halo);
* restriction of the owned coarse rows reads the fine ghost element row below
  (p rows of r); prolongation of the owned fine rows reads the first coarse
  node row above.

Ghost slabs are contiguous in the row-major layout (no packing).  Inner
products are summed over owned rows on the device (smg_dot / smg_dot2 /
smg_cg_update2 into a device scalar block) and all-reduced in place on the
device -- the host reads ||r|| and the breakdown flag once per cycle, as the
single-GPU solver does.  The singular p = 1 coarse problem is all-gathered
into a preallocated global array and solved redundantly on every rank.

Halo traffic per level of order p and overlap n_o (rows of N_x = p n_x
doubles): u forward p + 1, r forward (2 n_o + 1) + correction reverse
(2 n_o + 1), r forward p before the restriction, 1 coarse row before the
prolongation -- e.g. C3 at p = 32, n_o = 1: 33 + 3 + 3 + 32 rows of 32 KB.
Redundant work: the ghost element rows of the operator and transfer kernels,
2/s of a strip (the masked Schwarz windows still cost their contractions).

The driver is written against two small interfaces so the same code runs
(a) one process per GPU over NCCL -- libsmg's own halo and collective entry
points (``NcclHaloTransport``, smg_halo_* in include/smg.h) or
torch.distributed's (``TorchTransport``), (b) CPU gloo ranks
in the tests with an oracle engine, and (c) several ranks emulated by
threads on one GPU (``ThreadTransport``) for single-device validation.
"""

from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass

import numpy as np

from .metrics import ConvergenceReport

G = 1  # ghost element rows on each side


@dataclass(frozen=True)
class StripPlan:
    n_x: int
    n_y: int
    l_x: float
    l_y: float
    world: int
    rank: int

    def __post_init__(self):
        if self.world < 1 or not 0 <= self.rank < self.world:
            raise ValueError(f"bad rank {self.rank} of {self.world}")
        if self.n_y % self.world:
            raise ValueError(f"{self.n_y} element rows do not split into {self.world} strips")
        if self.n_y // self.world < 1:
            raise ValueError("empty strip")

    @property
    def s(self) -> int:
        return self.n_y // self.world

    @property
    def ey0(self) -> int:
        return self.rank * self.s

    @property
    def local_ny(self) -> int:
        return self.s + 2 * G

    @property
    def dy(self) -> float:
        return self.l_y / self.n_y

    def local_mesh_args(self):
        return (self.n_x, self.local_ny, self.l_x, self.dy * self.local_ny)

    def own(self, p: int) -> slice:
        """Owned node rows in the local array of level p."""
        return slice(G * p, (G + self.s) * p)

    def global_rows(self, p: int) -> np.ndarray:
        """Global node row of every local row of level p (periodic)."""
        N_y = p * self.n_y
        return (np.arange(p * self.local_ny) + (self.ey0 - G) * p) % N_y

    def ghost_mask(self) -> np.ndarray:
        """(local_ny, n_x) bool: element rows whose Schwarz windows are off."""
        m = np.zeros((self.local_ny, self.n_x), dtype=bool)
        m[:G] = True
        m[G + self.s:] = True
        return m

    def check_level(self, p: int, n_o: int):
        """The reverse halo of a strip must not overlap itself."""
        if self.s * p < 2 * n_o + 1:
            raise ValueError(f"strip of {self.s} element rows too thin for p={p}, n_o={n_o}")

    def below(self) -> int:
        return (self.rank - 1) % self.world

    def above(self) -> int:
        return (self.rank + 1) % self.world


# ---------------------------------------------------------------------------
# transports


def _rows(plan, p):
    own = plan.own(p)
    return own.start, own.stop


class TorchTransport:
    """torch.distributed point-to-point + collectives (NCCL on device buffers;
    gloo for CPU tensors, or host-staged when given CUDA tensors)."""

    def __init__(self, plan: StripPlan, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.plan = plan
        self.group = group
        self.host_staged = dist.get_backend(group) != "nccl"

    def _p2p(self, send_down, send_up, recv_from_above, recv_from_below):
        """send_down -> rank below, send_up -> rank above; receive the
        matching messages (fixed op order: deterministic, deadlock-free)."""
        import torch
        dist, pl = self.dist, self.plan
        stage = self.host_staged and send_down.is_cuda
        sd, su = (send_down.cpu(), send_up.cpu()) if stage else (send_down, send_up)
        ra = torch.empty_like(sd) if stage else recv_from_above
        rb = torch.empty_like(su) if stage else recv_from_below
        ops = []
        if sd.numel():
            ops += [dist.P2POp(dist.isend, sd, pl.below(), self.group),
                    dist.P2POp(dist.irecv, ra, pl.above(), self.group)]
        if su.numel():
            ops += [dist.P2POp(dist.isend, su, pl.above(), self.group),
                    dist.P2POp(dist.irecv, rb, pl.below(), self.group)]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if stage:
            recv_from_above.copy_(ra)
            recv_from_below.copy_(rb)

    def exchange(self, t, p: int, below: int, above: int):
        """Forward halo: `below` ghost rows under the strip and `above` over it
        from the neighbours' owned rows."""
        pl = self.plan
        lo, hi = _rows(pl, p)
        if pl.world == 1:
            if above:
                t[hi:hi + above] = t[lo:lo + above]
            if below:
                t[lo - below:lo] = t[hi - below:hi]
            return
        # my bottom `above` rows are the lower neighbour's top ghost rows, and
        # my top `below` rows its upper neighbour's bottom ghost rows
        self._p2p(t[lo:lo + above], t[hi - below:hi], t[hi:hi + above], t[lo - below:lo])

    def exchange_add(self, t, p: int, below: int, above: int):
        """Reverse halo: the contributions in the ghost rows go to the owners,
        which add them to their boundary rows (from below first, then above)."""
        import torch
        pl = self.plan
        lo, hi = _rows(pl, p)
        if pl.world == 1:
            if above:
                t[lo:lo + above] += t[hi:hi + above]
            if below:
                t[hi - below:hi] += t[lo - below:lo]
            return
        from_above = torch.empty_like(t[lo - below:lo])
        from_below = torch.empty_like(t[hi:hi + above])
        self._p2p(t[lo - below:lo], t[hi:hi + above], from_above, from_below)
        if above:
            t[lo:lo + above] += from_below
        if below:
            t[hi - below:hi] += from_above

    def allreduce_(self, x):
        """In-place sum of a (device) tensor over the ranks."""
        if self.plan.world == 1:
            return x
        if self.host_staged and x.is_cuda:
            h = x.cpu()
            self.dist.all_reduce(h, group=self.group)
            x.copy_(h)
        else:
            self.dist.all_reduce(x, group=self.group)
        return x

    def allgather_rows(self, own, full):
        """full (N_y, N_x) <- every rank's owned rows `own`, in rank order,
        gathered straight into the preallocated array."""
        if self.plan.world == 1:
            full.copy_(own)
            return
        src = own.contiguous()
        if self.host_staged and src.is_cuda:
            import torch
            parts = [torch.empty_like(src.cpu()) for _ in range(self.plan.world)]
            self.dist.all_gather(parts, src.cpu(), group=self.group)
            full.copy_(torch.cat(parts, 0))
        elif src.is_cuda:
            self.dist.all_gather_into_tensor(full, src, group=self.group)
        else:
            parts = list(full.chunk(self.plan.world, 0))
            self.dist.all_gather(parts, src, group=self.group)


class NcclHaloTransport:
    """The strip halos and collectives through libsmg's own NCCL entry points
    (``smg_halo_*``, include/smg.h): device buffers, the caller's stream, no
    host round trip -- a strip V-cycle with its halos captures into one CUDA
    graph.  The communicator id is drawn by rank 0 and broadcast over the
    torch.distributed group (any backend); one rank needs no process group
    and exchanges with itself (NCCL self send/recv).  Same semantics and the
    same fixed addition order as ``TorchTransport``."""

    def __init__(self, plan: StripPlan, group=None, device=None):
        import ctypes as C
        import torch
        from . import _native as NV
        self.plan = plan
        self.NV = NV
        lib = NV.lib()
        if not lib.smg_halo_available():
            raise RuntimeError("smg_halo: NCCL could not be loaded")
        uid = C.create_string_buffer(128)
        if plan.rank == 0:
            NV.check(lib.smg_halo_unique_id(uid, 128), "smg_halo_unique_id")
        raw = uid.raw
        if plan.world > 1:
            import torch.distributed as dist
            box = [raw if plan.rank == 0 else None]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(box, src=src, group=group)
            raw = box[0]
        self.device = torch.cuda.current_device() if device is None else int(device)
        h = C.c_void_p()
        NV.check(lib.smg_halo_create(raw, 128, plan.world, plan.rank, self.device, C.byref(h)), "smg_halo_create")
        self.h = h
        self._ws = {}

    def close(self):
        """Destroy the communicator.  Release every CUDA graph that captured
        this transport's calls first (StripSolver.release_graph): NCCL keeps
        captured work alive and ncclCommDestroy waits for it."""
        if self.h is not None and self.h.value:
            self.NV.check(self.NV.lib().smg_halo_destroy(self.h), "smg_halo_destroy")
        self.h = None

    @staticmethod
    def _field(t):
        if t.dim() != 2 or not t.is_contiguous() or not t.is_cuda:
            raise ValueError("halo fields are contiguous 2-D device arrays")
        return t.shape[1]

    def exchange(self, t, p: int, below: int, above: int):
        lo, hi = _rows(self.plan, p)
        NV = self.NV
        NV.check(NV.lib().smg_halo_exchange(self.h, t.data_ptr(), t.shape[0], self._field(t), lo, hi, below, above,
                                            NV.stream()), "smg_halo_exchange")

    def exchange_add(self, t, p: int, below: int, above: int):
        import torch
        lo, hi = _rows(self.plan, p)
        NV = self.NV
        row_len = self._field(t)
        key = (row_len, below, above)
        ws = self._ws.get(key)
        if ws is None:
            ws = self._ws[key] = torch.empty(max(1, NV.lib().smg_halo_ws_doubles(*key)), dtype=torch.float64,
                                             device=t.device)
        NV.check(NV.lib().smg_halo_exchange_add(self.h, t.data_ptr(), t.shape[0], row_len, lo, hi, below, above,
                                                ws.data_ptr(), NV.stream()), "smg_halo_exchange_add")

    def allreduce_(self, x):
        if not x.is_contiguous():
            raise ValueError("allreduce_ needs a contiguous tensor")
        NV = self.NV
        NV.check(NV.lib().smg_halo_allreduce(self.h, x.data_ptr(), x.numel(), NV.stream()), "smg_halo_allreduce")
        return x

    def allgather_rows(self, own, full):
        if not own.is_contiguous() or not full.is_contiguous() or full.numel() != own.numel() * self.plan.world:
            raise ValueError("allgather_rows: contiguous own rows and a (world x own) full array")
        NV = self.NV
        NV.check(NV.lib().smg_halo_allgather(self.h, own.data_ptr(), full.data_ptr(), own.numel(), NV.stream()),
                 "smg_halo_allgather")


def make_transport(plan: StripPlan, group=None):
    """The transport for a GPU strip solver: libsmg's NCCL halos
    (``NcclHaloTransport``) unless SMG_HALO=torch selects torch.distributed's
    point-to-point (``TorchTransport``; also the choice for non-NCCL groups)."""
    import os
    choice = os.environ.get("SMG_HALO", "nccl")
    if choice == "torch":
        return TorchTransport(plan, group)
    if choice != "nccl":
        raise ValueError(f"SMG_HALO must be 'nccl' or 'torch', not {choice!r}")
    if plan.world > 1:
        import torch.distributed as dist
        if dist.get_backend(group) != "nccl":
            return TorchTransport(plan, group)
    return NcclHaloTransport(plan, group)


class ThreadTransport:
    """Several ranks emulated by threads of one process (one GPU): exchanges
    are device copies between the ranks' arrays between barriers."""

    def __init__(self, plan: StripPlan, shared):
        self.plan = plan
        self.sh = shared  # dict with 'barrier', 'slots'

    def _sync(self):
        import torch
        torch.cuda.synchronize()
        self.sh["barrier"].wait()

    def _neighbours(self, t):
        self.sh["slots"][self.plan.rank] = t
        self._sync()
        return self.sh["slots"][self.plan.below()], self.sh["slots"][self.plan.above()]

    def exchange(self, t, p: int, below: int, above: int):
        lo, hi = _rows(self.plan, p)
        bel, abv = self._neighbours(t)
        top = abv[lo:lo + above].clone()
        bot = bel[hi - below:hi].clone()
        self._sync()
        t[hi:hi + above] = top
        t[lo - below:lo] = bot
        self._sync()

    def exchange_add(self, t, p: int, below: int, above: int):
        lo, hi = _rows(self.plan, p)
        bel, abv = self._neighbours(t)
        from_below = bel[hi:hi + above].clone()
        from_above = abv[lo - below:lo].clone()
        self._sync()
        if above:
            t[lo:lo + above] += from_below
        if below:
            t[hi - below:hi] += from_above
        self._sync()

    def allreduce_(self, x):
        import torch
        self.sh["slots"][self.plan.rank] = x.clone()
        self._sync()
        parts = [self.sh["slots"][r] for r in range(self.plan.world)]
        acc = parts[0].clone()
        for q in parts[1:]:
            acc += q.to(acc.device)
        self._sync()
        x.copy_(acc)
        return x

    def allgather_rows(self, own, full):
        import torch
        self.sh["slots"][self.plan.rank] = own
        self._sync()
        parts = [self.sh["slots"][r] for r in range(self.plan.world)]
        full.copy_(torch.cat(parts, 0))
        self._sync()


def run_threads(world: int, fn):
    """Run fn(rank, shared) on `world` threads (emulated ranks); returns results."""
    shared = {"barrier": threading.Barrier(world), "slots": [None] * world}
    out = [None] * world
    err = []

    def body(r):
        try:
            out[r] = fn(r, shared)
        except BaseException as e:  # surface the first failure
            err.append(e)
            shared["barrier"].abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


# ---------------------------------------------------------------------------
# the strip-parallel algorithm (engine-agnostic)


class StripSolver:
    """V-cycle, MG and MGCG on one rank's strip.

    ``engine`` provides, per level l (0 = p=1 coarse), on LOCAL arrays:
      orders, n_o, n_pre, n_post        per-level lists
      us, fs                            per-level solution / right-hand side
      zeros(l), work(l), clone(a), copy(dst, src), fill_zero(a)
      residual(l, u, f, out)            out = f - A u     (f None: out = A u)
      correct(l, r, u, zero)            u += M r (zero: u := M r), ghost windows off
      restrict(l, fine, out)            out (level l-1) = P^T fine
      prolong_add(l, coarse, fine)
      coarse_local(f0_full, u0)         global p=1 solve, the rank's rows into u0
      full0                             preallocated global p=1 array
      scalars()                         (scal[8], flag) device block
      dot(a, b, out)                    out[0] = a . b   (owned slices)
      dot2(z, r, r_old, out)            out[0] = z.(r - r_old), out[1] = z.r
      cg_update(u, r, r_new, d, q, scal, flag)   krylov.py:95-103 on owned slices
      cg_beta_finish(scal), cg_direction(d, z, scal)
      read(scal, flag) -> (host floats, int)    the per-cycle sync
    """

    def __init__(self, plan: StripPlan, engine, transport):
        self.plan, self.eng, self.tr = plan, engine, transport
        self.L = len(engine.orders) - 1
        for l in range(1, self.L + 1):
            plan.check_level(engine.orders[l], engine.n_o[l])

    def own(self, l):
        return self.plan.own(self.eng.orders[l])

    # -- halos per stage (rows below, rows above)
    def _residual(self, l, u, f, out):
        p = self.eng.orders[l]
        self.tr.exchange(u, p, p, 1)
        self.eng.residual(l, u, f, out)

    def _correct(self, l, r, u, zero):
        e, p = self.eng, self.eng.orders[l]
        n_o = e.n_o[l]
        self.tr.exchange(r, p, n_o, n_o + 1)
        if not zero:
            own = self.own(l)
            u[:own.start] = 0.0
            u[own.stop:] = 0.0
        e.correct(l, r, u, zero)
        self.tr.exchange_add(u, p, n_o, n_o + 1)

    def _smooth(self, l, u, f, n_it, zero):
        for it in range(n_it):
            if zero and it == 0:
                self._correct(l, f, u, True)
            else:
                r = self.eng.work(l)
                self._residual(l, u, f, r)
                self._correct(l, r, u, False)

    def v_cycle(self, u, f, u_zero=False):
        """Algorithm 3 (multigrid.py:231-251) on the strip; u updated in place."""
        e = self.eng
        L = self.L
        us, fs = e.us, e.fs
        us[L], fs[L] = u, f
        for l in range(L, 0, -1):
            p = e.orders[l]
            zero = u_zero if l == L else True
            if e.n_pre[l]:
                self._smooth(l, us[l], fs[l], e.n_pre[l], zero)
                zero = False
            elif zero:
                e.fill_zero(us[l])
            r = e.work(l)
            if zero:
                e.copy(r, fs[l])
            else:
                self._residual(l, us[l], fs[l], r)
            self.tr.exchange(r, p, p, 0)
            e.restrict(l, r, fs[l - 1])
        # replicated coarse solve
        f0_full = e.full0
        self.tr.allgather_rows(fs[0][self.own(0)], f0_full)
        e.coarse_local(f0_full, us[0])
        for l in range(1, L + 1):
            self.tr.exchange(us[l - 1], e.orders[l - 1], 0, 1)
            e.prolong_add(l, us[l - 1], us[l])
            if e.n_post[l]:
                self._smooth(l, us[l], fs[l], e.n_post[l], False)
        return u

    def v_cycle_graph(self, u, f):
        """The strip V-cycle captured once as a CUDA graph for fixed (u, f)
        buffers and replayed (opt-in: the NCCL point-to-point and all-gather
        are captured with it -- validated on one GPU only, with the world-1
        transport, since the pool has one GPU per call)."""
        import torch
        key = (u.data_ptr(), f.data_ptr())
        if getattr(self, "_graph_key", None) != key:
            self.v_cycle(u, f)                      # this call's cycle, eagerly (sets kernel attributes)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):  # recorded, not executed
                self.v_cycle(u, f)
            torch.cuda.current_stream().wait_stream(side)
            self._graph, self._graph_key = g, key
            return u
        self._graph.replay()
        return u

    def release_graph(self):
        """Drop the captured V-cycle graph (before closing an NCCL transport)."""
        import torch
        torch.cuda.synchronize()
        self._graph, self._graph_key = None, None

    def solve_mg(self, f, u, tol=1e10, max_cycles=200):
        """krylov.py:49-67 on strips; f, u local (u = initial guess, updated)."""
        t0 = time.perf_counter()
        e, L = self.eng, self.L
        o = self.own(L)
        r = e.zeros(L)
        scal, flag = e.scalars()

        def norm():
            self._residual(L, u, f, r)
            e.dot(r[o], r[o], scal[2:3])
            self.tr.allreduce_(scal[2:3])
            host, _ = e.read(scal, flag)
            return math.sqrt(host[2])

        res = [norm()]
        r_max = res[0] / tol
        ok = res[0] <= r_max
        cycles = 0
        while not ok and cycles < max_cycles:
            self.v_cycle(u, f)
            cycles += 1
            res.append(norm())
            ok = res[-1] <= r_max
        return u, ConvergenceReport(res, ok, cycles, time.perf_counter() - t0)

    def solve_mgcg(self, f, u, tol=1e10, max_cycles=200):
        """krylov.py:70-115 on strips (beta = z^T (r - r_old) / delta as coded),
        every scalar on the device: scal[0] delta, [1] p.q, [2] ||r||^2,
        [3:5] the dot2 sums, [5] beta, [6] alpha."""
        t0 = time.perf_counter()
        e, L = self.eng, self.L
        o = self.own(L)
        scal, flag = e.scalars()
        tr = self.tr
        r = e.zeros(L)
        self._residual(L, u, f, r)
        e.dot(r[o], r[o], scal[2:3])
        tr.allreduce_(scal[2:3])
        host, _ = e.read(scal, flag)
        res = [math.sqrt(host[2])]
        r_max = res[0] / tol
        ok = res[0] <= r_max
        broke = False
        cycles = 0
        if not ok:
            d = e.zeros(L)
            q = e.zeros(L)
            z = e.zeros(L)
            r_new = e.zeros(L)
            self.v_cycle(d, e.clone(r), u_zero=True)
            e.dot(d[o], r[o], scal[0:1])
            tr.allreduce_(scal[0:1])
            first = True
            for _ in range(max_cycles):
                self._residual(L, d, None, q)
                e.dot(d[o], q[o], scal[1:2])
                tr.allreduce_(scal[1:2])
                e.cg_update(u[o], r[o], r_new[o], d[o], q[o], scal, flag)
                tr.allreduce_(scal[2:3])
                host, brk = e.read(scal, flag)
                if brk:
                    broke = True
                    break
                cycles += 1
                res.append(math.sqrt(host[2]))
                if res[-1] <= r_max:
                    ok = True
                    break
                self.v_cycle(z, e.clone(r_new), u_zero=True)
                e.dot2(z[o], r_new[o], None if first else r[o], scal[3:5])
                tr.allreduce_(scal[3:5])
                e.cg_beta_finish(scal)
                e.cg_direction(d[o], z[o], scal)
                r, r_new = r_new, r
                first = False
        rep = ConvergenceReport(res, ok, cycles, time.perf_counter() - t0)
        rep.breakdown = broke
        return u, rep


# ---------------------------------------------------------------------------
# GPU engine: the library's kernels on the local mesh


class GpuEngine:
    """Per-level device handles built on the rank's local (strip + ghosts)
    mesh, the Schwarz windows of the ghost element rows switched off."""

    def __init__(self, plan: StripPlan, p: int, rule, kind="w5", n_pre=1, n_post=0, orders=None,
                 nu_hat=None, nu_shift=0.2, coarse=None, coarse_tol=1e-12):
        import torch
        from . import _native as N
        from .mesh import MeshConfig
        from .schwarz import WeightKind
        self.torch = torch
        self.N = N
        self.plan = plan
        lm = MeshConfig(*plan.local_mesh_args())
        gm = MeshConfig(plan.n_x, plan.n_y, plan.l_x, plan.l_y)
        kind = WeightKind(kind) if isinstance(kind, str) else kind
        self.h = _local_hierarchy(plan, lm, gm, p, rule, kind, n_pre, n_post, orders, nu_hat, nu_shift,
                                  coarse_tol)
        levels = self.h.levels
        self.orders = [lv.basis.p for lv in levels]
        self.n_o = [lv.n_o for lv in levels]
        self.n_pre = [lv.n_pre for lv in levels]
        self.n_post = [lv.n_post for lv in levels]
        self.us = [lv.u for lv in levels]
        self.fs = [lv.f for lv in levels]
        self._work = [lv.work for lv in levels]
        # global p=1 coarse problem, replicated on every rank
        self.hc = _coarse_only(gm, nu_hat, nu_shift, coarse, coarse_tol)
        self.full0 = torch.zeros((plan.n_y, plan.n_x), dtype=torch.float64, device="cuda")
        self.u0_full = torch.zeros_like(self.full0)
        self.rows0 = torch.as_tensor(plan.global_rows(self.orders[0]), dtype=torch.long, device="cuda")
        self.ws = torch.zeros(N.lib().smg_reduce_ws_doubles(), dtype=torch.float64, device="cuda")
        self._scal = torch.zeros(8, dtype=torch.float64, device="cuda")
        self._flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._hscal = torch.zeros(8, dtype=torch.float64).pin_memory()
        self._hflag = torch.zeros(1, dtype=torch.int32).pin_memory()

    def zeros(self, l):
        return self.torch.zeros(self.h.levels[l].op.layout.shape, dtype=self.torch.float64, device="cuda")

    def work(self, l):
        return self._work[l]

    def clone(self, a):
        return a.clone()

    def copy(self, dst, src):
        dst.copy_(src)

    def fill_zero(self, a):
        a.zero_()

    def residual(self, l, u, f, out):
        self.h.levels[l].op.residual_into(u, f, out)

    def correct(self, l, r, u, zero):
        N = self.N
        lv = self.h.levels[l]
        if zero:
            rc = N.lib().smg_schwarz_smooth(lv.smoother._h.raw, lv.op._handle.raw, N.ptr(u), N.ptr(r),
                                            N.ptr(self._work[l]), N.ptr(lv.smoother.ring), 1, 1, N.stream())
        else:
            rc = N.lib().smg_schwarz_correct(lv.smoother._h.raw, N.ptr(r), N.ptr(u), N.ptr(lv.smoother.ring),
                                             N.stream())
        N.check(rc, "strip correct")

    def restrict(self, l, fine, out):
        N = self.N
        tr = self.h.levels[l].transfer
        N.check(N.lib().smg_restrict_ws(tr.handle.raw, N.ptr(fine), N.ptr(out), tr.ws_ptr(), N.stream()),
                "strip restrict")

    def prolong_add(self, l, coarse, fine):
        N = self.N
        N.check(N.lib().smg_prolongate(self.h.levels[l].transfer.handle.raw, N.ptr(coarse), N.ptr(fine), 1,
                                       N.stream()), "strip prolong")

    def coarse_local(self, f0_full, u0):
        """The replicated global p=1 solve into preallocated buffers (graph-
        capturable for the pseudo-inverse), the rank's rows gathered by a
        device index."""
        from .multigrid import _coarse_into
        _coarse_into(self.hc, f0_full, self.u0_full)
        self.torch.index_select(self.u0_full, 0, self.rows0, out=u0)

    # -- BLAS-1 on owned slices, device scalars
    def scalars(self):
        self._scal.zero_()
        self._flag.zero_()
        return self._scal, self._flag

    def dot(self, a, b, out):
        N = self.N
        N.check(N.lib().smg_dot(N.ptr(a), N.ptr(b), a.numel(), N.ptr(out), N.ptr(self.ws), N.stream()), "strip dot")

    def dot2(self, z, r, r_old, out):
        N = self.N
        N.check(N.lib().smg_dot2(N.ptr(z), N.ptr(r), N.ptr(r_old) if r_old is not None else None, z.numel(),
                                 N.ptr(out), N.ptr(self.ws), N.stream()), "strip dot2")

    def cg_update(self, u, r, r_new, d, q, scal, flag):
        N = self.N
        N.check(N.lib().smg_cg_update2(N.ptr(u), N.ptr(r), N.ptr(r_new), N.ptr(d), N.ptr(q), u.numel(), N.ptr(scal),
                                       N.ptr(flag), N.ptr(self.ws), N.stream()), "strip cg_update")

    def cg_beta_finish(self, scal):
        N = self.N
        N.check(N.lib().smg_cg_beta_finish(N.ptr(scal), N.stream()), "strip cg_beta_finish")

    def cg_direction(self, d, z, scal):
        N = self.N
        N.check(N.lib().smg_cg_direction(N.ptr(d), N.ptr(z), d.numel(), N.ptr(scal), N.stream()),
                "strip cg_direction")

    def read(self, scal, flag):
        self._hscal.copy_(scal, non_blocking=True)
        self._hflag.copy_(flag, non_blocking=True)
        self.torch.cuda.current_stream().synchronize()
        return [float(v) for v in self._hscal], int(self._hflag[0])


def _local_hierarchy(plan, lm, gm, p, rule, kind, n_pre, n_post, orders, nu_hat, nu_shift, coarse_tol):
    """The rank's levels on the local mesh: operators (nu sampled at GLOBAL
    coordinates for diffusion), transfers, and smoothers whose ghost-row
    windows are off (nu_bar = inf there)."""
    import torch
    from . import multigrid as MG
    from .basis import gll_basis, interp_matrix
    from .mesh import layout_for
    from .operators import DiffusionOperator, PoissonOperator, diffusivity_field
    from .schwarz import AdditiveSchwarz
    if orders is None:
        if p < 2 or (p & (p - 1)) != 0:
            raise ValueError(f"top-level order must be a power of two >= 2, got {p}")
        orders = [1 << l for l in range(p.bit_length())]
    ghost = plan.ghost_mask()
    levels = []
    for l, p_l in enumerate(orders):
        b = gll_basis(p_l)
        if nu_hat is None:
            op = PoissonOperator(b, lm)
            nb = np.ones((plan.local_ny, plan.n_x))
        else:
            nu_l = diffusivity_field(gm, b, nu_hat, nu_shift)[plan.global_rows(p_l)]
            op = DiffusionOperator(b, lm, nu_l)
            nb = np.array(op.element_mean_nu(), dtype=np.float64)
        nb = np.where(ghost, np.inf, nb)
        lay = layout_for(lm, p_l)
        if l == 0:
            lv = MG.Level(l, b, op, None, 0, 0, 0)
        else:
            n_o = rule.layers(p_l)
            sm = AdditiveSchwarz(b, lay, lm.dx, lm.dy, n_o, kind, nu_bar=nb)
            lv = MG.Level(l, b, op, sm, n_pre, n_post, n_o)
            lv.transfer = MG._Transfer(orders[l - 1], p_l, lm.n_x, lm.n_y, interp_matrix(levels[-1].basis, b).matrix)
        lv.u = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
        lv.f = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
        lv.work = torch.zeros(lay.shape, dtype=torch.float64, device="cuda")
        levels.append(lv)
    return MG.MultigridHierarchy(lm, levels, coarse_tol=coarse_tol, coarse="cg")


def _coarse_only(gm, nu_hat, nu_shift, coarse, coarse_tol):
    """A hierarchy holding only the global p=1 level (for coarse_solve)."""
    import torch
    from . import multigrid as MG
    from .basis import gll_basis
    from .operators import DiffusionOperator, PoissonOperator, diffusivity_field
    b = gll_basis(1)
    op = PoissonOperator(b, gm) if nu_hat is None else DiffusionOperator(b, gm, diffusivity_field(gm, b, nu_hat, nu_shift))
    lv = MG.Level(0, b, op, None, 0, 0, 0)
    lv.u = torch.zeros(op.layout.shape, dtype=torch.float64, device="cuda")
    lv.f = torch.zeros(op.layout.shape, dtype=torch.float64, device="cuda")
    if coarse is None:
        coarse = "pinv" if nu_hat is None else "pcg"
    return MG.MultigridHierarchy(gm, [lv], coarse_tol=coarse_tol, coarse=coarse)


def local_window(plan: StripPlan, full, p: int):
    """The rank's local (strip + ghosts) rows of a global level-p array."""
    return full[plan.global_rows(p)]
