"""Benchmark: weighted-Schwarz smoother + p-multigrid V-cycle DOF/s on B200.

Workload (BASELINE.json configs[1], "C2"): periodic Poisson on [0,1]^2,
64x64 elements, p = 16 (1,048,576 DOF), FP64, f = N(0,1) from seed 0 with
the mean removed, weighted additive Schwarz (w5, fixed:1 overlap), V-cycle
with one pre-smoothing and no post-smoothing, coarse p=1 pseudo-inverse.
A step is one V-cycle u <- V(u, f) of the stand-alone MG iteration (full
work: the top level applies A to a nonzero u).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Timing: CUDA events on the launching stream around each step, L2 flushed
(256 MiB write) before every timed step, K steps bracketed by barrier +
synchronize, max over ranks.  N > 1 (torchrun, one process per GPU): BASELINE
configs[2] (C3: 128x128 elements, p = 32, 16.8M DOF) STRONG-scaled over
element-row strips (paper_1512_02390_b200/strips.py: 128/N element rows per
rank, NCCL halo send/recv on device buffers, device-side dot products
all-reduced by NCCL, replicated coarse solve), plus one C4 MGCG solve; the
N = 1 line carries the single-GPU C3 V-cycle as the strong-scaling reference.

--impl reference times the UNMODIFIED reference package (pip-installed into
baseline/_ref from /root/reference, pure Python + NumPy/OpenBLAS on every host
core) through its own v_cycle on the same C2 workload; if baseline/_ref is
missing it falls back to the numpy restatement in oracle/ and says so.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(n_x=64, n_y=64, l_x=1.0, l_y=1.0, p=16, rule="fixed:1", seed=0)
C3 = dict(n_x=128, n_y=128, l_x=1.0, l_y=1.0, p=32, rule="fixed:1", seed=0)
C4 = dict(n_x=256, n_y=256, l_x=8.0, l_y=1.0, p=16, rule="fixed:1", seed=0)
# one workload string for both arms (the driver compares the config of the two lines)
WORKLOAD_C2 = ("C2: periodic Poisson [0,1]^2, 64x64 elements, p=16 (1,048,576 DOF), stand-alone V-cycle "
               "(1 pre-, 0 post-smoothing), w5, fixed:1")
WORKLOAD_C3 = ("C3: periodic Poisson [0,1]^2, 128x128 elements, p=32 (16,777,216 DOF), V-cycle (1,0), w5, "
               "fixed:1, element-row strips")
METRIC = "weighted-Schwarz smoother + V-cycle DOF/s, fraction of FP64/HBM roofline"
FP64_PEAK_TFLOPS = 37.15   # measured: DMMA m8n8k4 on this pool's B200 (tools/peaks, profiles/fp64_peaks.txt)
FP64_DFMA_TFLOPS = 34.2    # measured: DFMA register-operand peak


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def fd_flops_per_element(m: int) -> float:
    """Dense FD as executed by schwarz.py:217-221: 4 contractions + scaling + weight."""
    return 8.0 * m ** 3 + 3.0 * m ** 2


def fd_eo_flops_per_element(m: int) -> float:
    """Even/odd FD as executed by fdt_kernel (declare and report against
    this): 4 contractions as two half-size ones each, 2 flops per FMA, + the
    1/(lam_y+lam_x) scaling (the weight is folded into the synthesis factors)."""
    he, ho = (m + 1) // 2, m // 2
    return 8.0 * m * (he * he + ho * ho) + m * m


def load_traffic():
    """ncu dram__bytes_{read,write}.sum per launch of the C2 top-level kernels,
    written by tools/ncu_traffic.py from one `ncu --set full` capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_c2.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def roofline_entry(name, t, flops, bytes_, p64, bw, traffic=None, note=None):
    """Roofline of one kernel (call): bound = the larger of flops/P64 and bytes/BW."""
    t_f, t_b = flops / p64, bytes_ / bw
    if t_b >= t_f:
        ent = {"bound": "hbm", "achieved": bytes_ / t / 1e9, "peak": bw / 1e9, "unit": "GB/s"}
    else:
        ent = {"bound": "tensor", "pipe": "fp64", "achieved": flops / t / 1e12, "peak": p64 / 1e12,
               "unit": "TFLOP/s"}
    ent["frac"] = ent["achieved"] / ent["peak"]
    ent.update({"kernel": name, "us_per_call": 1e6 * t, "algorithmic_flops": flops, "algorithmic_bytes": bytes_,
                "t_roof_us": 1e6 * max(t_f, t_b), "traffic": traffic})
    if note:
        ent["note"] = note
    return ent


def vcycle_roofline_seconds(n_x, n_y, orders, n_o_of, p64, bw):
    """sum over levels l >= 1 of max(F/P64, B/BW) for the sweep,
    the residual+restriction and the prolongation (coarse solve excluded)."""
    t = 0.0
    n_el = n_x * n_y
    for l in range(1, len(orders)):
        p, pc = orders[l], orders[l - 1]
        N, Nc = p * p * n_el, pc * pc * n_el
        m = p + 1 + 2 * n_o_of(p)
        npp = p + 1
        f_apply = n_el * (4 * npp ** 3 + 3 * npp ** 2) + N
        top = l == len(orders) - 1
        # sweep: residual (top level only; lower levels start from zero) + FD
        if top:
            t += max(f_apply / p64, 24.0 * N / bw)
        t += max(n_el * fd_eo_flops_per_element(m) / p64, 24.0 * N / bw)
        # residual + restriction, prolongation
        t += max(f_apply / p64, 24.0 * N / bw)
        f_tr = 2.0 * n_el * ((p + 1) * (pc + 1) ** 2 + (p + 1) ** 2 * (pc + 1))
        t += max(f_tr / p64, (8.0 * N + 8.0 * Nc) / bw)
        t += max(f_tr / p64, (16.0 * N + 8.0 * Nc) / bw)
    return t


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    polled every ~0.5 ms from a thread (the timed region is only milliseconds
    long), nvidia-smi as the fallback."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.rows = []   # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            hd = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(hd, pynvml.NVML_CLOCK_SM)
            why = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def sample():
                return (pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM), mx, why(hd))
        except Exception:
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active")

            def sample():
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip().split(",")
                return float(out[0]), float(out[1]), int(out[2].strip(), 16)

        def run():
            while not self._stop.is_set():
                try:
                    self.rows.append(sample())
                except Exception:
                    pass
                self._stop.wait(0.0005)
        self.rows.append(sample())
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(r[0]) for r in self.rows]
        reasons = sorted({nm for r in self.rows for nm, bit in self.REASONS.items() if int(r[2]) & bit})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(float(r[1]) for r in self.rows) if self.rows else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = [i for i in threadpool_info() if i.get("internal_api") in ("openblas", "mkl", "blis")]
        if info:
            return int(info[0]["num_threads"])
    except Exception:
        pass
    return os.cpu_count() or 1


def oracle_problem():
    from oracle import smg_oracle as O
    c = CFG
    h = O.Hierarchy(c["n_x"], c["n_y"], c["l_x"], c["l_y"], c["p"], rule=c["rule"])
    N = (c["p"] * c["n_y"], c["p"] * c["n_x"])
    f = O.project_mean(np.random.default_rng(c["seed"]).standard_normal(N))
    return O, h, f


def reference_problem():
    """The unmodified reference (baseline/_ref, pip-installed from
    /root/reference) on the C2 workload, or None when it is not installed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "schwarzmg")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from schwarzmg import mesh, multigrid, operators
    except Exception:
        return None
    c = CFG
    msh = mesh.MeshConfig(c["n_x"], c["n_y"], c["l_x"], c["l_y"])
    h = multigrid.build_hierarchy(msh, c["p"], multigrid.OverlapRule.parse(c["rule"]))
    N = (c["p"] * c["n_y"], c["p"] * c["n_x"])
    f = operators.project_mean(np.random.default_rng(c["seed"]).standard_normal(N))
    return multigrid.v_cycle, h, f


def time_cpu_vcycles(budget_s: float, max_steps: int | None = None, warmup: int = 0):
    """The reference's own v_cycle (multigrid.py:231-251) from baseline/_ref on
    all host threads; the oracle port if the reference is not installed.
    Returns (per-step seconds, DOF, kind)."""
    rp = reference_problem()
    if rp is not None:
        vcyc, h, f = rp
        kind = "reference"
    else:
        O, h, f = oracle_problem()
        vcyc = O.v_cycle
        kind = "port"
    u = np.zeros_like(f)
    for _ in range(warmup):
        u = vcyc(h, u, f)
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        u = vcyc(h, u, f)
        times.append(time.perf_counter() - t0)
        if max_steps is not None and len(times) >= max_steps:
            break
        if max_steps is None and time.perf_counter() - t_start > budget_s:
            break
    return times, f.size, kind


def _cpu_sample(kind, n):
    if kind == "reference":
        return (f"{n} C2 V-cycles of the unmodified reference (schwarzmg.multigrid.v_cycle from baseline/_ref, "
                "coarse plain CG as the reference does), NumPy/OpenBLAS on every host core")
    return (f"{n} C2 V-cycles of the numpy restatement (oracle/smg_oracle.py; baseline/_ref not installed)")


def run_reference(args):
    times, ndof, kind = time_cpu_vcycles(0.0, max_steps=args.steps, warmup=min(args.warmup, 3))
    t = float(np.sum(times))
    value = ndof * len(times) / t
    cores = cpu_threads()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": args.gpus,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * t / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N(0,1) RHS, mean removed)",
            "config": {"workload": WORKLOAD_C2, "coarse": "plain CG to 1e-12 (the reference's)",
                       "parallelism": "cpu"},
            "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": cores, "kind": kind,
                             "sample": _cpu_sample(kind, len(times))},
            "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


_JSON_OUT = None


def _claim_stdout():
    """Keep stdout for the one JSON line: native libraries (NCCL prints its
    version banner on fd 1) write to stderr from here on."""
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _strip_setup(cfg, world, rank, dev):
    import torch
    import paper_1512_02390_b200 as P
    from paper_1512_02390_b200.strips import GpuEngine, StripPlan, StripSolver, make_transport
    plan = StripPlan(cfg["n_x"], cfg["n_y"], cfg["l_x"], cfg["l_y"], world, rank)
    eng = GpuEngine(plan, cfg["p"], P.OverlapRule.parse(cfg["rule"]))
    sol = StripSolver(plan, eng, make_transport(plan))
    p = cfg["p"]
    N = (p * cfg["n_y"], p * cfg["n_x"])
    f_host = P.project_mean(np.random.default_rng(cfg["seed"]).standard_normal(N))
    rows = plan.global_rows(p)
    f = torch.from_numpy(f_host[rows].copy()).to(dev)
    return plan, sol, f, f_host, rows, N


def run_strips(args, world, rank, local, dev):
    """N > 1: BASELINE configs[2] (C3, 128x128 elements, p = 32) STRONG-scaled
    over element-row strips (strips.py): 128/N element rows per rank, one ghost
    element row each side, NCCL halo send/recv on device buffers, replicated
    coarse pseudo-inverse.  A step is one V-cycle of the MG iteration.  Then
    one C4 MGCG solve on the same ranks (device dots all-reduced by NCCL)."""
    import torch
    import torch.distributed as dist
    from paper_1512_02390_b200 import _native as NV

    lib = NV.lib()
    plan, sol, f, f_host, rows, N = _strip_setup(C3, world, rank, dev)
    own = plan.own(C3["p"])
    ndof = N[0] * N[1]
    u = torch.zeros_like(f)
    sol.v_cycle(u, f)
    torch.cuda.synchronize()
    n0 = lib.smg_launch_count()
    sol.v_cycle(u, f)
    torch.cuda.synchronize()
    launches_per_step = lib.smg_launch_count() - n0
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    # replay the strip V-cycle (NCCL halos and all-gather included) as one
    # captured CUDA graph: the default with libsmg's own halos (smg_halo_*,
    # every call on the compute stream; the capture is tested on one GPU through
    # NCCL self send/recv, tests/test_gpu_halo.py); SMG_STRIP_GRAPH=0/1 overrides
    from paper_1512_02390_b200.strips import NcclHaloTransport
    native = isinstance(sol.tr, NcclHaloTransport)
    use_graph = os.environ.get("SMG_STRIP_GRAPH", "1" if native else "0") == "1"
    step = (lambda: sol.v_cycle_graph(u, f)) if use_graph else (lambda: sol.v_cycle(u, f))
    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    dist.barrier()
    torch.cuda.synchronize()
    t_steps = 0.0
    for _ in range(args.steps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        t_steps += a.elapsed_time(b) / 1e3
    dist.barrier()
    clocks = sampler.stop()
    tt = torch.tensor([t_steps], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_steps = float(tt.item())
    # end to end: the rank's rows of f from pinned host, its owned rows of u back
    f_pin = torch.from_numpy(f_host[rows].copy()).pin_memory()
    u_pin = torch.empty(f.shape, dtype=torch.float64).pin_memory()
    dist.barrier()
    t_e2e = 0.0
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f.copy_(f_pin, non_blocking=True)
        sol.v_cycle(u, f)
        u_pin[own].copy_(u[own], non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        t_e2e += a.elapsed_time(b) / 1e3
    tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_e2e = float(tt.item())
    # C4 MGCG on the same ranks (time to solution, max over ranks)
    c4 = None
    if not args.no_c4:
        plan4, sol4, f4, _, _, N4 = _strip_setup(C4, world, rank, dev)
        sol4.solve_mgcg(f4.clone(), torch.zeros_like(f4), max_cycles=2)   # warm-up (handles, attributes)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rep = sol4.solve_mgcg(f4.clone(), torch.zeros_like(f4))
        torch.cuda.synchronize()
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        c4 = {"workload": "C4: [0,8]x[0,1], 256x256 elements (AR 8), p=16 (16,777,216 DOF), MGCG to 1e10",
              "cycles": rep.cycles, "converged": rep.converged, "breakdown": rep.breakdown,
              "rbar": rep.rbar, "time_to_solution_s": float(tt.item()),
              "dof_cycles_per_s": N4[0] * N4[1] * rep.cycles / float(tt.item()),
              "timing": "host wall clock around solve_mgcg (one sync per cycle for the convergence test), "
                        "max over ranks"}
    if rank == 0:
        own_bytes = 8 * (own.stop - own.start) * N[1]
        line = {"metric": METRIC, "value": ndof * args.steps / t_steps, "unit": "DOF/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_steps / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded N(0,1) RHS, mean removed)",
                "config": {"workload": WORKLOAD_C3, "coarse": "p=1 pseudo-inverse, replicated",
                           "global_dofs": ndof, "parallelism": f"{world} element-row strips "
                           f"({plan.s} rows + 1 ghost row each side), NCCL halo send/recv, NCCL all-gather + "
                           "replicated coarse solve",
                           "halo": ("libsmg smg_halo_* (NCCL, compute stream)" if native
                                    else "torch.distributed point-to-point"),
                           "l2": "flushed (256 MiB write) before every timed step", "cuda_graph": use_graph,
                           "strong_scaling_reference": "the N=1 line's c3_single_gpu"},
                "e2e": {"value": ndof * args.steps / t_e2e, "unit": "DOF/s",
                        "h2d_bytes_per_step": 8 * f.numel() * world, "d2h_bytes_per_step": own_bytes * world},
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks}
        if c4 is not None:
            line["c4_mgcg"] = c4
        emit(line)
    dist.destroy_process_group()


def c3_single_gpu(args, dev, flush):
    """Strong-scaling reference for the N > 1 lines: the C3 V-cycle on one GPU
    (graph replay of the public path, L2 flushed before each step)."""
    import torch
    import paper_1512_02390_b200 as P
    from paper_1512_02390_b200.multigrid import _v_cycle
    c = C3
    h = P.build_hierarchy(P.MeshConfig(c["n_x"], c["n_y"], c["l_x"], c["l_y"]), c["p"], P.OverlapRule.parse(c["rule"]))
    shape = h.top.op.layout.shape
    f = torch.from_numpy(P.project_mean(np.random.default_rng(c["seed"]).standard_normal(shape))).to(dev)
    u = torch.zeros_like(f)
    _v_cycle(h, u, f)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        _v_cycle(h, u, f)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        _v_cycle(h, u, f)
    for _ in range(3):
        g.replay()
    evs = []
    n = max(5, min(args.steps, 20))
    for _ in range(n):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    t = float(sum(a.elapsed_time(b) for a, b in evs)) / 1e3 / n
    del g
    return {"workload": WORKLOAD_C3.replace(", element-row strips", ", one GPU"), "value": shape[0] * shape[1] / t,
            "unit": "DOF/s", "ms_per_step": 1e3 * t, "steps": n}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-micro", action="store_true", help="skip the smoother microbenchmark")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-c4", action="store_true", help="N > 1: skip the C4 MGCG solve")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return

    import torch
    import torch.distributed as dist
    _claim_stdout()
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # the driver counts ranks / sees NVLS in the log
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # ... on stderr: stdout carries only the JSON line
        ngpu = torch.cuda.device_count()
        local = local % max(ngpu, 1)
        torch.cuda.set_device(local)
        backend = os.environ.get("SMG_DIST_BACKEND", "nccl" if ngpu >= world else "gloo")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # more ranks than GPUs (testing only): gloo, host-staged halos
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    import paper_1512_02390_b200 as P
    from paper_1512_02390_b200 import _native as NV
    from paper_1512_02390_b200.multigrid import _v_cycle

    lib = NV.lib()
    if world == 1 and os.environ.get("SMG_BENCH_STRIPS") == "1":
        # testing aid: the N > 1 code path (strips, NCCL halos, graph) on one
        # rank, its halos wrapping onto itself
        import socket
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=dev)
        return run_strips(args, world, rank, local, dev)
    if world > 1:
        return run_strips(args, world, rank, local, dev)
    c = CFG
    mesh = P.MeshConfig(c["n_x"], c["n_y"], c["l_x"], c["l_y"])
    rule = P.OverlapRule.parse(c["rule"])
    h = P.build_hierarchy(mesh, c["p"], rule)
    shape = h.top.op.layout.shape
    ndof = shape[0] * shape[1]
    f_host = P.project_mean(np.random.default_rng(c["seed"]).standard_normal(shape))
    f = torch.from_numpy(f_host).to(dev)
    u = torch.zeros(shape, dtype=torch.float64, device=dev)
    bw, bw_src = _peaks()
    p64 = FP64_PEAK_TFLOPS * 1e12

    # eager warm-up (sets kernel attributes) and launch count per step
    _v_cycle(h, u, f)
    torch.cuda.synchronize()
    n0 = lib.smg_launch_count()
    _v_cycle(h, u, f)
    torch.cuda.synchronize()
    launches_per_step = lib.smg_launch_count() - n0

    # capture one step as a CUDA graph
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        _v_cycle(h, u, f)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        _v_cycle(h, u, f)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        g.replay()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    for a, b in ev:
        flush.fill_(1.0)
        a.record()
        g.replay()
        b.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall = time.perf_counter() - t_wall
    clocks = sampler.stop()
    t_steps = float(sum(a.elapsed_time(b) for a, b in ev)) / 1e3
    if world > 1:
        tt = torch.tensor([t_steps], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_steps = float(tt.item())
    value = ndof * world * args.steps / t_steps
    ms_per_step = 1e3 * t_steps / args.steps
    orders = [lv.basis.p for lv in h.levels]
    t_roof_vc = vcycle_roofline_seconds(mesh.n_x, mesh.n_y, orders, rule.layers, p64, bw * 1e9)

    # ---- top-level kernels, each timed alone on the launching stream (CUDA
    # events; torch's current stream IS the stream the kernels go to).  Two
    # methods: (1) "rotating": NB back-to-back launches over NB distinct
    # buffer sets whose total (>= 320 MB) exceeds the 126 MB L2, so every
    # launch streams its inputs from HBM -- the per-launch duration the
    # roofline uses; (2) "flushed": one launch after a 256 MiB L2 flush, event
    # to event (includes the launch latency and the flush's dirty write-back).
    # `roofline` is the kernel the north star names, the fused Schwarz correction;
    # `largest_share_of_step` names whichever call has the largest share of a V-cycle.
    top = h.top
    st = NV.stream()
    fshape = h.levels[-2].f.shape
    nset = 16

    def rnd(sh):
        return torch.randn(sh, dtype=torch.float64, device=dev)
    sets = [dict(r=rnd(shape), u=rnd(shape), o=rnd(shape), fc=torch.empty(fshape, dtype=torch.float64, device=dev),
                 uc=rnd(fshape)) for _ in range(nset)]
    # per V-cycle (1 pre-smoothing sweep, u != 0): r = f - A u, the Schwarz correction, the
    # residual restricted in place (r = f - A u is not stored: smg_residual_restrict_ws), the
    # prolongation; the stand-alone restriction is listed for reference (0 calls per cycle when
    # the fused residual + restriction is engaged)
    fused_rr = top.transfer.ws is not None
    calls = {
        "residual": (lambda S: NV.check(lib.smg_op_residual(top.op._handle.raw, NV.ptr(S["u"]), NV.ptr(S["r"]),
                                                            NV.ptr(S["o"]), st)), 1 if fused_rr else 2),
        "schwarz": (lambda S: NV.check(lib.smg_schwarz_correct(top.smoother._h.raw, NV.ptr(S["r"]), NV.ptr(S["o"]),
                                                              NV.ptr(top.smoother.ring), st)), 1),
        "residual_restrict": (lambda S: NV.check(lib.smg_residual_restrict_ws(
            top.transfer.handle.raw, top.op._handle.raw, NV.ptr(S["u"]), NV.ptr(S["r"]), NV.ptr(S["fc"]),
            NV.ptr(S["o"]), top.transfer.ws_ptr(), top.op.ring_ptr(), st)), 1 if fused_rr else 0),
        "restrict": (lambda S: NV.check(lib.smg_restrict(top.transfer.handle.raw, NV.ptr(S["r"]), NV.ptr(S["fc"]),
                                                         st)), 0 if fused_rr else 1),
        "prolong": (lambda S: NV.check(lib.smg_prolongate(top.transfer.handle.raw, NV.ptr(S["uc"]), NV.ptr(S["o"]), 1,
                                                          st)), 1),
    }
    t_call, t_call_flushed = {}, {}
    for nm, (fn, _) in calls.items():
        for S in sets:
            fn(S)
        torch.cuda.synchronize()
        reps = 4
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            for S in sets:
                fn(S)
        b.record()
        torch.cuda.synchronize()
        t_call[nm] = a.elapsed_time(b) / 1e3 / (reps * nset)
        evs = []
        for _ in range(20):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn(sets[0])
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        t_call_flushed[nm] = float(np.mean([a.elapsed_time(b) for a, b in evs])) / 1e3
    del sets
    m = c["p"] + 1 + 2 * rule.layers(c["p"])
    pc = h.levels[-2].basis.p
    npp = c["p"] + 1
    n_el = mesh.n_el
    ndof_c = n_el * pc * pc
    f_tr = 2.0 * n_el * ((c["p"] + 1) * (pc + 1) ** 2 + (c["p"] + 1) ** 2 * (pc + 1))
    tr_all = load_traffic()

    def tb(*names):
        v = [tr_all[n]["bytes_per_launch"] for n in names if n in tr_all]
        return float(sum(v)) if len(v) == len(names) else None
    eng, tile_x, tile_y = top.smoother.kernel_info()
    schwarz_kernel = "fdp_kernel" if eng == "pair" else "fdt_kernel"
    schwarz_label = (f"{schwarz_kernel}<{c['p']},{rule.layers(c['p'])},{tile_x},{tile_y}> + fdt_fixup "
                     f"(one Schwarz correction; engine {eng})")
    kern = {
        "residual": roofline_entry("opw_kernel<16,2,2> (r = f - A u, warp per element)", t_call["residual"],
                                   n_el * (4 * npp ** 3 + 3 * npp ** 2) + ndof, 24.0 * ndof, p64, bw * 1e9,
                                   tb("opw_kernel")),
        "schwarz": roofline_entry(schwarz_label, t_call["schwarz"],
                                  n_el * fd_eo_flops_per_element(m), 24.0 * ndof, p64, bw * 1e9,
                                  tb(schwarz_kernel, "fdt_fixup"),
                                  note="even/odd flop count (SURVEY 8(d)); dense-FD equivalent "
                                       f"{n_el * fd_flops_per_element(m) / t_call['schwarz'] / 1e12:.2f} TF"),
        "residual_restrict": roofline_entry(
            "opw_kernel<16,2,2,RESTR> + restrict_fixup<8> (f_c = R (f - A u), r not stored)"
            if fused_rr else "opw_kernel<16,2,2> + restrict_blk_kernel<8,16>", t_call["residual_restrict"],
            n_el * (4 * npp ** 3 + 3 * npp ** 2) + ndof + f_tr, 16.0 * ndof + 8.0 * ndof_c, p64, bw * 1e9,
            tb("opw_kernel_restr", "restrict_fixup")),
        "restrict": roofline_entry("restrict_blk_kernel<8,16> (stand-alone restriction)", t_call["restrict"], f_tr,
                                   8.0 * ndof + 8.0 * ndof_c, p64, bw * 1e9, tb("restrict_blk_kernel")),
        "prolong": roofline_entry("prolong_warp_kernel<8,16> (u_f += P u_c)", t_call["prolong"], f_tr,
                                  16.0 * ndof + 8.0 * ndof_c, p64, bw * 1e9, tb("prolong_warp_kernel")),
    }
    for nm in kern:
        kern[nm]["us_per_call_flushed"] = 1e6 * t_call_flushed[nm]
        kern[nm]["timing"] = (f"{nset} distinct buffer sets (>= 320 MB, > L2) launched back to back x 4, "
                              "mean per launch; us_per_call_flushed: single launch after a 256 MiB L2 flush")
    # `roofline` is the kernel the north star names -- the fused Schwarz correction -- whether
    # or not it still has the largest share of the step (the operator is applied twice per
    # cycle, once as the plain residual and once inside the restricted residual; every
    # top-level kernel is listed under top_level_kernels with its own fraction)
    dom = max(calls, key=lambda k: calls[k][1] * t_call[k])
    roofline = dict(kern["schwarz"])
    roofline["share_of_step"] = calls["schwarz"][1] * t_call["schwarz"] / (ms_per_step / 1e3)
    roofline["largest_share_of_step"] = {"kernel": dom, "share": calls[dom][1] * t_call[dom] / (ms_per_step / 1e3)}
    roofline["peak_source"] = (f"HBM {bw} GB/s ({bw_src}); FP64 {FP64_PEAK_TFLOPS} TF = measured DMMA "
                               "peak (tools/peaks/fp64_peaks.cu; MEASURED_PEAKS.json has no FP64 entry)")
    # ---- end to end through the public API with host buffers.  Every step
    # copies ITS f from pinned host memory (H2D) and reads ITS u back (D2H);
    # the copies run on their own streams so step k's D2H and step k+1's H2D
    # overlap step k+1's / k's V-cycle (a solver service streaming right-hand
    # sides).  The serial variant (copy, V-cycle, copy on one stream) is
    # reported beside it.
    f_pin = torch.from_numpy(f_host).pin_memory()
    u_pin = [torch.empty(shape, dtype=torch.float64).pin_memory() for _ in range(2)]
    f_stage = [torch.empty_like(f) for _ in range(2)]
    u_stage = [torch.empty_like(u) for _ in range(2)]
    cs = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def e2e_pipelined(n):
        ev_in = [torch.cuda.Event() for _ in range(n)]      # f_stage[k%2] filled
        ev_used = [torch.cuda.Event() for _ in range(n)]    # f_stage[k%2] consumed, u_stage[k%2] filled
        ev_out = [torch.cuda.Event() for _ in range(n)]     # u_stage[k%2] drained
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(s_in)
        s_out.wait_stream(s_in)
        cs.wait_stream(s_in)
        for k in range(n):
            j = k % 2
            with torch.cuda.stream(s_in):
                if k >= 2:
                    s_in.wait_event(ev_used[k - 2])
                f_stage[j].copy_(f_pin, non_blocking=True)
                ev_in[k].record(s_in)
            cs.wait_event(ev_in[k])
            if k >= 2:
                cs.wait_event(ev_out[k - 2])
            flush.fill_(1.0)
            f.copy_(f_stage[j])
            g.replay()
            u_stage[j].copy_(u)
            ev_used[k].record(cs)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_used[k])
                u_pin[j].copy_(u_stage[j], non_blocking=True)
                ev_out[k].record(s_out)
        s_out.wait_stream(cs)
        b.record(s_out)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 1e3

    def e2e_serial(n):
        evs = []
        for _ in range(n):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f.copy_(f_pin, non_blocking=True)
            g.replay()
            u_pin[0].copy_(u, non_blocking=True)
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        return float(sum(a.elapsed_time(b) for a, b in evs)) / 1e3

    e2e_pipelined(args.warmup)
    e2e_serial(args.warmup)
    t_e2e = e2e_pipelined(args.steps)
    t_e2e_serial = e2e_serial(args.steps)
    got = u_pin[(args.steps - 1) % 2]
    if not bool(torch.isfinite(got).all()):
        raise RuntimeError("e2e: non-finite V-cycle output")
    if world > 1:
        tt = torch.tensor([t_e2e, t_e2e_serial], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e, t_e2e_serial = (float(x) for x in tt.tolist())
    e2e = {"value": ndof * world * args.steps / t_e2e, "unit": "DOF/s",
           "h2d_bytes_per_step": 8 * ndof, "d2h_bytes_per_step": 8 * ndof,
           "path": "per step: pinned host f -> H2D (copy stream) -> v_cycle (graph replay of the public "
                   "v_cycle) -> D2H u (copy stream); copies of neighbouring steps overlap the V-cycle; "
                   "L2 flushed (256 MiB write) on the compute stream before every step",
           "serial_value": ndof * world * args.steps / t_e2e_serial,
           "serial_path": "H2D f, v_cycle, D2H u on one stream, L2 flushed before each step"}

    # ---- smoother-only microbenchmark (64^2 and 256^2 elements, n_o = 1)
    micro = None
    if not args.no_micro:
        micro = {}
        for n_el1d in (64, 256):
            for p in (4, 8, 12, 16, 24, 32):
                msh = P.MeshConfig(n_el1d, n_el1d, 1.0, 1.0)
                lay = P.layout_for(msh, p)
                sm2 = P.AdditiveSchwarz(P.gll_basis(p), lay, msh.dx, msh.dy, 1, P.WeightKind.QUINTIC)
                rr = torch.randn(lay.shape, dtype=torch.float64, device=dev)
                uu = torch.zeros(lay.shape, dtype=torch.float64, device=dev)
                sm2.correct(rr, uu)
                evs = []
                for _ in range(10):
                    flush.fill_(1.0)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    sm2.correct(rr, uu)
                    b.record()
                    evs.append((a, b))
                torch.cuda.synchronize()
                tt = float(np.median([a.elapsed_time(b) for a, b in evs])) / 1e3
                mm = p + 3
                fl = msh.n_el * fd_eo_flops_per_element(mm)
                by = 24.0 * lay.size
                t_roof = max(fl / p64, by / (bw * 1e9))
                micro[f"{n_el1d}x{n_el1d}_p{p}"] = {
                    "gdof_s": lay.size / tt / 1e9, "us": 1e6 * tt, "tflops_eo": fl / tt / 1e12,
                    "gbs": by / tt / 1e9, "bound": "hbm" if by / (bw * 1e9) >= fl / p64 else "fp64",
                    "frac": t_roof / tt,
                    "tflops_dense_equiv": msh.n_el * fd_flops_per_element(mm) / tt / 1e12}
                del sm2, rr, uu

    # ---- the same V-cycle with the reference's own coarse solver (plain CG to
    # 1e-12 on the device, coarse="cg"; not graph-capturable: it tests
    # convergence on the host every 32 iterations) -- the like-for-like
    # companion of the reference arm, whose V-cycle runs that CG on the CPU
    hcg = P.build_hierarchy(mesh, c["p"], rule, coarse="cg")
    ucg = torch.zeros_like(u)
    _v_cycle(hcg, ucg, f)
    evs = []
    for _ in range(max(5, min(args.steps, 20))):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _v_cycle(hcg, ucg, f)
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    t_cg = float(np.mean([a.elapsed_time(b) for a, b in evs])) / 1e3
    vc_cg = {"value": ndof / t_cg, "unit": "DOF/s", "ms_per_step": 1e3 * t_cg,
             "coarse": "plain CG to 1e-12 on the device (the reference's coarse solver)",
             "coarse_iterations": hcg.coarse_iterations[-1] if hcg.coarse_iterations else None,
             "timing": "eager launches, CUDA events, L2 flushed before each step"}
    del hcg, ucg

    # ---- solve-level end to end through the public API: solve(h, f_host, cfg,
    # u0) with numpy f (H2D inside), MG to 1e10 (13 cycles), u read back to the
    # host; value = DOF x V-cycles / wall time
    sols = []
    for k in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        us_, rep = P.solve(h, f_host, P.SolveConfig(solver="mg"), u0=np.zeros_like(f_host))
        u_host = us_.cpu().numpy()
        t1 = time.perf_counter() - t0
        if k:
            sols.append((t1, rep.cycles))
    t_sol = float(np.median([t for t, _ in sols]))
    e2e_solve = {"value": ndof * sols[-1][1] / t_sol, "unit": "DOF/s", "cycles": sols[-1][1],
                 "time_to_solution_ms": 1e3 * t_sol, "converged": bool(rep.converged),
                 "h2d_bytes": 8 * ndof * 2, "d2h_bytes": 8 * ndof,
                 "path": "solve(h, f_host (numpy), SolveConfig('mg'), u0=zeros (numpy)) -> u.cpu(); host wall "
                         "clock, median of 3 after one warm-up; one host sync per cycle (convergence test)"}
    assert np.isfinite(u_host).all()

    c3 = c3_single_gpu(args, dev, flush)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        times, _, kind = time_cpu_vcycles(args.cpu_budget)
        tc = float(np.sum(times))
        cpu = {"value": ndof * len(times) / tc, "unit": "DOF/s", "cores": cpu_threads(), "kind": kind,
               "sample": _cpu_sample(kind, len(times))}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded N(0,1) RHS, mean removed)",
                "config": {"workload": WORKLOAD_C2, "coarse": "p=1 pseudo-inverse (exact; vcycle_coarse_cg: "
                                                              "the reference's CG)",
                           "global_dofs": ndof * world, "levels": orders,
                           "parallelism": "single GPU" if world == 1 else f"{world} independent replicas",
                           "l2": "flushed (256 MiB write) before every timed step",
                           "cuda_graph": True},
                "vcycle_roofline": {"t_roof_us": 1e6 * t_roof_vc, "t_measured_us": ms_per_step * 1e3,
                                    "frac": t_roof_vc / (ms_per_step / 1e3),
                                    "model": "SURVEY.md §8(d) sum of max(F/P64, B/BW) over levels, "
                                             f"P64={FP64_PEAK_TFLOPS} TF, BW={bw} GB/s ({bw_src}), coarse excluded"},
                "roofline": roofline, "top_level_kernels": kern, "e2e": e2e, "e2e_solve": e2e_solve,
                "vcycle_coarse_cg": vc_cg, "c3_single_gpu": c3,
                "gpu_launches": launches_per_step * args.steps,
                "clocks": clocks, "wall_s_timed_region": t_wall}
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if micro is not None:
            line["smoother_microbench"] = micro
        emit(line)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
