#!/usr/bin/env python
"""Benchmark: ISM pressure solve (arXiv 1309.7128) on B200 — fine-grid cell-updates/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--grid 4096|16384]

--grid 16384 runs BASELINE.json configs[2] (config 3, coarse 512^2) instead of the
default config 2; every other setting is the same.

Workload (BASELINE.json configs[1]): lid-driven
cavity 4096^2, Re = 1000, u_lid = 0.1, h = 1, dt = Re/n, ISM two-level with
32h tiles (coarse 128^2), tol_fine 1e-6, tol_coarse 1e-5, 20000-sweep budget,
stall 0.9, fp64, synthetic quiescent start (seed 0).

A "step" is one projection step (predictor, divergence, ISM pressure solve,
correction). W warm-up steps run on a throwaway state; the K timed steps are
steps 1..K of the time integration from the quiescent start (the reference arm
samples step 1 as well). Metric = fine-grid cell-updates per second =
sum(I_f) * nx * ny / time.

  value   device-resident state, CUDA events around the K steps on the library
          stream (torch's current stream), max over ranks.
  e2e     the same K steps through the public API with the state in pinned host
          memory: per step H2D of (u, v, p), step, D2H of (u, v, p).
  roofline  the dominant kernel (fused fine pass, 24 algorithmic B/cell) timed
          with CUDA events per launch on the library stream, against the
          measured HBM copy bandwidth in MEASURED_PEAKS.json.
  cpu_baseline  the unmodified reference (oracle/_ref, compiled from its own
          headers) on 1 host core, bounded sample: step 1 capped at 3000 sweeps.

--impl reference runs that reference CPU path with every host core it can use:
the reference solve is single-threaded (cycles.hpp; bench.hpp:266-313 only
parallelises independent cases), so it runs one independent capped step-1
sample per core and reports the aggregate cell-updates/s.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

N_DEFAULT = 4096
RE = 1000.0
TILE = 32
REF_SAMPLE_CAP = 3000  # max_total_sweeps of the bounded CPU sample (step 1)


JET_NX = 8192  # config 4: jet 8192 x 16384


def config_name(n, kind="lid"):
    if kind == "jet":
        return "config 4" if n == JET_NX else "jet %dx%d" % (n, 2 * n)
    return "config 3" if n == 16384 else ("config 2" if n == 4096 else "lid %d^2" % n)


def workload(n=N_DEFAULT, kind="lid"):
    """The bench workloads. lid: config 2 / 3, lid cavity n x n, Re 1000,
    tile 32. jet: config 4, setup_jet(n, 2n, 0.1, 16) (bench.hpp:73-88), dt 1, tile 16
    (jet.cfg:15): non-singular (fixed-pressure top), so no anchoring."""
    from paper_1309_7128_b200.api import CycleConfig, setup_jet, setup_lid_cavity
    if kind == "jet":
        case = setup_jet(n, 2 * n, 0.1, 16)
        tile = 16
    else:
        case = setup_lid_cavity(n, RE)
        case.dt = RE / n  # dt = Re/n: the reference default dt = 1 diverges
        tile = TILE
    case.steps, case.t_max, case.steady_tol = 10 ** 9, 0.0, 0.0
    cfg = CycleConfig(tile=tile, tol_fine=1e-6, tol_coarse=1e-5, max_total_sweeps=20000, stall_factor=0.9)
    return case, cfg


def grid_side(args):
    """nx of the workload: --grid for the lid; for the jet 8192 (config 4) unless --grid is given."""
    if args.case == "jet" and args.grid == N_DEFAULT:
        return JET_NX
    return args.grid


def workload_desc(n, kind):
    if kind == "jet":
        return "turbulent jet %dx%d, v0 0.1, inlet 16, nu 0.01, dt 1, ISM 16h two-level (%s)" % (
            n, 2 * n, config_name(n, kind))
    return "lid-driven cavity %dx%d Re=1000, dt=Re/n, ISM 32h two-level (%s)" % (n, n, config_name(n))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            p = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except Exception:
                continue
            for k, name in enumerate(names):
                if len(p) > 3 + k and p[3 + k].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def fine_traffic(n=N_DEFAULT):
    """DRAM bytes per launch of the fine pass from the committed ncu --set full capture
    (profiles/fine_pass_traffic.json, dram__bytes_read.sum + dram__bytes_write.sum), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "fine_pass_traffic.json")) as f:
            return float(json.load(f)["by_grid"][str(n)]["dram_bytes_per_launch"])
    except Exception:
        return None


def cpu_sample(kind, n=N_DEFAULT, cap=REF_SAMPLE_CAP, case_kind="lid"):
    """One bounded reference sample: step 1 with the sweep budget capped. Returns (I_f, seconds)."""
    from pyoracle import Oracle
    from paper_1309_7128_b200.api import FluidState
    case, cfg = workload(n, case_kind)
    cfg.max_total_sweeps = cap
    st = FluidState(case.grid)
    st.dt, st.nu = case.dt, case.nu
    o = Oracle(kind)
    t0 = time.perf_counter()
    rows, secs = o.run_steps(case.grid, cfg, st, 1)
    wall = time.perf_counter() - t0
    return rows[0].fine_sweeps, (secs if secs is not None else wall)


def cpu_kind():
    from pyoracle import available
    return "reference" if available("reference") else "port"


def cpu_fine_iterations(kind, n, iters, case_kind="lid"):
    """Bounded reference sample for grids whose capped step 1 never reaches a fine sweep:
    `iters` outer fine iterations of step 1 (cycles.hpp:148-161: rbgs_sweep, fine_residual
    into the residual field, anchor_mean, restrict_sum) on the step-1 rhs, timed on one core.
    Returns (fine sweeps, seconds)."""
    from pyoracle import Oracle
    from paper_1309_7128_b200.api import FluidState, MacVelocity, ScalarField
    case, cfg = workload(n, case_kind)
    g = case.grid
    nx, ny = g.nx, g.ny
    o = Oracle(kind)
    st = FluidState(g)
    o.apply_velocity_bc(g, st.vel)
    vstar = MacVelocity(nx, ny)
    o.predictor(g, st.vel, st.p, case.dt, case.nu, vstar)
    o.apply_velocity_bc(g, vstar)
    b = ScalarField(nx, ny)
    o.divergence(g, vstar, b)
    b.data *= g.h * g.h / case.dt
    gt = dataclasses.replace(g, tile=cfg.tile)  # restrict_sum tiles the grid by the cycle's tile
    x = ScalarField(nx, ny)
    if kind == "reference":  # stage and fields built once inside the reference, iterations timed there
        import ctypes as C
        secs = C.c_double()
        o._check(o._fn("fine_iterations")(C.byref(gt.to_c()), C.c_void_p(x.data.ctypes.data),
                                          C.c_void_p(b.data.ctypes.data), C.c_long(iters), C.byref(secs)))
        return iters, secs.value
    res = ScalarField(nx, ny)
    cb = ScalarField((nx + cfg.tile - 1) // cfg.tile, (ny + cfg.tile - 1) // cfg.tile)
    t0 = time.perf_counter()
    for _ in range(iters):
        o.rbgs_sweep(gt, x, b)
        o.fine_residual(gt, x, b, res)
        o.anchor_mean(gt, x)
        o.restrict_sum(gt, res, cb)
    return iters, time.perf_counter() - t0


def run_reference_arm(args, rank, world):
    """--impl reference: the unmodified reference CPU solve on all host cores."""
    if rank != 0:
        return
    import psutil
    kind = cpu_kind()
    ck = args.case
    n = grid_side(args)
    ncpu = os.cpu_count() or 1
    mem_gb = psutil.virtual_memory().available / 2 ** 30
    cells = n * n * (2 if ck == "jet" else 1)
    cores = max(1, min(ncpu, int(mem_gb // (2.5 * cells / 4096 ** 2))))
    small = n == N_DEFAULT and ck == "lid"  # else a capped step 1 never reaches a fine sweep: sample fine iterations

    def round_(cap):
        res = [None] * cores

        def work(k):
            res[k] = cpu_sample(kind, n, cap, ck) if small else cpu_fine_iterations(kind, n, 1 if cap < 1000 else 2, ck)
        th = [threading.Thread(target=work, args=(k,)) for k in range(cores)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        wall = time.perf_counter() - t0
        if small:
            return sum(r[0] for r in res), wall
        # fine-iteration samples: the setup (predictor, divergence) is outside each sample's own
        # clock, so the aggregate is the sum of the concurrent samples' rates
        rate = sum(r[0] / r[1] for r in res)
        return rate * wall, wall

    for _ in range(args.warmup):
        round_(200)
    tot_if, tot_t = 0, 0.0
    for _ in range(args.steps):
        i_f, t = round_(REF_SAMPLE_CAP)
        tot_if += i_f
        tot_t += t
    value = tot_if * cells / tot_t
    what = ("step 1 of lid %d^2 Re 1000 (dt = Re/n, tile 32) capped at %d sweeps" % (n, REF_SAMPLE_CAP) if small else
            "2 outer fine iterations of step 1 of %s (rbgs_sweep, fine_residual, anchor_mean, restrict_sum)"
            % workload_desc(n, ck))
    sample = ("%s, %d independent single-threaded solves in parallel (the reference solve has no intra-solve "
              "threading)" % (what, cores))
    line = {
        "impl": "reference", "metric": "fine-grid cell-updates/s", "value": value, "unit": "cell-updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(n, ck),
                   "global_batch": 1, "seq_len": 0, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1309_7128_b200 as P
    from paper_1309_7128_b200.api import FluidState, RunMetrics

    torch.cuda.set_device(local_rank)
    stream = torch.cuda.current_stream()
    ctx = P.Context(local_rank, stream.cuda_stream)
    ck = args.case
    n = grid_side(args)
    case, cfg = workload(n, ck)
    g = case.grid
    nx, ny = g.nx, g.ny
    cells = nx * ny
    dist = world > 1
    if dist:  # strip decomposition: one NCCL communicator over the ranks
        import torch.distributed as tdist
        uid = [P.nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(uid, src=0)
        ctx.attach_comm(uid[0], rank, world)
    solver = P.PressureSolver(g, cfg, ctx)

    def fresh_state():
        st = FluidState(g)
        st.dt, st.nu = case.dt, case.nu
        return st

    # --- warm-up on a throwaway state
    ds = P.DeviceState(g, ctx, fresh_state())
    mw = RunMetrics(cells)
    for _ in range(args.warmup):
        ds.step(solver, mw)
    del ds
    torch.cuda.synchronize()

    # --- timed region: device-resident state, steps 1..K
    ds = P.DeviceState(g, ctx, fresh_state())
    m = RunMetrics(cells)
    l0 = ctx.launch_count()
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            ds.step(solver, m)
        e1.record(stream)
        torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count() - l0
    fine = sum(r.fine_sweeps for r in m.rows)
    coarse = sum(r.coarse_sweeps for r in m.rows)
    # the ranks share ONE solve (strips of the same grid): the job's cell updates are
    # I_f * nx * ny, timed as the max over ranks
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms_max = float(t[0])
    else:
        ms_max = ms
    fine_all = float(fine)
    value = fine_all * cells / (ms_max * 1e-3)

    # --- e2e: public API with the state in pinned host memory
    def pinned(nelem):
        return torch.empty(nelem, dtype=torch.float64, pin_memory=True).numpy()

    host = fresh_state()
    for name in ("u_data", "v_data"):
        a = pinned(getattr(host.vel, name).size)
        a[:] = 0.0
        setattr(host.vel, name, a)
    pdata = pinned(host.p.data.size)
    pdata[:] = 0.0
    host.p.data = pdata
    ds2 = P.DeviceState(g, ctx)
    m2 = RunMetrics(cells)
    bytes_io = (host.vel.u_data.nbytes + host.vel.v_data.nbytes + host.p.data.nbytes)
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        ds2.upload(host)  # H2D: u, v, p (+ t, dt, nu, step)
        ds2.step(solver, m2)
        ds2.download(host)  # D2H: u, v, p
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    fine2 = sum(r.fine_sweeps for r in m2.rows)
    if dist:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    e2e_value = fine2 * cells / (e2e_ms * 1e-3)

    # --- roofline: the fused fine pass on this GPU alone, CUDA events per launch on
    #     the library stream (a single-GPU context: the hook times one device)
    hbm, src = peaks()
    if dist:
        ctx = P.Context(local_rank, stream.cuda_stream)
        solver = P.PressureSolver(g, cfg, ctx)
    xs = P.DeviceField(nx, ny, ctx)
    bs = P.DeviceField(nx, ny, ctx)
    # rhs of the timed run's first step, rebuilt through the public kernels
    vel = P.DeviceVelocity(nx, ny, ctx)
    vstar = P.DeviceVelocity(nx, ny, ctx)
    pf = P.DeviceField(nx, ny, ctx)
    P.apply_velocity_bc(vel, g)
    vstar.upload(vel.download())
    P.predictor(vel, pf, case.dt, case.nu, g, vstar)
    P.apply_velocity_bc(vstar, g)
    P.divergence(vstar, g, bs, g.h * g.h / case.dt)
    pass_ms = solver.bench_fine_pass(xs, bs, 20)
    alg_bytes = 24.0 * cells
    achieved = alg_bytes / (pass_ms * 1e-3) / 1e9

    # --- CPU baseline: the reference on one core, bounded sample (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        kind = cpu_kind()
        if n == N_DEFAULT and ck == "lid":
            i_f, secs = cpu_sample(kind, n)
            smp = "step 1 of the same workload capped at %d sweeps (I_f %d in %.1f s)" % (REF_SAMPLE_CAP, i_f, secs)
        else:  # a capped step 1 at 16384^2 spends its whole budget in the first coarse visit
            i_f, secs = cpu_fine_iterations(kind, n, 2, ck)
            smp = ("%d outer fine iterations of step 1 (rbgs_sweep, fine_residual, anchor_mean, restrict_sum) "
                   "in %.1f s" % (i_f, secs))
        cpu = {"value": i_f * cells / secs, "unit": "cell-updates/s", "cores": 1, "kind": kind, "sample": smp}

    if rank == 0:
        line = {
            "metric": "fine-grid cell-updates/s", "value": value, "unit": "cell-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (quiescent %s, seed 0)" % ("jet box" if ck == "jet" else "lid-driven cavity"),
            "config": {"workload": workload_desc(n, ck),
                       "global_batch": 1, "seq_len": 0,
                       "parallelism": ("y-strips x%d (halo rows pushed over NVLink by the fine pass, partials "
                                       "and coarse-rhs rows pulled from peer memory; coarse solve replicated)"
                                       % world) if dist else "single GPU",
                       "steps_timed": "projection steps 1..%d" % args.steps,
                       "l2": "inputs larger than L2 (x, scratch, b: 3 x %.0f MB vs 126 MB L2)" % (8.0 * (nx + 2) * (ny + 2) / 1e6),
                       "fine_sweeps": int(fine_all), "coarse_sweeps": int(coarse)},
            "pressure_solves_per_s": args.steps / (ms_max * 1e-3),
            "e2e": {"value": e2e_value, "unit": "cell-updates/s", "h2d_bytes_per_step": bytes_io,
                    "d2h_bytes_per_step": bytes_io},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": fine_traffic(n if ck == "lid" else "jet%d" % n), "kernel": "fine_pass_w_kernel (sweep mode)",
                         "alg_bytes_per_launch": alg_bytes, "ms_per_launch": pass_ms, "peak_source": src},
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", type=int, default=N_DEFAULT, help="grid side: 4096 (config 2) or 16384 (config 3)")
    ap.add_argument("--case", default="lid", choices=["lid", "jet"],
                    help="lid: lid cavity --grid^2 (configs 2, 3); jet: config 4, jet nx x 2nx (nx = 8192 unless --grid)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and "RANK" in os.environ:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1 and "RANK" in os.environ:
        import torch.distributed as tdist
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
