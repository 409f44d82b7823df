#!/usr/bin/env python
"""Benchmark: ISM pressure solve (arXiv 1309.7128) on B200 — fine-grid cell-updates/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--case lid|jet] [--grid N]

Default workload (BASELINE.json north star, configs[2] = SURVEY.md §8(d)
config 3): lid-driven cavity 16384^2, Re = 1000, u_lid = 0.1, h = 1,
dt = Re/n, ISM two-level with 32h tiles (coarse 512^2), tol_fine 1e-6,
tol_coarse 1e-5, 20000-sweep budget, stall 0.9, fp64, synthetic quiescent
start (seed 0). --grid 4096 gives config 2; --case jet gives config 4
(setup_jet(8192, 16384, 0.1, 16), tile 16; --grid N runs the jet N x 2N).

A "step" is one projection step (predictor, divergence, ISM pressure solve,
correction). W warm-up steps run on a throwaway state; the K timed steps are
steps 1..K of the time integration from the quiescent start. Metric = fine-grid
cell-updates per second = sum(I_f) * nx * ny / time.

  value     device-resident state, CUDA events around the K steps on the library
            stream (torch's current stream), max over ranks.
  e2e       the same K steps through the public API with the state in pinned host
            memory: per step H2D of (u, v, p), step, D2H of (u, v, p).
  roofline  the dominant kernel (fused fine pass, 24 algorithmic B/cell) timed with
            CUDA events per launch on the library stream, against the measured HBM
            copy bandwidth in MEASURED_PEAKS.json; `solve_level` = value x 24 B.
  cpu_baseline  the unmodified reference (oracle/_ref, compiled from its own headers)
            on 1 host core, SAME WORK: its own per-operation costs on this workload
            (ref_op_costs: rbgs_sweep, fine_residual, anchor_mean, restrict_sum,
            prolongate_bilinear, gs_sweep_lex, coarse_residual, coarse anchor, and one
            step() from rest for the per-step fixed cost) times this run's exact
            per-step counts (I_f, I_c, restrictions, prolongations). Validated against
            whole reference runs: model / measured = 0.96 (1024^2, 3 steps), 0.82
            (2048^2, 1 step) - the model flatters the CPU.

--impl reference runs that reference CPU path with every host core it can use:
the reference solve is single-threaded (cycles.hpp; bench.hpp:266-313 only
parallelises independent cases), so each core runs its own instance of the
per-operation timings concurrently (memory-bandwidth contention included); the
aggregate rate is cores x the per-instance rate on the same K-step workload,
whose counts are the reference's own (tests/golden/scale/*.npz) for the steps it
was run to and, beyond them, profiles/r02_counts_*.json (this implementation's
counts, identical to the reference's wherever both exist).
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

LID_N = 16384   # config 3 (north star)
JET_NX = 8192   # config 4: jet 8192 x 16384
RE = 1000.0
TILE = 32


def config_name(n, kind="lid"):
    if kind == "jet":
        return "config 4" if n == JET_NX else "jet %dx%d" % (n, 2 * n)
    return "config 3" if n == 16384 else ("config 2" if n == 4096 else "lid %d^2" % n)


def workload(n=LID_N, kind="lid"):
    """The bench workloads. lid: configs 2 / 3, lid cavity n x n, Re 1000,
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
    """nx of the workload: --grid if given, else 16384 for the lid (config 3), 8192 for the jet (config 4)."""
    if args.grid:
        return args.grid
    return JET_NX if args.case == "jet" else LID_N


def workload_desc(n, kind):
    if kind == "jet":
        return "turbulent jet %dx%d, v0 0.1, inlet 16, nu 0.01, dt 1, ISM 16h two-level (%s)" % (
            n, 2 * n, config_name(n, kind))
    return "lid-driven cavity %dx%d Re=1000, dt=Re/n, ISM 32h two-level (%s)" % (n, n, config_name(n))


def counts_key(n, kind):
    return "%s%d" % (kind, n)


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


def fine_traffic(n=LID_N):
    """DRAM bytes per launch of the fine pass from the committed ncu --set full capture
    (profiles/fine_pass_traffic.json, dram__bytes_read.sum + dram__bytes_write.sum), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "fine_pass_traffic.json")) as f:
            return float(json.load(f)["by_grid"][str(n)]["dram_bytes_per_launch"])
    except Exception:
        return None


def cpu_kind():
    from pyoracle import available
    return "reference" if available("reference") else "port"


def cpu_model():
    """CPU model string of this host (lscpu / /proc/cpuinfo)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def op_costs(n, kind, reps=1):
    """The reference's per-operation costs on this workload (seconds per call), 1 core."""
    from pyoracle import Oracle
    case, cfg = workload(n, kind)
    return Oracle("reference").op_costs(case.grid, cfg, case.dt, case.nu, reps)


def model_seconds(o, rows):
    """Reference wall time of projection steps with the given per-step counts
    (I_f, I_c, restrictions, prolongations), from per-operation costs o
    (pyoracle.op_costs order), following solve_two_level (cycles.hpp:101-165):
    every fine sweep is rbgs_sweep + fine_residual + anchor_mean; every restriction
    restrict_sum + the entry coarse_residual; every coarse sweep gs_sweep_lex +
    coarse_residual + coarse anchor_mean; every prolongation prolongate_bilinear +
    fine_residual + anchor_mean; o[8] (one step from rest with a 1-sweep budget)
    carries each step's fixed cost and its first restriction and coarse sweep."""
    t = 0.0
    for i_f, i_c, r, p in rows:
        t += (o[8] + i_f * (o[0] + o[1] + o[2]) + max(0, r - 1) * (o[3] + o[6]) +
              max(0, i_c - 1) * (o[5] + o[6] + o[7]) + p * (o[4] + o[1] + o[2]))
    return t


def reference_counts(n, kind, steps):
    """Per-step (I_f, I_c, restrictions, prolongations) of projection steps 1..steps of the
    workload: the reference's own rows (tests/golden/scale/*.npz, made by the compiled
    reference), then profiles/r02_counts_<workload>.json (this implementation's counts, equal
    to the reference's wherever both exist); the last known step repeats beyond both."""
    import numpy as np
    fx = {("lid", 16384): "c3", ("lid", 4096): "c2", ("lid", 256): "c1", ("jet", 8192): "c4",
          ("jet", 512): "jet512", ("jet", 1024): "jet1024"}.get((kind, n))
    rows, src = [], []
    if fx and os.path.exists(os.path.join(ROOT, "tests", "golden", "scale", fx + ".npz")):
        z = np.load(os.path.join(ROOT, "tests", "golden", "scale", fx + ".npz"))
        rows = [(int(r[1]), int(r[2]), int(r[5]), int(r[6])) for r in z["rows"]][:steps]
        src.append("steps 1-%d: the reference's own (tests/golden/scale/%s.npz)" % (len(rows), fx))
    path = os.path.join(ROOT, "profiles", "r02_counts_%s.json" % counts_key(n, kind))
    if len(rows) < steps and os.path.exists(path):
        with open(path) as f:
            more = [tuple(r) for r in json.load(f)["rows"]]
        k0 = len(rows)
        rows += more[k0:steps]
        if len(rows) > k0:
            src.append("steps %d-%d: %s" % (k0 + 1, len(rows), os.path.relpath(path, ROOT)))
    if not rows:
        raise RuntimeError("no per-step counts for %s %d" % (kind, n))
    k0 = len(rows)
    while len(rows) < steps:
        rows.append(rows[-1])
    if k0 < steps:
        src.append("steps %d-%d: step %d repeated" % (k0 + 1, steps, k0))
    return rows, "; ".join(src)


def run_reference_arm(args, rank, world):
    """--impl reference: the unmodified reference CPU path on all host cores."""
    if rank != 0:
        return
    import psutil
    kind = cpu_kind()
    ck = args.case
    n = grid_side(args)
    case, _ = workload(n, ck)
    cells = case.grid.nx * case.grid.ny
    ncpu = os.cpu_count() or 1
    mem_gb = psutil.virtual_memory().available / 2 ** 30
    per_inst = 12 * 8 * cells / 2 ** 30 + 1.0  # u, v, p, vstar, rhs, dp, x, b, res, diag, ... (fp64)
    cores = max(1, min(ncpu, int(mem_gb * 0.8 // per_inst)))
    rows, src = reference_counts(n, ck, args.steps)
    fine_all = sum(r[0] for r in rows)

    def round_(reps):
        res = [None] * cores

        def work(k):
            res[k] = op_costs(n, ck, reps)
        th = [threading.Thread(target=work, args=(k,)) for k in range(cores)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        return res, time.perf_counter() - t0

    for _ in range(min(args.warmup, 1)):
        round_(1)
    per_inst_s, rounds_wall = [], 0.0
    for _ in range(args.steps if args.steps <= 3 else 3):  # K-step model; up to 3 timing rounds
        res, wall = round_(1)
        rounds_wall += wall
        per_inst_s.append(statistics.mean(model_seconds(o, rows) for o in res))
    t_model = statistics.median(per_inst_s)  # one instance's time for the K-step workload
    value = cores * fine_all * cells / t_model
    sample = ("same work as the GPU arm: the reference's per-operation costs on %s (ref_op_costs, "
              "one instance per core, %d concurrent) x per-step counts of projection steps 1..%d (%s); "
              "host %s" % (workload_desc(n, ck), cores, args.steps, src, cpu_model()))
    line = {
        "impl": "reference", "metric": "fine-grid cell-updates/s", "value": value, "unit": "cell-updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_model / args.steps / cores,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(n, ck), "global_batch": 1, "seq_len": 0,
                   "parallelism": "%d independent single-threaded reference instances" % cores,
                   "steps_timed": "projection steps 1..%d (counts model)" % args.steps},
        "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores, "kind": kind, "sample": sample,
                         "cpu_model": cpu_model(), "timing_rounds_wall_s": rounds_wall},
        "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


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
    engine = solver.last_stats()["coarse_engine"]
    del ds
    torch.cuda.synchronize()
    if engine in (0, 1) and max(solver.visit_log() or [(0, 0)])[0] > 1000 and not args.allow_slow_coarse:
        raise SystemExit("bench: the coarse visit fell back to the %s engine at this size (no fast plan); "
                         "refusing a run that would take hours (--allow-slow-coarse to force)"
                         % ("global-memory" if engine == 0 else "shared-memory"))

    # --- timed region: device-resident state, steps 1..K
    ds = P.DeviceState(g, ctx, fresh_state())
    m = RunMetrics(cells)
    l0 = ctx.launch_count()
    coarse_ms = 0.0
    coarse_engines = set()
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            ds.step(solver, m)
            s_ = solver.last_stats()  # host-side copy of the solve's device-timed stats (no sync added)
            coarse_ms += s_["coarse_ms"]
            coarse_engines.add(int(s_["coarse_engine"]))
        e1.record(stream)
        torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count() - l0
    rows = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations) for r in m.rows]
    fine = sum(r[0] for r in rows)
    coarse = sum(r[1] for r in rows)
    n_conv = sum(1 for r in m.rows if r.converged)
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
    if args.save_counts and rank == 0:
        with open(args.save_counts, "w") as f:
            json.dump({"workload": workload_desc(n, ck), "what": "per-step (I_f, I_c, restrictions, prolongations) "
                       "of projection steps 1..%d, this implementation (bench.py --save-counts)" % args.steps,
                       "rows": rows}, f)

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

    # --- CPU baseline: the reference on one core, same work (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        kind = cpu_kind()
        if kind == "reference":
            o = op_costs(n, ck, 1)
            t_cpu = model_seconds(o, rows)
            smp = ("same work: the reference's per-operation costs on this workload (ref_op_costs, 1 core) x this "
                   "run's per-step counts (steps 1..%d: I_f %d, I_c %d, restrictions %d, prolongations %d) = %.0f s "
                   "of reference time; host %s" % (args.steps, fine, coarse, sum(r[2] for r in rows),
                                                   sum(r[3] for r in rows), t_cpu, cpu_model()))
            cpu = {"value": fine_all * cells / t_cpu, "unit": "cell-updates/s", "cores": 1, "kind": kind,
                   "sample": smp, "same_work": True,
                   "op_costs_s": {k: float(v) for k, v in zip(
                       ("rbgs_sweep", "fine_residual", "anchor_mean", "restrict_sum", "prolongate_bilinear",
                        "gs_sweep_lex", "coarse_residual", "coarse_anchor", "step_fixed"), o)}}

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
                       "fine_sweeps": int(fine_all), "coarse_sweeps": int(coarse),
                       "solves_converged": n_conv, "solves_budget_capped": args.steps - n_conv},
            "pressure_solves_per_s": args.steps / (ms_max * 1e-3),
            "coarse": {"engine": sorted(coarse_engines), "ms_per_step": coarse_ms / args.steps,
                       "share": coarse_ms / ms if ms > 0 else None,
                       "us_per_sweep": 1e3 * coarse_ms / max(1, coarse),
                       "cell_updates_per_s": coarse * solver_coarse_cells(g, cfg) / max(1e-9, coarse_ms * 1e-3)},
            "e2e": {"value": e2e_value, "unit": "cell-updates/s", "h2d_bytes_per_step": bytes_io,
                    "d2h_bytes_per_step": bytes_io},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": fine_traffic(n if ck == "lid" else "jet%d" % n), "kernel": "fine_pass_w_kernel (sweep mode)",
                         "alg_bytes_per_launch": alg_bytes, "ms_per_launch": pass_ms, "peak_source": src,
                         "solve_level": {"achieved": value * 24.0 / 1e9, "frac": value * 24.0 / 1e9 / hbm,
                                         "what": "fine cell-updates/s x 24 B (x r/w + b r per update)"}},
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        emit(line)


def solver_coarse_cells(g, cfg):
    return ((g.nx + cfg.tile - 1) // cfg.tile) * ((g.ny + cfg.tile - 1) // cfg.tile)


_STDOUT_FD = None  # the real stdout while libraries' banners (NCCL) are sent to stderr


def quiet_stdout():
    """Send fd 1 to stderr until emit(): NCCL prints its version banner on stdout
    from C code when a communicator is created, ahead of the one JSON line."""
    global _STDOUT_FD
    if _STDOUT_FD is None:
        sys.stdout.flush()
        _STDOUT_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line):
    """The bench's one JSON line, on the real stdout."""
    text = json.dumps(line) + "\n"
    sys.stdout.flush()
    if _STDOUT_FD is None:
        sys.stdout.write(text)
        sys.stdout.flush()
    else:
        os.write(_STDOUT_FD, text.encode())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", type=int, default=None,
                    help="grid side: lid 16384 (config 3, default) or 4096 (config 2); jet nx (8192 = config 4)")
    ap.add_argument("--case", default="lid", choices=["lid", "jet"],
                    help="lid: lid cavity --grid^2 (configs 2, 3); jet: config 4, jet nx x 2nx (nx = 8192 unless --grid)")
    ap.add_argument("--save-counts", default=None, help="write the timed steps' per-step counts (JSON) here")
    ap.add_argument("--allow-slow-coarse", action="store_true",
                    help="run even when the coarse visit has no fast plan at this size")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and "RANK" in os.environ:
        quiet_stdout()  # NCCL's version banner must not precede the JSON line
        import torch
        import torch.distributed as tdist
        if args.impl == "ours":  # the reference arm is CPU-only (gloo), no device needed
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
