"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family of the library on tiny grids, so the
instrumented run finishes in minutes.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import paper_1309_7128_b200 as P
from cases import random_field
from paper_1309_7128_b200.api import CycleConfig, RunMetrics, ScalarField, Scheme, setup_jet, setup_lid_cavity

which = sys.argv[1:] or ["fused", "jet", "schemes", "visit"]
if "fused" in which:  # fused solve + projection step (fine passes, sweep-pipeline coarse visits, predictor ...)
    case = setup_lid_cavity(64, 100.0)
    case.dt, case.steps, case.t_max, case.steady_tol = 100.0 / 64, 2, 0.0, 0.0
    res = P.run_case(case, CycleConfig(tile=8))
    print("fused lid64:", [(r.fine_sweeps, r.coarse_sweeps) for r in res.metrics.rows], flush=True)
if "jet" in which:  # non-singular level, Dirichlet top
    case = setup_jet(32, 64, 0.1, 8)
    case.steps, case.t_max, case.steady_tol = 2, 0.0, 0.0
    res = P.run_case(case, CycleConfig(tile=4))
    print("fused jet32x64:", [(r.fine_sweeps, r.coarse_sweeps) for r in res.metrics.rows], flush=True)
if "schemes" in which:  # op-level kernels: plain GS, GMG, ACM
    g = setup_lid_cavity(32, 100.0).grid
    b = random_field(32, 32, np.random.default_rng(3))
    b.shift_interior(-b.interior_mean())
    for s in (Scheme.plain_gs, Scheme.gmg, Scheme.acm):
        cfg = CycleConfig(scheme=s, tile=8, depth=3, tol_fine=1e-6, tol_coarse=1e-6, max_total_sweeps=400)
        rep = P.PressureSolver(g, cfg).solve(ScalarField(32, 32), b, RunMetrics(1024))
        print("scheme", int(s), rep.converged, rep.fine_sweeps, rep.coarse_sweeps, flush=True)
if "visit" in which:  # multi-sweep coarse visits on several CTAs (sweep-to-sweep hand-off)
    for engine in ("sp", "cl"):
        os.environ["ISMG_COARSE_KERNEL"] = engine
        g = setup_lid_cavity(256, 1000.0).grid
        cfg = CycleConfig(tile=4, tol_fine=1e-300, tol_coarse=1e-300, max_total_sweeps=6)
        s = P.PressureSolver(g, cfg)
        cb = random_field(64, 64, np.random.default_rng(1), -1e-3, 1e-3)
        cb.shift_interior(-cb.interior_mean())
        dcb, dce = P.DeviceField(64, 64, s.ctx, cb), P.DeviceField(64, 64, s.ctx)
        n, rc, ms = s.bench_coarse_visit(dcb, dce, 6, 6)
        print("visit", engine, s.last_stats()["coarse_engine"], n, rc, flush=True)
    os.environ.pop("ISMG_COARSE_KERNEL")
print("ok")
