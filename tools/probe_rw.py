"""Coarse-visit cost of the fused engine: one visit of a fixed number of sweeps
(tol 1e-300) on the coarse level of lid n^2 / tile, one group (first = budget),
CUDA-event time per visit; ISMG_RW_TRACE=1 adds the slow-path counters."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_1309_7128_b200 as P
from cases import random_field
from paper_1309_7128_b200.api import CycleConfig, setup_lid_cavity
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 32
g = setup_lid_cavity(n, 1000.0).grid
ncx = (n + tile - 1) // tile
BUDGETS = [int(x) for x in os.environ.get("PROBE_BUDGETS", "1,2,4,8,32,128,512,2048").split(",")]
for budget in BUDGETS:
    cfg = CycleConfig(tile=tile, tol_fine=1e-300, tol_coarse=1e-300, max_total_sweeps=budget)
    s = P.PressureSolver(g, cfg)
    cb = random_field(ncx, ncx, np.random.default_rng(1), -1e-3, 1e-3)
    cb.shift_interior(-cb.interior_mean())
    dcb, dce = P.DeviceField(ncx, ncx, s.ctx, cb), P.DeviceField(ncx, ncx, s.ctx)
    s.bench_coarse_visit(dcb, dce, budget, budget)
    ms = min(s.bench_coarse_visit(dcb, dce, budget, budget)[2] for _ in range(3))
    print("coarse %d^2 engine %d: %5d sweeps in one group: %8.3f ms  (%.2f us/sweep)"
          % (ncx, s.last_stats()["coarse_engine"], budget, ms, 1e3 * ms / budget), flush=True)
    if os.environ.get("ISMG_SP_TRACE"):  # a -DISMG_SP_TRACE build: CTA 0's phase clock per visit
        import ctypes
        from paper_1309_7128_b200 import _lib
        tr = (ctypes.c_ulonglong * 6)()
        _lib.lib().ismg_debug_sp_trace(tr)  # reset, then one more visit
        s.bench_coarse_visit(dcb, dce, budget, budget)
        _lib.lib().ismg_debug_sp_trace(tr)
        v = max(1, tr[5])
        print("   phases (us per visit): setup %.1f  sweep0 %.1f  rest %.1f  gridsync %.1f  write %.1f  (visits %d)"
              % tuple([tr[i] / v / 1e3 for i in range(5)] + [tr[5]]), flush=True)
