"""Coarse-visit profiling probe: one lid-cavity step with a capped sweep budget."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_7128_b200 as P
from paper_1309_7128_b200.api import CycleConfig, FluidState, RunMetrics, setup_lid_cavity

n, tile, budget = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
tol_c = float(sys.argv[4]) if len(sys.argv) > 4 else None  # e.g. 1e-300: the visit runs the whole budget
case = setup_lid_cavity(n, 1000.0)
case.dt = 1000.0 / n
cfg = CycleConfig(tile=tile, max_total_sweeps=budget)
if tol_c is not None:
    cfg.tol_coarse = tol_c
    cfg.tol_fine = min(cfg.tol_fine, tol_c)
solver = P.PressureSolver(case.grid, cfg)
st = FluidState(case.grid); st.dt, st.nu = case.dt, case.nu
ds = P.DeviceState(case.grid, solver.ctx, st)
m = RunMetrics(n * n)
ds.step(solver, m)
s = solver.last_stats()
print("solve %.1f ms, coarse %.1f ms over %d wavefront steps (%.2f us/step), I_f %d I_c %d, visits %s"
      % (s["solve_ms"], s["coarse_ms"], s["coarse_steps"], 1e3 * s["coarse_ms"] / max(1, s["coarse_steps"]),
         m.rows[-1].fine_sweeps, m.rows[-1].coarse_sweeps, solver.visit_log()[:4]))
