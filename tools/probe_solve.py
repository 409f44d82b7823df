"""Quick timing probe: projection steps of a lid cavity on the GPU (not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1309_7128_b200 as P
from paper_1309_7128_b200.api import CycleConfig, RunMetrics, setup_lid_cavity

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 32
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
mode = int(sys.argv[4]) if len(sys.argv) > 4 else 0
case = setup_lid_cavity(n, 1000.0)
case.dt = 1000.0 / n
cfg = CycleConfig(tile=tile)
solver = P.PressureSolver(case.grid, cfg)
st = P.api.FluidState(case.grid); st.dt, st.nu = case.dt, case.nu
ds = P.DeviceState(case.grid, solver.ctx, st)
m = RunMetrics(n * n)
for k in range(steps):
    t0 = time.perf_counter()
    rep = ds.step(solver, m)
    t1 = time.perf_counter()
    s = solver.last_stats()
    r = m.rows[-1]
    print("step %d: %.1f ms wall, solve %.1f ms | I_f %d I_c %d restr %d prol %d conv %d res %.3e | %.2f Gcell-upd/s | syncs %d launches %d"
          % (k + 1, (t1 - t0) * 1e3, s["solve_ms"], r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations,
             r.converged, r.residual_final, r.fine_sweeps * n * n / (s["solve_ms"] * 1e-3) / 1e9, s["host_syncs"], s["kernel_launches"]), flush=True)
    if os.environ.get("VISITS"):
        v = solver.visit_log()
        cs = [c for c, f in v]
        print("  visits %d: coarse sweeps first 12 %s; max %d; >=64: %d; zero: %d" % (len(v), cs[:12], max(cs), sum(c >= 64 for c in cs), sum(c == 0 for c in cs)))
