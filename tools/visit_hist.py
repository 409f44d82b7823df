"""Visit-length histogram of lid-cavity projection steps (coarse sweeps per visit)."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_7128_b200 as P
from paper_1309_7128_b200.api import CycleConfig, FluidState, RunMetrics, setup_lid_cavity

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 32
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
case = setup_lid_cavity(n, 1000.0)
case.dt = 1000.0 / n
solver = P.PressureSolver(case.grid, CycleConfig(tile=tile))
st = FluidState(case.grid); st.dt, st.nu = case.dt, case.nu
ds = P.DeviceState(case.grid, solver.ctx, st)
m = RunMetrics(n * n)
for k in range(steps):
    ds.step(solver, m)
    s = solver.last_stats()
    v = solver.visit_log()
    cs = [c for c, f in v]
    fs = [f for c, f in v]
    buckets = collections.Counter()
    for c in cs:
        b = 0 if c == 0 else (1 << (c.bit_length() - 1))
        buckets[b] += 1
    tot = sum(cs)
    print("step %d: solve %.1f ms (coarse %.1f ms, %d wavefront steps, %.2f us/step), visits %d, coarse sweeps %d, fine %d"
          % (k + 1, s["solve_ms"], s["coarse_ms"], s["coarse_steps"], 1e3 * s["coarse_ms"] / max(1, s["coarse_steps"]),
             len(v), tot, sum(fs)))
    print("  visits by sweeps (pow2 bucket: count, sweeps):",
          ", ".join("%d:%d/%d" % (b, buckets[b], sum(c for c in cs if (0 if c == 0 else 1 << (c.bit_length() - 1)) == b))
                    for b in sorted(buckets)))
    print("  first 20 visits:", v[:20])
