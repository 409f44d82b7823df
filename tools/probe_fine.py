"""Fine-pass probe: N fused sweep passes on the 4096^2 lid-cavity first-step rhs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_7128_b200 as P
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
case, cfg = bench.workload(n)
g = case.grid
solver = P.PressureSolver(g, cfg)
x, b = P.DeviceField(n, n), P.DeviceField(n, n)
vel, vstar, pf = P.DeviceVelocity(n, n), P.DeviceVelocity(n, n), P.DeviceField(n, n)
P.apply_velocity_bc(vel, g)
vstar.upload(vel.download())
P.predictor(vel, pf, case.dt, case.nu, g, vstar)
P.apply_velocity_bc(vstar, g)
P.divergence(vstar, g, b, g.h * g.h / case.dt)
solver.bench_fine_pass(x, b, 1)  # warm-up (module load)
ms = solver.bench_fine_pass(x, b, iters)
print("fine pass %dx%d: %.1f us/pass, %.0f GB/s algorithmic (24 B/cell)" % (n, n, ms * 1e3, 24.0 * n * n / (ms * 1e-3) / 1e9))
