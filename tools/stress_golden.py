"""Stress the golden solves: repeat every golden grid x scheme solve N times (argv[1]) and print
every count mismatch with the solver stats. A rare b = 0 upload race (legacy-stream memset
against the non-blocking context stream) showed here as 1-2 mismatches in 465 solves; 0 in 1240
after ISMG_ZERO / ISMG_H2D (profiles/r02_stress_golden.log).

    python tools/stress_golden.py 40 [grid]
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_1309_7128_b200 as P
from cases import golden_grids
from paper_1309_7128_b200.api import CycleConfig, RunMetrics, ScalarField, Scheme
z = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
only = sys.argv[2] if len(sys.argv) > 2 else None
bad = tot = 0
for it in range(reps):
    for name, g in golden_grids():
        if only and name != only:
            continue
        bb = ScalarField(g.nx, g.ny, z[name + "/b"].copy())
        bb.shift_interior(-bb.interior_mean())
        for s in Scheme:
            key = "%s/solve_%d" % (name, int(s))
            if key + "/x" not in z:
                continue
            cfg = CycleConfig(scheme=s, tile=g.tile, depth=3, tol_fine=1e-9, tol_coarse=1e-8, max_total_sweeps=4000)
            solver = P.PressureSolver(g, cfg)
            m = RunMetrics(g.nx * g.ny)
            x = ScalarField(g.nx, g.ny)
            rep = solver.solve(x, bb, m)
            counts = [int(rep.converged), rep.fine_sweeps, rep.coarse_sweeps, m.current.restrictions, m.current.prolongations]
            tot += 1
            if counts != z[key + "/counts"].tolist():
                bad += 1
                print("MISMATCH it %d %s %s got %s want %s stats %s residual %r" % (
                    it, name, s, counts, z[key + "/counts"].tolist(), solver.last_stats(), rep.residual), flush=True)
print("mismatches %d of %d" % (bad, tot), flush=True)
