"""Debug: one coarse visit of the register-wavefront engine with its per-group
residual maxima (ISMG_RW_TRACE) next to the oracle's per-sweep coarse residuals."""
import os, sys
os.environ["ISMG_RW_TRACE"] = "1"
os.environ["ISMG_COARSE_KERNEL"] = "rw"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_1309_7128_b200 as P
from pyoracle import Oracle
from cases import random_field
from paper_1309_7128_b200.api import CycleConfig, ScalarField, setup_jet
first = int(sys.argv[1]) if len(sys.argv) > 1 else 32
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 40
g = setup_jet(256, 512, 0.1, 8).grid
g.tile = 4
port = Oracle("port")
ncx, ncy, w = port.build_ismg_operator(g)
cb = random_field(ncx, ncy, np.random.default_rng(3 + first), -1e-3, 1e-3)
ce = ScalarField(ncx, ncy)
ref = []
for k in range(budget):
    port.gs_sweep_lex(w, 0, 0, 0, ce, cb)
    ref.append(port.coarse_residual(w, 0, 0, 0, ce, cb))
cfg = CycleConfig(tile=4, tol_fine=1e-300, tol_coarse=1e-300, max_total_sweeps=budget)
s = P.PressureSolver(g, cfg)
dcb, dce = P.DeviceField(ncx, ncy, s.ctx, cb), P.DeviceField(ncx, ncy, s.ctx)
print("ref residuals:", " ".join("%.17g" % v for v in ref), flush=True)
print(s.bench_coarse_visit(dcb, dce, budget, first), flush=True)
