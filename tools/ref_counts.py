"""Full-size parity of iteration counts: the compiled reference (oracle/_ref) on
BASELINE config 2 (lid 4096^2, Re 1000, dt = Re/n, tile 32), steps 1..K on one
host core; prints the per-step (I_f, I_c, restrictions, prolongations) to compare
with tools/visit_hist.py on the GPU. Needs /root/reference (this container).

    python tools/ref_counts.py 4096 2        # ~10 minutes
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import Oracle  # noqa: E402
from paper_1309_7128_b200.api import CycleConfig, FluidState, setup_lid_cavity  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
case = setup_lid_cavity(n, 1000.0)
case.dt = 1000.0 / n
st = FluidState(case.grid)
st.dt, st.nu = case.dt, case.nu
t0 = time.time()
rows, secs = Oracle("reference").run_steps(case.grid, CycleConfig(tile=32), st, steps)
for r in rows:
    print("ref step: I_f %d I_c %d restr %d prol %d conv %d" % (r.fine_sweeps, r.coarse_sweeps, r.restrictions,
                                                               r.prolongations, r.converged), flush=True)
print("seconds", secs if secs is not None else time.time() - t0)
