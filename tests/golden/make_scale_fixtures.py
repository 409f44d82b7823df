"""Reference fixtures at the BASELINE sizes (TEST INFRASTRUCTURE).

Runs the UNMODIFIED reference (oracle/_ref/libismg_ref.so: the reference's own
headers compiled by oracle/build.sh) through `run_case` semantics
(`bench.hpp:127-158`, seed 0, no steady exit) and records, after every
projection step `step()` (`projection.hpp:139-190`):

  * the closed metrics row (`metrics.hpp:61-67`): step, I_f, I_c, NCC_f, NCC_c,
    restrictions, prolongations, converged, N_Lap, residual_final;
  * for u, v, p (reference layout, ghost ring included): the full-array L2 norm
    and the full middle row and column; after step 1 and the last step also a
    strided sample `a[o::s, o::s]`.

Small grids (config 1) store the full fields instead.  The GPU tests
(tests/test_gpu_scale.py) rerun the same steps through the C-ABI and compare
counts exactly and fields within the north star's 1e-10 relative L2.

    python tests/golden/make_scale_fixtures.py c1 c2 jet512 jet1024   # parallel
    python tests/golden/make_scale_fixtures.py c3 c4                  # large, serial

Wall times on this container's Xeon (1 core per case) are printed per step.
Needs /root/reference (this container) — the GPU box only reads the .npz files.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
OUT = os.path.join(HERE, "scale")


def cases():
    """name -> (case factory, tile, steps, sample stride or 0 for full fields, steps per call)."""
    from paper_1309_7128_b200.api import setup_jet, setup_lid_cavity

    def lid(n, re):
        def f():
            c = setup_lid_cavity(n, re)
            c.dt = re / n  # the reference default dt = 1 diverges
            return c
        return f

    def jet(nx, ny):
        return lambda: setup_jet(nx, ny, 0.1, 16)

    return {
        "c1": (lid(256, 100.0), 16, 1500, 0, 1500),       # BASELINE config 1, every step of the run
        "c2": (lid(4096, 1000.0), 32, 3, 16, 1),          # config 2, steps 1-3
        "c3": (lid(16384, 1000.0), 32, 3, 64, 1),         # config 3, steps 1-3
        "jet512": (jet(512, 1024), 16, 12, 4, 1),         # config 4 scaled (coarse 32x64)
        "jet1024": (jet(1024, 2048), 16, 20, 8, 1),       # config 4 scaled (coarse 64x128)
        "c4": (jet(8192, 16384), 16, 1, 64, 1),           # config 4 full size, step 1
    }


def sample(a2d: np.ndarray, s: int, full: bool):
    o = s // 2
    out = {"norm": np.array([np.linalg.norm(a2d)]), "row": a2d[a2d.shape[0] // 2].copy(),
           "col": a2d[:, a2d.shape[1] // 2].copy()}
    if full:  # the strided sample only after step 1 and the last step (keeps the fixtures small)
        out["samp"] = np.ascontiguousarray(a2d[o::s, o::s])
    return out


def run(name: str) -> None:
    from pyoracle import Oracle
    from paper_1309_7128_b200.api import CycleConfig, FluidState

    make, tile, nsteps, stride, per_call = cases()[name]
    c = make()
    g = c.grid
    cfg = CycleConfig(tile=tile)
    st = FluidState(g)
    st.dt, st.nu = c.dt, c.nu
    R = Oracle("reference")
    z = {"meta/grid": np.array([g.nx, g.ny, tile, nsteps, stride]), "meta/dt_nu": np.array([c.dt, c.nu])}
    rows, rowsf = [], []
    done = 0
    t_all = time.time()
    while done < nsteps:
        k = min(per_call, nsteps - done)
        t0 = time.time()
        rr, _ = R.run_steps(g, cfg, st, k)
        for r in rr:
            rows.append([r.step, r.fine_sweeps, r.coarse_sweeps, r.sync_fine, r.sync_coarse, r.restrictions,
                         r.prolongations, int(r.converged)])
            rowsf.append([r.lap_equiv, r.residual_final])
        done += k
        if stride:
            for fname, arr in (("u", st.vel.u_grid), ("v", st.vel.v_grid), ("p", st.p.data.reshape(g.ny + 2, g.nx + 2))):
                for key, val in sample(arr, stride, done in (1, nsteps)).items():
                    z["step%d/%s/%s" % (done, fname, key)] = val
        print("%s: steps ..%d  %.1f s  last row %s" % (name, done, time.time() - t0, rows[-1]), flush=True)
    z["rows"] = np.array(rows, dtype=np.int64)
    z["rowsf"] = np.array(rowsf)
    if not stride:
        z["u"], z["v"], z["p"] = st.vel.u_data.copy(), st.vel.v_data.copy(), st.p.data.copy()
    z["meta/seconds"] = np.array([time.time() - t_all])
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **z)
    print("wrote %s (%.1f KB, %.0f s)" % (path, os.path.getsize(path) / 1024, time.time() - t_all), flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or ["c1", "c2", "jet512", "jet1024"]
    if len(names) == 1:
        run(names[0])
    else:
        procs = [mp.Process(target=run, args=(n,)) for n in names]
        for p in procs:
            p.start()
        for p in procs:
            p.join()
        sys.exit(max(p.exitcode or 0 for p in procs))
