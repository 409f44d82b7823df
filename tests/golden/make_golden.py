"""Generate golden input/output vectors from the UNMODIFIED reference.

Run here (where /root/reference exists) after `oracle/build.sh`:

    python tests/golden/make_golden.py

It drives oracle/_ref/libismg_ref.so — the reference's own headers compiled
by include path — on small seeded cases and writes tests/golden/golden.npz.
The GPU box has no /root/reference; the committed .npz carries the reference's
answers there. Every array is produced by the reference itself; the inputs are
seeded numpy draws.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from pyoracle import Oracle, OracleError  # noqa: E402

from paper_1309_7128_b200.api import (  # noqa: E402
    BcKind, BoundaryCondition, CycleConfig, FluidState, GridSpec, ScalarField, Scheme, Side, all_sides,
    setup_channel_jets, setup_jet, setup_lid_cavity)


def golden_grids():
    """(name, GridSpec) pairs covering every boundary kind and short tiles."""
    out = []
    out.append(("cav7x5", GridSpec(nx=7, ny=5, tile=2)))
    g = GridSpec(nx=6, ny=4, tile=2)
    g.set_side(Side.west, BoundaryCondition.wrap()).set_side(Side.east, BoundaryCondition.wrap())
    out.append(("perx6x4", g))
    g = GridSpec(nx=6, ny=4, tile=2)
    for s in all_sides:
        g.set_side(s, BoundaryCondition.wrap())
    out.append(("torus6x4", g))
    g = GridSpec(nx=5, ny=6, tile=2)
    g.set_side(Side.north, BoundaryCondition.symmetry(0.0)).set_side(Side.south, BoundaryCondition.inflow(0.1, 1, 3))
    out.append(("inlet5x6", g))
    g = GridSpec(nx=20, ny=12, tile=8)
    g.set_side(Side.south, BoundaryCondition.inflow(0.1, 8, 4)).set_side(Side.north, BoundaryCondition.symmetry(0.0))
    out.append(("pad20x12", g))
    g = GridSpec(nx=37, ny=29, tile=8)
    g.set_side(Side.west, BoundaryCondition.symmetry(0.0))
    out.append(("sym37x29", g))
    g = GridSpec(nx=40, ny=21, tile=4)
    g.set_side(Side.west, BoundaryCondition.wrap()).set_side(Side.east, BoundaryCondition.wrap())
    g.set_side(Side.north, BoundaryCondition.symmetry(0.0))
    out.append(("chan40x21", g))
    g = GridSpec(nx=64, ny=48, tile=16)
    out.append(("cav64x48", g))
    return out


def main():
    R = Oracle("reference")
    rng = np.random.default_rng(20260918)
    z = {}
    for name, g in golden_grids():
        n = (g.nx + 2) * (g.ny + 2)
        x0 = rng.uniform(-1, 1, n)
        b = rng.uniform(-1, 1, n)
        z[name + "/x0"], z[name + "/b"] = x0, b
        x = ScalarField(g.nx, g.ny, x0.copy())
        B = ScalarField(g.nx, g.ny, b)
        for k in range(3):
            R.rbgs_sweep(g, x, B)
        z[name + "/rbgs3"] = x.data.copy()
        r = ScalarField(g.nx, g.ny)
        z[name + "/rmax"] = np.array([R.fine_residual(g, x, B, r)])
        z[name + "/res"] = r.data.copy()
        z[name + "/x_after_res"] = x.data.copy()  # periodic ghosts refreshed
        R.anchor_mean(g, x)
        z[name + "/anchored"] = x.data.copy()
        z[name + "/diag"] = R.build_fine_diag(g).data.copy()
        ncx, ncy, w = R.build_ismg_operator(g)
        z[name + "/ismg_w"] = w.copy()
        z[name + "/gmg_w"] = R.build_gmg_operator(g)[2].copy()
        cb = ScalarField(ncx, ncy)
        R.restrict_sum(g, r, cb)
        z[name + "/restrict"] = cb.data.copy()
        f = ScalarField(g.nx, g.ny, x0.copy())
        R.prolongate_bilinear(g, cb, f)
        z[name + "/prolong"] = f.data.copy()
        px = g.side(Side.west).kind == BcKind.periodic
        py = g.side(Side.south).kind == BcKind.periodic
        ce = ScalarField(ncx, ncy)
        for k in range(5):
            R.gs_sweep_lex(w, px, py, 0, ce, cb)
        z[name + "/gs5"] = ce.data.copy()
        cr = ScalarField(ncx, ncy)
        z[name + "/crmax"] = np.array([R.coarse_residual(w, px, py, 0, ce, cb, cr)])
        z[name + "/cres"] = cr.data.copy()
        # full solves, every scheme, on a zero-mean rhs
        bb = ScalarField(g.nx, g.ny, b.copy())
        bb.shift_interior(-bb.interior_mean())
        for scheme in (Scheme.plain_gs, Scheme.ismg, Scheme.gmg, Scheme.acm):
            if scheme == Scheme.acm and min(g.nx, g.ny) < 4:
                continue
            cfg = CycleConfig(scheme=scheme, tile=g.tile, depth=3, tol_fine=1e-9, tol_coarse=1e-8,
                              max_total_sweeps=4000)
            X = ScalarField(g.nx, g.ny)
            key = "%s/solve_%d" % (name, int(scheme))
            try:
                rep, cur, _ = R.solve(g, cfg, X, bb)
            except OracleError as e:  # the reference's own exception, kept as the golden answer
                z[key + "/error"] = np.array([e.code])
                continue
            z[key + "/x"] = X.data.copy()
            z[key + "/counts"] = np.array([rep.converged, rep.fine_sweeps, rep.coarse_sweeps, cur.restrictions,
                                           cur.prolongations], dtype=np.int64)
            z[key + "/scalars"] = np.array([rep.residual, cur.lap_equiv])
    # multi-step projection runs (step rows + final fields)
    cases = []
    c = setup_lid_cavity(32, 100.0)
    c.dt = 100.0 / 32
    cases.append(("lid32", c, CycleConfig(tile=8), 25))
    c = setup_jet(32, 64, 0.1, 8)
    cases.append(("jet32x64", c, CycleConfig(tile=8), 12))
    c = setup_channel_jets(24, 48, 0.1, 6)
    cases.append(("chan24x48", c, CycleConfig(tile=8), 8))
    for name, c, cfg, nsteps in cases:
        st = FluidState(c.grid)
        st.dt, st.nu = c.dt, c.nu
        rows, _ = R.run_steps(c.grid, cfg, st, nsteps)
        z["run/%s/rows" % name] = np.array(
            [[r.step, r.fine_sweeps, r.coarse_sweeps, r.sync_fine, r.sync_coarse, r.restrictions, r.prolongations,
              int(r.converged)] for r in rows], dtype=np.int64)
        z["run/%s/rowsf" % name] = np.array([[r.lap_equiv, r.residual_final] for r in rows])
        z["run/%s/u" % name] = st.vel.u_data.copy()
        z["run/%s/v" % name] = st.vel.v_data.copy()
        z["run/%s/p" % name] = st.p.data.copy()
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **z)
    print("wrote %s (%d arrays, %.1f KB)" % (path, len(z), os.path.getsize(path) / 1024))


if __name__ == "__main__":
    main()
