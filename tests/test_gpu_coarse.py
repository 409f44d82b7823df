"""GPU parity of ONE coarse visit (cycles.hpp:120-137) for every coarse-visit
kernel of the fused path, through the ismg_bench_coarse_visit hook: the
visit's iterate against the oracle's gs_sweep_lex (coarsening.hpp:552-567)
repeated the same number of times, and its stop sweep against the oracle's
coarse_residual test (coarsening.hpp:531-549) after every sweep.

The kernels relax in the reference's lexicographic order, so a non-singular
level (the jet: fixed-pressure top) must match bit for bit; a singular level
(the lid cavity) is anchored once per visit instead of after every sweep, so
it matches to round-off of the mean.
"""
import numpy as np
import pytest

from cases import periodic_flags, random_field
from paper_1309_7128_b200.api import CycleConfig, GridSpec, ScalarField, setup_jet, setup_lid_cavity

pytestmark = pytest.mark.gpu
ENGINES = {"global": 0, "smem": 1, "tmem": 2, "cl": 3, "rw": 4, "sp": 5, "sp2": 6}


@pytest.fixture(scope="module")
def dev():
    import paper_1309_7128_b200 as P
    if P.device_count() < 1:
        pytest.skip("no GPU")
    return P


def level(name):
    if name == "lid256":
        return setup_lid_cavity(256, 1000.0).grid, 4, True
    if name == "lid512":
        return setup_lid_cavity(512, 1000.0).grid, 4, True
    if name == "jet256":
        return setup_jet(256, 512, 0.1, 8).grid, 4, False
    if name == "jet512t8":
        return setup_jet(512, 1024, 0.1, 16).grid, 8, False
    if name == "lid520":  # 130 x 130: five 32-row blocks, the last of 2 rows
        return setup_lid_cavity(520, 1000.0).grid, 4, True
    if name == "jet200x600":  # 50 x 150: ncy not a multiple of 32, rectangular
        return setup_jet(200, 600, 0.1, 8).grid, 4, False
    if name == "lid2048":  # 512 x 512: sixteen blocks (config 3's coarse level)
        return setup_lid_cavity(2048, 1000.0).grid, 4, True
    if name == "jet4096t8":  # 512 x 1024: config 4's coarse level (32 blocks)
        return setup_jet(4096, 8192, 0.1, 64).grid, 8, False
    raise KeyError(name)


def oracle_visit(port, w, px, py, cb, sweeps, tol, singular):
    """cycles.hpp:122-132 with the anchor applied once at the end (as the kernels do)."""
    ce = ScalarField(cb.nx, cb.ny)
    rc = port.coarse_residual(w, px, py, 0, ce, cb)
    k = 0
    while rc > tol and k < sweeps:
        port.gs_sweep_lex(w, px, py, 0, ce, cb)
        rc = port.coarse_residual(w, px, py, 0, ce, cb)
        k += 1
    if singular and k > 0:
        ce.shift_interior(-ce.interior_mean())
    return ce, k, rc


@pytest.mark.parametrize("engine", ["sp", "sp2", "rw", "cl", "tmem", "smem", "global"])
@pytest.mark.parametrize("name", ["jet256", "lid256", "lid512", "jet512t8", "lid520", "jet200x600", "lid2048",
                                  "jet4096t8"])
@pytest.mark.parametrize("budget,first", [(1, 1), (5, 3), (37, 32), (100, 7)])
def test_fixed_length_visit(dev, port, monkeypatch, engine, name, budget, first):
    P = dev
    monkeypatch.setenv("ISMG_COARSE_KERNEL", engine)
    g, tile, singular = level(name)
    cfg = CycleConfig(tile=tile, tol_fine=1e-300, tol_coarse=1e-300, max_total_sweeps=budget)
    solver = P.PressureSolver(g, cfg)
    gt = g.copy()
    gt.tile = tile
    ncx, ncy, w = port.build_ismg_operator(gt)
    px, py = periodic_flags(g)
    cb = random_field(ncx, ncy, np.random.default_rng(ncx + budget), -1e-3, 1e-3)
    if singular:
        cb.shift_interior(-cb.interior_mean())
    dcb, dce = P.DeviceField(ncx, ncy, solver.ctx, cb), P.DeviceField(ncx, ncy, solver.ctx)
    try:
        n, rc, ms = solver.bench_coarse_visit(dcb, dce, budget, first)
    except Exception as e:  # the engine has no plan for this level
        pytest.skip("engine %s: %s" % (engine, e))
    if solver.last_stats()["coarse_engine"] != ENGINES[engine]:
        pytest.skip("engine %s has no plan for %s (fell back to %d)" % (engine, name,
                                                                       solver.last_stats()["coarse_engine"]))
    want, k, rc_want = oracle_visit(port, w, px, py, cb, budget, 1e-300, singular)
    got = dce.download()
    assert n == budget == k
    if singular:
        d = got.interior() - want.interior()
        assert np.linalg.norm(d) <= 1e-12 * np.linalg.norm(want.interior())
    else:
        assert np.array_equal(got.interior(), want.interior())
        assert rc == rc_want


@pytest.mark.parametrize("engine", ["sp", "sp2", "rw", "cl"])
@pytest.mark.parametrize("name", ["jet256", "lid256", "lid512"])
@pytest.mark.parametrize("first", [1, 4, 32])
def test_visit_stops_at_the_reference_sweep(dev, port, monkeypatch, engine, name, first):
    """tol_coarse reached mid-group: the kernel stops at the reference's sweep
    (checkpoint and replay), whatever the first group's size."""
    P = dev
    monkeypatch.setenv("ISMG_COARSE_KERNEL", engine)
    g, tile, singular = level(name)
    gt = g.copy()
    gt.tile = tile
    ncx, ncy, w = port.build_ismg_operator(gt)
    px, py = periodic_flags(g)
    cb = random_field(ncx, ncy, np.random.default_rng(3 + first), -1e-3, 1e-3)
    if singular:
        cb.shift_interior(-cb.interior_mean())
    # a tolerance the oracle reaches after about 60 sweeps
    ce = ScalarField(ncx, ncy)
    for _ in range(60):
        port.gs_sweep_lex(w, px, py, 0, ce, cb)
    tol = port.coarse_residual(w, px, py, 0, ce, cb) * 1.0000001
    cfg = CycleConfig(tile=tile, tol_fine=tol, tol_coarse=tol, max_total_sweeps=20000)
    solver = P.PressureSolver(g, cfg)
    dcb, dce = P.DeviceField(ncx, ncy, solver.ctx, cb), P.DeviceField(ncx, ncy, solver.ctx)
    n, rc, ms = solver.bench_coarse_visit(dcb, dce, 20000, first)
    if solver.last_stats()["coarse_engine"] != ENGINES[engine]:
        pytest.skip("engine %s has no plan for %s" % (engine, name))
    want, k, rc_want = oracle_visit(port, w, px, py, cb, 20000, tol, singular)
    assert n == k
    got = dce.download()
    if singular:
        d = got.interior() - want.interior()
        assert np.linalg.norm(d) <= 1e-12 * np.linalg.norm(want.interior())
    else:
        assert np.array_equal(got.interior(), want.interior())
