"""GPU parity of the fused fine-pass kernels (column pairs, fine_pass.cu; one-warp
strips of column quads, fine_pass_w.cu) on grids wider than one CTA strip, with ragged widths,
several row-chunk heights and every fast/generic path split: interior strips,
boundary strips, partial last strips and the halo recompute between strips.

Non-singular grids (a Dirichlet side, no anchoring) make the fused pass a pure
red-black sweep per cell, so x after N passes must equal the oracle's N
rbgs_sweep calls bit for bit. Whole solves are checked against the oracle's
counts and fields.
"""
import numpy as np
import pytest

from cases import cavity, random_field, with_side
from paper_1309_7128_b200.api import BoundaryCondition, CycleConfig, RunMetrics, ScalarField, Side

pytestmark = pytest.mark.gpu
REL_L2 = 1e-10

GRIDS = [(1100, 70, 4), (1030, 41, 8), (1536, 64, 32), (2051, 37, 16), (96, 33, 4), (515, 20, 2)]


@pytest.fixture(scope="module")
def dev():
    import paper_1309_7128_b200 as P
    if P.device_count() < 1:
        pytest.skip("no GPU")
    return P


def rel_l2(a, b):
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


@pytest.mark.parametrize("kernel", ["warp", "pair"])
@pytest.mark.parametrize("rows", ["8", "16", "64", "96", "default"])
@pytest.mark.parametrize("nx,ny,tile", GRIDS)
def test_fine_pass_bitwise_vs_oracle_sweeps(dev, port, monkeypatch, kernel, rows, nx, ny, tile):
    P = dev
    monkeypatch.setenv("ISMG_FINE_KERNEL", kernel)
    if rows != "default":
        monkeypatch.setenv("ISMG_FINE_H", rows)
    g = with_side(cavity(nx, ny, tile), Side.west, BoundaryCondition.symmetry())
    rng = np.random.default_rng(nx * 7 + ny)
    x0, b = random_field(nx, ny, rng), random_field(nx, ny, rng)
    solver = P.PressureSolver(g, CycleConfig(tile=tile))
    xd, bd = P.DeviceField.from_host(x0), P.DeviceField.from_host(b)
    npass = 5
    solver.bench_fine_pass(xd, bd, npass)
    want = ScalarField(nx, ny, x0.data.copy())
    for _ in range(npass):
        port.rbgs_sweep(g, want, b)
    assert np.array_equal(xd.download().interior(), want.interior())


@pytest.mark.parametrize("kernel", ["warp", "pair"])
@pytest.mark.parametrize("nx,ny,tile,side", [(1100, 70, 4, None), (1030, 41, 8, Side.east), (1536, 64, 32, None),
                                             (2051, 37, 16, Side.north)])
def test_wide_solves_match_oracle(dev, port, monkeypatch, kernel, nx, ny, tile, side):
    P = dev
    monkeypatch.setenv("ISMG_FINE_KERNEL", kernel)
    monkeypatch.setenv("ISMG_FINE_H", "16")
    g = cavity(nx, ny, tile)
    if side is not None:
        g = with_side(g, side, BoundaryCondition.symmetry())
    rng = np.random.default_rng(5)
    b = random_field(nx, ny, rng)
    if side is None:
        b.shift_interior(-b.interior_mean())
    cfg = CycleConfig(tile=tile, tol_fine=1e-9, tol_coarse=1e-8, max_total_sweeps=3000)
    m = RunMetrics(nx * ny)
    x = ScalarField(nx, ny)
    rep = P.PressureSolver(g, cfg).solve(x, b, m)
    xr = ScalarField(nx, ny)
    rr, mr, _ = port.solve(g, cfg, xr, b)
    got = (int(rep.converged), rep.fine_sweeps, rep.coarse_sweeps, m.current.restrictions, m.current.prolongations)
    want = (int(rr.converged), rr.fine_sweeps, rr.coarse_sweeps, mr.restrictions, mr.prolongations)
    assert got == want
    assert rel_l2(x.interior(), xr.interior()) <= REL_L2
