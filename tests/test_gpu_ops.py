"""GPU parity, op level: each sm_100a kernel, called through the C-ABI, against
the reference's own answers (golden vectors) and the C oracle.

Bit-exact for every op whose arithmetic is per-cell (sweep, residual,
restriction in the op-level serial order, prolongation, coarse GS/residual,
divergence, correction, predictor, BCs). The anchor mean is a fixed-order tree
sum (not the serial sum), so it is checked to 1e-15 relative.
"""
import numpy as np
import pytest

from cases import cavity, golden_grids, periodic_flags, random_field, torus, with_side
from paper_1309_7128_b200.api import (BoundaryCondition, CycleConfig, FluidState, MacVelocity, ScalarField, Scheme,
                                      Side)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import paper_1309_7128_b200 as P
    if P.device_count() < 1:
        pytest.skip("no GPU")
    return P


def solver_for(P, g, scheme=Scheme.ismg):
    return P.PressureSolver(g, CycleConfig(scheme=scheme, tile=g.tile))


@pytest.mark.parametrize("name,g", golden_grids(), ids=[n for n, _ in golden_grids()])
def test_fine_ops_bitwise_vs_golden(dev, golden, name, g):
    P, z = dev, golden
    s = solver_for(P, g)
    x = P.DeviceField.from_host(ScalarField(g.nx, g.ny, z[name + "/x0"]))
    b = P.DeviceField.from_host(ScalarField(g.nx, g.ny, z[name + "/b"]))
    for _ in range(3):
        s.rbgs_sweep(x, b)
    assert np.array_equal(x.download().data, z[name + "/rbgs3"])
    r = P.DeviceField(g.nx, g.ny)
    assert s.fine_residual(x, b, r) == z[name + "/rmax"][0]
    assert np.array_equal(r.download().data, z[name + "/res"])
    assert np.array_equal(x.download().data, z[name + "/x_after_res"])
    s.anchor_mean(x)
    got, want = x.download().data, z[name + "/anchored"]
    assert np.allclose(got, want, rtol=0, atol=1e-15 * max(1.0, np.abs(want).max()))
    # coarse side (ISMG operator of this grid)
    cb = P.DeviceField(s.ncx, s.ncy)
    s.restrict_sum(r, cb)
    assert np.array_equal(cb.download().data, z[name + "/restrict"])
    f = P.DeviceField.from_host(ScalarField(g.nx, g.ny, z[name + "/x0"]))
    s.prolongate_bilinear(cb, f)
    assert np.array_equal(f.download().data, z[name + "/prolong"])
    ce = P.DeviceField(s.ncx, s.ncy)
    for _ in range(5):
        s.gs_sweep_lex(ce, cb)
    assert np.array_equal(ce.download().data, z[name + "/gs5"])
    cr = P.DeviceField(s.ncx, s.ncy)
    assert s.coarse_residual(ce, cb, cr) == z[name + "/crmax"][0]
    assert np.array_equal(cr.download().data, z[name + "/cres"])


@pytest.mark.parametrize("nx,ny,tile", [(256, 256, 16), (1000, 600, 16), (513, 129, 32)])
def test_fine_ops_bitwise_vs_oracle_large(dev, port, nx, ny, tile):
    P = dev
    rng = np.random.default_rng(nx * 7 + ny)
    for g in (cavity(nx, ny, tile), with_side(cavity(nx, ny, tile), Side.north, BoundaryCondition.symmetry())):
        s = solver_for(P, g)
        xh, bh = random_field(nx, ny, rng), random_field(nx, ny, rng)
        x, b = P.DeviceField.from_host(xh), P.DeviceField.from_host(bh)
        for _ in range(2):
            s.rbgs_sweep(x, b)
            port.rbgs_sweep(g, xh, bh)
        assert np.array_equal(x.download().data, xh.data)
        rh, r = ScalarField(nx, ny), P.DeviceField(nx, ny)
        assert s.fine_residual(x, b, r) == port.fine_residual(g, xh, bh, rh)
        assert np.array_equal(r.download().data, rh.data)
        cbh, cb = ScalarField(s.ncx, s.ncy), P.DeviceField(s.ncx, s.ncy)
        port.restrict_sum(g, rh, cbh)
        s.restrict_sum(r, cb)
        assert np.array_equal(cb.download().data, cbh.data)
        port.prolongate_bilinear(g, cbh, xh)
        s.prolongate_bilinear(cb, x)
        assert np.array_equal(x.download().data, xh.data)
        _, _, w = port.build_ismg_operator(g)
        px, py = periodic_flags(g)
        ceh, ce = ScalarField(s.ncx, s.ncy), P.DeviceField(s.ncx, s.ncy)
        for _ in range(3):
            port.gs_sweep_lex(w, px, py, 0, ceh, cbh)
            s.gs_sweep_lex(ce, cb)
        assert np.array_equal(ce.download().data, ceh.data)


def test_projection_kernels_bitwise(dev, port):
    P = dev
    rng = np.random.default_rng(5)
    grids = [cavity(37, 29), torus(24, 16),
             with_side(with_side(with_side(cavity(30, 20), Side.west, BoundaryCondition.wrap()), Side.east,
                                 BoundaryCondition.wrap()), Side.south, BoundaryCondition.inflow(0.1, 5, 7)),
             with_side(with_side(cavity(19, 33), Side.north, BoundaryCondition.moving_wall(0.1, 0.02)), Side.west,
                       BoundaryCondition.symmetry())]
    for g in grids:
        vel = MacVelocity(g.nx, g.ny)
        vel.u_data[:] = rng.uniform(-0.05, 0.05, vel.u_data.size)
        vel.v_data[:] = rng.uniform(-0.05, 0.05, vel.v_data.size)
        p = random_field(g.nx, g.ny, rng, -0.05, 0.05, ghosts=True)
        dv = P.DeviceVelocity(g.nx, g.ny, host=vel)
        dpf = P.DeviceField.from_host(p)
        port.apply_velocity_bc(g, vel)
        P.apply_velocity_bc(dv, g)
        got = dv.download()
        assert np.array_equal(got.u_data, vel.u_data) and np.array_equal(got.v_data, vel.v_data)
        port.apply_scalar_bc(g, p)
        P.apply_scalar_bc(dpf, g)
        assert np.array_equal(dpf.download().data, p.data)
        out = vel.copy()
        dout = P.DeviceVelocity(g.nx, g.ny, host=out)
        port.predictor(g, vel, p, 0.7, 0.03, out)
        P.predictor(dv, dpf, 0.7, 0.03, g, dout)
        got = dout.download()
        assert np.array_equal(got.u_data, out.u_data) and np.array_equal(got.v_data, out.v_data)
        div, ddiv = ScalarField(g.nx, g.ny), P.DeviceField(g.nx, g.ny)
        port.divergence(g, vel, div)
        P.divergence(dv, g, ddiv)
        assert np.array_equal(ddiv.download().data, div.data)
        dp = random_field(g.nx, g.ny, rng)
        ddp = P.DeviceField.from_host(dp)
        port.correct(g, vel, dp, 0.9)
        P.correct(dv, ddp, 0.9, g)
        got = dv.download()
        assert np.array_equal(got.u_data, vel.u_data) and np.array_equal(got.v_data, vel.v_data)
        assert np.array_equal(ddp.download().data, dp.data)
