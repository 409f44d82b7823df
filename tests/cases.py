"""Shared parity cases (grids, seeded inputs) for the oracle and GPU tests."""
from __future__ import annotations

import numpy as np

from paper_1309_7128_b200.api import (
    BcKind, BoundaryCondition, GridSpec, ScalarField, Side, all_sides)


def cavity(nx, ny, tile=16):
    return GridSpec(nx=nx, ny=ny, tile=tile)


def torus(nx, ny, tile=16):
    g = GridSpec(nx=nx, ny=ny, tile=tile)
    for s in all_sides:
        g.set_side(s, BoundaryCondition.wrap())
    return g


def with_side(g, s, b):
    g = g.copy()
    g.set_side(s, b)
    return g


def periodic_flags(g):
    return (g.side(Side.west).kind == BcKind.periodic, g.side(Side.south).kind == BcKind.periodic)


def random_field(nx, ny, rng, lo=-1.0, hi=1.0, ghosts=False):
    """Seeded uniform field; ghosts stay zero (as after ScalarField(nx, ny)) unless ghosts=True."""
    if ghosts:
        return ScalarField(nx, ny, rng.uniform(lo, hi, (nx + 2) * (ny + 2)))
    f = ScalarField(nx, ny)
    f.interior()[:] = rng.uniform(lo, hi, (ny, nx))
    return f


def golden_grids():
    """Same list as tests/golden/make_golden.py (kept in one place there)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "make_golden", os.path.join(os.path.dirname(__file__), "golden", "make_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.golden_grids()


def a3_rhs(n: int) -> ScalarField:
    """acceptance.cpp:162-207 frozen instance: XorShift64 noise with the cos
    modes kx, ky <= 4 projected out, zero mean, amplitude 1e-4."""
    import math
    s = 0x243F6A8885A308D3
    mask = (1 << 64) - 1
    b = ScalarField(n, n)
    vals = np.empty(n * n)
    for k in range(n * n):
        s ^= (s << 13) & mask
        s ^= s >> 7
        s ^= (s << 17) & mask
        vals[k] = float(s >> 11) * 2.0 ** -53 * 2.0 - 1.0
    bi = b.interior()
    bi[:] = vals.reshape(n, n)
    for kx in range(5):
        for ky in range(5):
            num = den = 0.0
            phi = np.empty((n, n))
            for j in range(n):
                for i in range(n):
                    phi[j, i] = math.cos(math.pi * kx * (i + 0.5) / n) * math.cos(math.pi * ky * (j + 0.5) / n)
            for j in range(n):
                for i in range(n):
                    num += bi[j, i] * phi[j, i]
                    den += phi[j, i] * phi[j, i]
            a = num / den
            for j in range(n):
                for i in range(n):
                    bi[j, i] -= a * math.cos(math.pi * kx * (i + 0.5) / n) * math.cos(math.pi * ky * (j + 0.5) / n)
    b.shift_interior(-b.interior_mean())
    scale = 1e-4 / b.interior_max_abs()
    bi *= scale
    b.shift_interior(-b.interior_mean())
    return b
