"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and its host-side geometry matches the oracle bit-for-bit."""
import ctypes as C

import numpy as np
import pytest

from cases import cavity, golden_grids, with_side
from paper_1309_7128_b200 import _lib
from paper_1309_7128_b200.api import BoundaryCondition, CycleConfig, GridSpec, Side


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    declared = _lib.header_symbols()
    assert len(declared) >= 50
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) | {"ismg_last_error"} == set(declared)
    assert L.ismg_abi_version() == 1


def test_no_device_is_reported_not_crashed():
    n = C.c_int(-1)
    _lib.call("ismg_device_count", C.byref(n))
    if n.value == 0:
        h = C.c_void_p()
        rc = _lib.lib().ismg_ctx_create(0, None, C.byref(h))
        assert rc == 6  # ISMG_ERR_NO_DEVICE
        assert "device" in _lib.lib().ismg_last_error().decode().lower()


def test_validation_codes_match_reference_exceptions():
    g = GridSpec(nx=0, ny=4)
    with pytest.raises(_lib.InvalidArgument):
        _lib.call("ismg_grid_validate", C.byref(g.to_c()))
    c = CycleConfig(tol_coarse=1e-8)
    with pytest.raises(_lib.InvalidArgument):
        _lib.call("ismg_cycle_validate", C.byref(c.to_c()))
    g = with_side(cavity(8, 8), Side.west, BoundaryCondition.wrap())
    with pytest.raises(_lib.InvalidArgument, match="pair"):
        _lib.call("ismg_grid_validate", C.byref(g.to_c()))
    d = np.zeros(9)
    with pytest.raises(_lib.DomainError):
        _lib.call("ismg_build_fine_diag", C.byref(cavity(1, 1).to_c()), d.ctypes.data_as(_lib.DP), 9)


@pytest.mark.parametrize("name,g", golden_grids(), ids=[n for n, _ in golden_grids()])
def test_host_operators_bit_identical_to_reference(golden, name, g):
    from paper_1309_7128_b200.solver import build_gmg_operator, build_ismg_operator
    assert np.array_equal(build_ismg_operator(g)[2], golden[name + "/ismg_w"])
    assert np.array_equal(build_gmg_operator(g)[2], golden[name + "/gmg_w"])
    d = np.zeros((g.nx + 2) * (g.ny + 2))
    _lib.call("ismg_build_fine_diag", C.byref(g.to_c()), d.ctypes.data_as(_lib.DP), d.size)
    assert np.array_equal(d, golden[name + "/diag"])


def test_large_operator_matches_port(port):
    from paper_1309_7128_b200.solver import build_ismg_operator
    for g in (cavity(4096, 4096, 32), with_side(cavity(1000, 600, 16), Side.north, BoundaryCondition.symmetry())):
        a = build_ismg_operator(g)
        b = port.build_ismg_operator(g)
        assert a[0] == b[0] and np.array_equal(a[2], b[2])
