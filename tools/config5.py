"""BASELINE config 5: ISM vs ACM on an all-Neumann n x n Poisson problem —
synchronisation events and time to tolerance (north star:
"the number of synchronisation events per solve is counted and reported
against ACM").

    python tools/config5.py [n=8192] [out.json]

rhs = the A3 recipe of acceptance.cpp:162-207 scaled to n: XorShift64 noise
(seed 0x243F6A8885A308D3) in [-1, 1), the cos modes kx, ky <= 4 projected out,
zero mean, amplitude 1e-4. ISM: two-level, 32h tiles; ACM: depth 6 (32h
coarsest). tol_fine 1e-6 (tol_coarse 1e-5). Reported per scheme: converged,
I_f, I_c, the reference's model sync counts NCC_f / NCC_c (metrics.hpp:46-58),
the lap-equivalent work N_Lap, and this implementation's measured events:
kernel launches, host round trips and device solve time.
"""
import ctypes as C
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_7128_b200 as P  # noqa: E402
from paper_1309_7128_b200.api import CycleConfig, GridSpec, RunMetrics, ScalarField, Scheme  # noqa: E402

_XS = r"""
#include <stdint.h>
void xorshift_fill(double* out, long n) {
    uint64_t s = 0x243F6A8885A308D3ull;
    for (long k = 0; k < n; ++k) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        out[k] = (double)(s >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    }
}
"""


def xorshift_noise(count):
    d = tempfile.mkdtemp()
    src, lib = os.path.join(d, "xs.c"), os.path.join(d, "xs.so")
    open(src, "w").write(_XS)
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", lib, src])
    f = C.CDLL(lib).xorshift_fill
    out = np.empty(count)
    f(out.ctypes.data_as(C.POINTER(C.c_double)), C.c_long(count))
    return out


def a3_rhs(n):
    b = ScalarField(n, n)
    bi = b.interior()
    bi[:] = xorshift_noise(n * n).reshape(n, n)
    xs = (np.arange(n) + 0.5) / n
    for kx in range(5):
        cx = np.cos(math.pi * kx * xs)
        for ky in range(5):
            cy = np.cos(math.pi * ky * xs)
            a = float(cy @ bi @ cx) / (float(cx @ cx) * float(cy @ cy))
            bi -= a * np.outer(cy, cx)
    bi -= bi.mean()
    bi *= 1e-4
    return b


def run(scheme, n, b, **kw):
    g = GridSpec(nx=n, ny=n, tile=32)
    cfg = CycleConfig(scheme=scheme, tile=32, tol_fine=1e-6, tol_coarse=1e-5, max_total_sweeps=20000, **kw)
    solver = P.PressureSolver(g, cfg)
    x = P.DeviceField(n, n)
    bd = P.DeviceField.from_host(b)
    m = RunMetrics(n * n)
    t0 = time.perf_counter()
    rep = solver.solve(x, bd, m)
    wall = time.perf_counter() - t0
    s = solver.last_stats()
    c = m.current
    return {"scheme": scheme.name, "converged": bool(rep.converged), "residual": rep.residual,
            "I_f": c.fine_sweeps, "I_c": c.coarse_sweeps, "NCC_f": c.sync_fine, "NCC_c": c.sync_coarse,
            "NCC_t": c.sync_fine + c.sync_coarse, "N_Lap": c.lap_equiv, "restrictions": c.restrictions,
            "prolongations": c.prolongations, "kernel_launches": s["kernel_launches"],
            "host_syncs": s["host_syncs"], "solve_ms": s["solve_ms"], "wall_s": wall}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    out = sys.argv[2] if len(sys.argv) > 2 else None
    b = a3_rhs(n)
    res = {"n": n, "rhs": "A3 recipe (acceptance.cpp:162-207) scaled to n", "tol_fine": 1e-6,
           "ism": run(Scheme.ismg, n, b), "acm": run(Scheme.acm, n, b, depth=6)}
    line = json.dumps(res)
    print(line)
    if out:
        open(out, "w").write(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
