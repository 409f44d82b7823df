"""Build the sm_100a library in-tree: paper_1309_7128_b200/libismg_b200.so.

    python -m paper_1309_7128_b200.build [--force] [--verbose]

Every translation unit is compiled by nvcc for `-gencode arch=compute_100a,
code=sm_100a` with `-fmad=false` (no multiply-add contraction: the kernels
keep the reference's rounding sequence) and `-lineinfo` (ncu source view).
Objects go to build/, the shared library next to this file so that it travels
with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libismg_b200.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden",
          "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]
SOURCES = ["objects.cu", "geometry.cpp", "ops.cu", "fine_pass.cu", "fine_pass_w.cu", "coarse.cu", "coarse_tmem.cu", "coarse_cl.cu", "coarse_rw.cu", "coarse_sp.cu", "coarse_sp2.cu", "fused_host.cu",
           "solver.cu", "comm.cpp", "capi.cpp"]
HEADERS = ["common.h", "engine.h", "kernels.cuh", "solver.h", "fused_impl.cuh"]


def _needs(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "ismg_b200.h")]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    extra = ["-Xptxas", "-v"] if (verbose and src.endswith(".cu")) else []
    cmd = [NVCC] + ARCH + COMMON + extra + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
    return r.stderr if verbose else ""


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    todo = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s)) and
            (force or _needs(os.path.join(OBJ, s + ".o"), os.path.join(CSRC, s)))]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            for src, log in zip(todo, ex.map(lambda s: _compile(s, verbose), todo)):
                if log:
                    sys.stderr.write("== %s\n%s" % (src, log))
    objs = [os.path.join(OBJ, s + ".o") for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if todo or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lnccl", "-L/usr/lib/x86_64-linux-gnu"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
