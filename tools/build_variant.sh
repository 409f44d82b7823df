#!/bin/bash
# build_variant.sh NAME [NVCC FLAGS...]: a copy of the library with one source
# (SRC, default fine_pass_w.cu) compiled under extra flags, written to
# exp/var_NAME/libismg_b200.so; load it with ISMG_LIB=exp/var_NAME/libismg_b200.so.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
src=${SRC:-fine_pass_w.cu}
out=exp/var_$name; mkdir -p $out
objs=$(SRC_NAME=$src python -c "import os; from paper_1309_7128_b200.build import SOURCES; print(' '.join('build/obj/%s.o' % s for s in SOURCES if s != os.environ['SRC_NAME']))")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC,-O3,-fvisibility=hidden \
  -I include --expt-relaxed-constexpr "$@" -c paper_1309_7128_b200/csrc/$src -o $out/${src%.cu}.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libismg_b200.so $objs $out/${src%.cu}.o -lnccl -L/usr/lib/x86_64-linux-gnu
echo $out/libismg_b200.so
