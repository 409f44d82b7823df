#!/bin/bash
# build_variant.sh NAME [NVCC FLAGS...]: a copy of the library with some sources
# (SRC, space-separated, default fine_pass_w.cu) compiled under extra flags,
# written to exp/var_NAME/libismg_b200.so; load it with
# ISMG_LIB=exp/var_NAME/libismg_b200.so.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
srcs=${SRC:-fine_pass_w.cu}
out=exp/var_$name; mkdir -p $out
objs=$(SRC_NAMES="$srcs" python -c "import os; from paper_1309_7128_b200.build import SOURCES; ex = os.environ['SRC_NAMES'].split(); print(' '.join('build/obj/%s.o' % s for s in SOURCES if s not in ex))")
vobjs=""
for src in $srcs; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC,-O3,-fvisibility=hidden \
    -I include --expt-relaxed-constexpr "$@" -c paper_1309_7128_b200/csrc/$src -o $out/${src%.*}.o
  vobjs="$vobjs $out/${src%.*}.o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libismg_b200.so $objs $vobjs -lnccl -L/usr/lib/x86_64-linux-gnu
echo $out/libismg_b200.so
