#!/usr/bin/env bash
# Build the CPU oracle (TEST INFRASTRUCTURE).
#  1. oracle/libismg_oracle.so  — the plain-C restatement (always).
#  2. oracle/_ref/libismg_ref.so — the UNMODIFIED reference, compiled from its
#     own headers where they lie (REF defaults to /root/reference), only when
#     the reference tree is present. Reference flags: -O3, no -march
#     (proj/CMakeLists.txt:14), i.e. no FMA contraction.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${REF:-/root/reference}"

gcc -std=c11 -O3 -ffp-contract=off -fPIC -shared -Wall -Wextra -Wno-unused-parameter \
    -o "$HERE/libismg_oracle.so" "$HERE/ismg_oracle.c" -lm

if [ -d "$REF/proj/include/ismg" ]; then
    mkdir -p "$HERE/_ref"
    g++ -std=c++20 -O3 -fPIC -shared \
        -I "$REF/proj/include" \
        -o "$HERE/_ref/libismg_ref.so" "$HERE/ref_shim.cpp"
    echo "built oracle/_ref/libismg_ref.so from $REF"
else
    echo "reference tree absent ($REF): oracle/_ref not rebuilt"
fi
