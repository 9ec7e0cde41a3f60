#!/bin/bash
# Build an A/B variant of libchase.so with extra nvcc flags (e.g. kernel
# shape macros) into build/variants/libchase_<name>.so; select it at run time
# with CHASE_LIB_OVERRIDE=<path> (tuning only; the product is libchase.so).
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=${CSRC:-$ROOT/paper_2303_02508_b200/csrc}
O=$ROOT/build/variants/$name
mkdir -p "$O"
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -fmad=false -Xptxas -v -Xcompiler -fPIC -I ${CINC:-$ROOT/include} -I $C "$@" \
    -c $C/kernels.cu -o $O/kernels.o 2>&1 | grep -A3 "entry function.*sweep_fast" | grep -E "spill|Used" || true
nvcc $ARCH -O2 -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -I ${CINC:-$ROOT/include} -I $C "$@" -c $C/chase_api.cpp -o $O/api.o
nvcc $ARCH -O2 -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -I ${CINC:-$ROOT/include} -I $C -c $C/envelope.cpp -o $O/env.o
nvcc $ARCH -shared -cudart static -o $ROOT/build/variants/libchase_$name.so $O/kernels.o $O/api.o $O/env.o -ldl
rm -rf "$O"
echo built $ROOT/build/variants/libchase_$name.so
