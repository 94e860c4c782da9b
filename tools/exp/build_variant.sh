#!/bin/bash
# A/B build of libf3d with extra -D flags on one source (default attn_tc.cu):
#   [SRC=gemm_tc.cu] tools/exp/build_variant.sh <name> -DMACRO=...  -> tools/exp/libf3d_<name>.so
# (select with F3D_LIB_PATH=tools/exp/libf3d_<name>.so; the in-tree build is untouched)
set -e
cd "$(dirname "$0")/../../paper_2412_16481_b200/csrc"
make -s >/dev/null
SRC=${SRC:-attn_tc.cu}
base=${SRC%.cu}
name=$1; shift
tmp=$(mktemp -d)
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -c $SRC -o "$tmp/$base.o"
objs=$(ls build/*.o | grep -v "/$base.o\$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/exp/libf3d_$name.so \
    "$tmp/$base.o" $objs -lcuda
rm -rf "$tmp"
echo tools/exp/libf3d_$name.so
