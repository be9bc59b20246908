#!/bin/bash
# Build a K1 variant of libdvsg.so: search_kernel.cu recompiled with extra -D
# flags, linked with the other objects of the current build.
#   scripts/build_variant.sh NAME "-DFLAG=V ..."  ->  paper_2512_02278_b200/variants/libdvsg_NAME.so
set -e
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/build/obj
OUT=$ROOT/paper_2512_02278_b200/variants
TMP=$ROOT/build/var_$NAME
mkdir -p "$OUT" "$TMP"
ARCH="-gencode arch=compute_100a,code=sm_100a"
/usr/local/cuda/bin/nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $FLAGS \
  -c "$ROOT/paper_2512_02278_b200/csrc/search_kernel.cu" -o "$TMP/search_kernel.o" 2> "$TMP/ptxas.log"
OBJS=$(ls $OBJ/*.o | grep -v search_kernel.o)
/usr/local/cuda/bin/nvcc $ARCH -shared -o "$OUT/libdvsg_$NAME.so" "$TMP/search_kernel.o" $OBJS -Xcompiler -pthread
grep -A1 "search_kernel" "$TMP/ptxas.log" | grep -o "Used [0-9]* registers.*" | sort | uniq -c | head -3
