#!/bin/bash
# Build a variant of libdvsg.so: one kernel source (SRC, default search_kernel)
# recompiled with extra -D flags, linked with the other objects of the current build.
#   [SRC=xchg_kernel] scripts/build_variant.sh NAME "-DFLAG=V ..."  ->  paper_2512_02278_b200/variants/libdvsg_NAME.so
set -e
NAME=$1; FLAGS=$2; SRC=${SRC:-search_kernel}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/build/obj
OUT=$ROOT/paper_2512_02278_b200/variants
TMP=$ROOT/build/var_$NAME
mkdir -p "$OUT" "$TMP"
ARCH="-gencode arch=compute_100a,code=sm_100a"
/usr/local/cuda/bin/nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $FLAGS \
  -c "$ROOT/paper_2512_02278_b200/csrc/$SRC.cu" -o "$TMP/$SRC.o" 2> "$TMP/ptxas.log"
OBJS=$(ls $OBJ/*.o | grep -v "/$SRC.o")
/usr/local/cuda/bin/nvcc $ARCH -shared -o "$OUT/libdvsg_$NAME.so" "$TMP/$SRC.o" $OBJS -Xcompiler -pthread
grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" "$TMP/ptxas.log" | sort | uniq -c | head -6
