#!/bin/bash
# Build-variant sweep of the bulk exchange kernels (emulated ranks on one GPU):
# each line of $VARIANTS is a set of -D flags; prints the emulated search ms.
set -u
VARIANTS=${VARIANTS:-"-DDVSG_XG_EXPAND_MINB=4"}
while IFS= read -r V; do
  [ -z "$V" ] && continue
  make -s -B -C paper_2512_02278_b200/csrc -j8 EXTRA="$V" > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  echo "[$V] $(DVSG_XG_LANES=${LANES:-1} EXCHANGES=bulk RANKS=${RANKS:-1} timeout 300 python scripts/shard_emu_bench.py 2>&1 | grep emulated | tr '\n' ' ')"
done <<< "$VARIANTS"
make -s -B -C paper_2512_02278_b200/csrc -j8 > /dev/null 2>&1
