#!/bin/bash
# ncu evidence for bench.py (run on the GPU box via gpurun; one GPU).
#   1. launch list of the bench command (gpu__time_duration per launch)
#   2. one --set full capture of K1 (dvsg::search_kernel) at the bench config
# Each ncu command runs only after the identical command exited 0 without ncu.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
NCU=/usr/local/cuda/bin/ncu
BENCH="python bench.py --steps 3 --warmup 3"
K1CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$BENCH > "$OUT/plain.log" 2>&1 && \
  $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
       --log-file "$OUT/launches.csv" $BENCH > "$OUT/ncu_launch.log" 2>&1
echo "launch-list rc=$?"
$K1CMD > "$OUT/plain_k1.log" 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 \
       -o "$OUT/k1_full" $K1CMD > "$OUT/ncu_full.log" 2>&1
echo "full rc=$?"
