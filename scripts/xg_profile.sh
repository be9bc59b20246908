#!/bin/bash
# ncu evidence for the bulk exchange (emulated ranks on one GPU): launch list
# of scripts/shard_emu_bench.py and one --set full capture of a mid-search
# xg_step launch.  LANES (default 2), RANKS (default 1), SKIP (default 6).
set -u
OUT=gpurun_out/xg; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
export EXCHANGES=bulk RANKS=${RANKS:-1} DVSG_XG_LANES=${LANES:-2}
CMD="python scripts/shard_emu_bench.py"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:xg_step -s ${SKIP:-6} -c 1 -o $OUT/step_full $CMD > $OUT/ncu_step.log 2>&1
echo "step rc=$?"
