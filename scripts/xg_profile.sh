set -u
OUT=gpurun_out/xg; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
export EXCHANGES=bulk RANKS=1 DVSG_XG_LANES=1
CMD="python scripts/shard_emu_bench.py"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:xg_score -s 3 -c 1 -o $OUT/score_full $CMD > $OUT/ncu_score.log 2>&1
echo "score rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:xg_expand -s 3 -c 1 -o $OUT/expand_full $CMD > $OUT/ncu_expand.log 2>&1
echo "expand rc=$?"
