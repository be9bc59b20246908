#!/bin/bash
# ncu evidence for the cfg3 bench (100M x 96): launch list of the bench
# command, one-pass DRAM/time metrics of every K1 launch at the full 1M-query
# batch, and a --set full capture of one K1 launch at a 100k-query batch.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg3_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-modes > gpurun_out/cfg3_launches.out 2>&1
ncu -k regex:search_kernel -c 2 --clock-control none --csv --log-file gpurun_out/cfg3_k1_dram.csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-modes > gpurun_out/cfg3_k1_dram.out 2>&1
timeout 1500 ncu -k regex:search_kernel -s 1 -c 1 --set full --clock-control none --import-source on \
  -o gpurun_out/cfg3_k1_full -f \
  python bench.py --steps 1 --warmup 1 --nq 100000 --no-cpu-baseline --no-e2e --no-modes > gpurun_out/cfg3_k1_full.out 2>&1
echo done
