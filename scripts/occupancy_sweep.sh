#!/bin/bash
# K1 occupancy sweep on the GPU box: register budget (DVSG_MINB CTAs/SM) x
# visited-hash placement (shared vs global/L2).  Rebuilds libdvsg.so per point.
set -u
for MINB in ${MINBS:-2 3 4}; do
  make -s -B -C paper_2512_02278_b200/csrc -j8 EXTRA="-DDVSG_MINB=$MINB" > /dev/null 2>&1 || { echo "build MINB=$MINB failed"; continue; }
  for HS in ${HASHES:-16384 0}; do
    out=$(DVSG_HASH_SMEM_MAX=$HS timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --recall-sample 200 2>/dev/null | tail -1)
    echo "MINB=$MINB hash_smem_max=$HS $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("qps=%.0f k1_ms=%.2f frac=%.3f" % (d["value"], r["k1_ms_per_step"], r["frac"]))' 2>&1)"
  done
done
