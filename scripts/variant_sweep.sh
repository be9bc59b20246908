#!/bin/bash
# Build-variant sweep of K1 on the GPU box: each line of $VARIANTS is a set of
# -D flags; prints QPS / K1 ms / roofline fraction per variant.
set -u
VARIANTS=${VARIANTS:-"-DDVSG_MINB=5"}
while IFS= read -r V; do
  [ -z "$V" ] && continue
  make -s -B -C paper_2512_02278_b200/csrc -j8 EXTRA="$V" > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  out=$(timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --recall-sample 200 2>/dev/null | tail -1)
  echo "[$V] $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("qps=%.0f k1_ms=%.2f frac=%.3f" % (d["value"], r["k1_ms_per_step"], r["frac"]))' 2>&1)"
done <<< "$VARIANTS"
