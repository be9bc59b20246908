#!/bin/bash
for S in ${SERVERS:-0 74 148 296}; do echo "servers=$S"; DVSG_SHARD_SERVERS=$S timeout 400 python scripts/shard_emu_bench.py 2>&1 | grep -v "^\[bench\]"; done
