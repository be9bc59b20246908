"""K1 vs node-sharded search (bench workload, default cfg3; `--nq` to shrink) (bulk and fused exchange) with R ranks emulated on one GPU (protocol overhead
without NVLink): K1 event time for the bench workload, plus parity."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_02278_b200 as dvs  # noqa: E402

import torch  # noqa: E402

args = bench.parse(sys.argv[1:])
ctx = dvs.Context(0)
w = bench.build_workload(args, 0, ctx, torch.device("cuda", 0))
queries = w.queries[:, :args.dim].cpu().numpy()
ctx.set_timing(True)
p = dvs.SearchParams(args.iterations, args.beam, args.k, args.entry, metric=args.metric, accum=args.accum)
ref = None
for _ in range(2):
    ref = ctx.beam_search(0, queries, p)
print("unsharded K1 ms", round(ctx.last_timings()["search_ms"], 2), flush=True)
modes = os.environ.get("EXCHANGES", "bulk,fused").split(",")
for mode in modes:
    ctx.set_shard_exchange(mode)
    for R in [int(r) for r in os.environ.get("RANKS", "1,2,4,8").split(",")]:
        for _ in range(2):
            got = ctx.beam_search_sharded_emulated(R, queries, p)
        same = all(np.array_equal(a, b) for a, b in zip(got, ref))
        print(f"{mode} emulated R={R} ms", round(ctx.last_timings()["search_ms"], 2), "identical", same, flush=True)
