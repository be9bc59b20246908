"""Recall / QPS calibration of the synthetic SIFT-like workload on one B200.

    python scripts/calibrate.py [--n 1000000] [--nq 2000]

Prints one JSON line per (clusters, fanout, iterations, beam) point:
recall@10 against exact brute force, K1 time, visited/query.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_02278_b200 as dvs  # noqa: E402
from paper_2512_02278_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--nq", type=int, default=2000)
    ap.add_argument("--clusters", type=str, default="1,8")
    ap.add_argument("--rank", type=int, default=16)
    args = ap.parse_args()
    t0 = time.time()
    data = synth.sift_like(args.n, 128, args.rank, seed=1)
    qs = synth.sift_like_queries(args.nq, 128, args.rank, data_seed=1, seed=2)
    print(json.dumps({"stage": "data", "s": round(time.time() - t0, 2)}), flush=True)
    truth = synth.brute_force_gt(data, qs, 10)
    print(json.dumps({"stage": "gt", "s": round(time.time() - t0, 2)}), flush=True)
    ctx = dvs.Context(0)
    ctx.set_timing(True)
    for C in [int(c) for c in args.clusters.split(",")]:
        t1 = time.time()
        idx = synth.build_index(ctx, data, C, 32)
        print(json.dumps({"stage": f"build C={C}", "s": round(time.time() - t1, 2),
                          "sizes": [g.size() for g in idx.graphs]}), flush=True)
        ctx.load_index(idx)
        for fo in sorted({1, 2, 3, min(4, C)} if C > 1 else {1}):
            if fo > C:
                continue
            for (I, w) in [(6, 64), (8, 64), (10, 64), (6, 96), (6, 128)]:
                for accum in ("f32", "f64"):
                    p = dvs.SearchParams(I, w, 10, w, accum=accum)
                    r = ctx.run_pipeline(qs, p, fo, 1, with_vectors=False)
                    t = ctx.last_timings()
                    rec = synth.recall_at_k(r.ids, r.counts, truth, 10)
                    print(json.dumps({"C": C, "fanout": fo, "I": I, "w": w, "accum": accum,
                                      "recall": round(rec, 4),
                                      "visited_per_q": r.visited_total / args.nq,
                                      "search_ms": round(t["search_ms"], 3),
                                      "total_ms": round(t["total_ms"], 3),
                                      "qps": round(args.nq / (t["total_ms"] / 1e3))}), flush=True)


if __name__ == "__main__":
    main()
