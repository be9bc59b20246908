#!/usr/bin/env python
"""Diagnostics of the cluster-restricted graph: adjacency overlap with the
exact kNN graph (K6) and search recall on each, at a size K6 can build."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_02278_b200 as dvs  # noqa: E402
from paper_2512_02278_b200 import ivf, synth  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def recall(ctx, x, adj, q, gt, it, w):
    ctx.reset()
    ctx.load_partition(0, dvs.GraphIndex(x, np.arange(x.shape[0], dtype=np.uint32), adj.shape[1], adj, None))
    ids, d, c, v = ctx.beam_search(0, q, dvs.SearchParams(it, w, 10, w))
    r = np.mean([len(set(ids[i, :c[i]].tolist()) & set(gt[i].tolist())) / 10 for i in range(len(q))])
    return float(r), float(v.mean())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=96)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--probe", type=int, default=8)
    ap.add_argument("--cluster-size", type=int, default=1536)
    args = ap.parse_args()
    ctx = dvs.Context(0)
    xt = ivf.sift_like_device(args.n, args.dim, args.rank, seed=1)
    info = ivf.build_graph_ivf(ctx, xt, probe=args.probe, cluster_size=args.cluster_size, dim=args.dim, log=log)
    pv, pa, _, _, n = ctx.partition_view_device(0)
    x = ivf.device_view(pv, (n, args.dim), torch.float32, "cuda").cpu().numpy()
    a1 = ivf.device_view(pa, (n, 32), torch.int32, "cuda").cpu().numpy().view(np.uint32).copy()
    q = ivf.sift_like_queries_device(2000, args.dim, args.rank, 1, 2).cpu().numpy()
    t0 = time.time()
    a0 = ctx.build_graph(x, 32)
    log(f"exact K6 graph {time.time() - t0:.1f}s")
    ov = np.mean([len(set(a0[i].tolist()) & set(a1[i].tolist())) / 32 for i in range(0, n, max(1, n // 20000))])
    gt = synth.brute_force_gt(x, q, 10, ctx=ctx)
    # GT of the numpy-generated SIFT-like data (last round's generator) for comparison
    out = {"n": n, "dim": args.dim, "adjacency_overlap": ov}
    for it, w in [(6, 64), (10, 64), (10, 128)]:
        out[f"exact_{it}x{w}"] = recall(ctx, x, a0, q, gt, it, w)
        out[f"ivf_{it}x{w}"] = recall(ctx, x, a1, q, gt, it, w)
    xs = synth.sift_like(n, args.dim, args.rank, seed=1)
    qs = synth.sift_like_queries(2000, args.dim, args.rank, 1, 2)
    a2 = ctx.build_graph(xs, 32)
    gt2 = synth.brute_force_gt(xs, qs, 10, ctx=ctx)
    out["numpy_gen_exact_6x64"] = recall(ctx, xs, a2, qs, gt2, 6, 64)
    out["x_stats"] = [float(x.mean()), float(x.std()), float(xs.mean()), float(xs.std())]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
