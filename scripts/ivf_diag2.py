#!/usr/bin/env python
"""Large-n diagnostics of the cluster-restricted graph: overlap of sampled
rows with their exact 32-NN (K7 brute force over all rows), recall vs I."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_02278_b200 as dvs  # noqa: E402
from paper_2512_02278_b200 import ivf  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=96)
    ap.add_argument("--probe", type=int, default=8)
    ap.add_argument("--cluster-size", type=int, default=1024)
    ap.add_argument("--coarse", type=int, default=32)
    ap.add_argument("--optimize", action="store_true")
    ap.add_argument("--shortlist", type=int, default=32)
    ap.add_argument("--sweep", default="6x64,12x64,24x64,48x64")
    args = ap.parse_args()
    ctx = dvs.Context(0)
    xt = ivf.sift_like_device(args.n, args.dim, 16, seed=1)
    info = ivf.build_graph_ivf(ctx, xt, probe=args.probe, cluster_size=args.cluster_size,
                               n_coarse=args.coarse, dim=args.dim, optimize=args.optimize,
                               shortlist=args.shortlist, log=log)
    del xt
    pv, pa, _, _, n = ctx.partition_view_device(0)
    vec = ivf.device_view(pv, (n, args.dim), torch.float32, "cuda")
    adj = ivf.device_view(pa, (n, 32), torch.int32, "cuda")
    vn = ivf.row_norms(ctx, vec)
    rows = torch.arange(0, n, n // 2000, device="cuda")[:2000]
    ex, _ = ivf.brute_force_topk(ctx, vec, vn, vec[rows].contiguous(), 32)
    ex = ex.cpu().numpy()
    a = adj[rows].cpu().numpy()
    r = rows.cpu().numpy()
    ov = np.mean([len(set(a[i].tolist()) & (set(ex[i].tolist()) - {r[i]})) / 31 for i in range(len(r))])
    # how far are the graph's neighbours vs the exact ones (mean dist ratio of the 32nd)
    q = ivf.sift_like_queries_device(2000, args.dim, 16, 1, 2)
    gt = ivf.brute_force_topk(ctx, vec, vn, q, 10)[0].cpu().numpy()
    out = {"n": n, "probe": args.probe, "cluster_size": args.cluster_size, "overlap": float(ov),
           "optimize": args.optimize, "coarse": args.coarse,
           "build_s": info["seconds"]["total"]}
    qn = q.cpu().numpy()
    for s in args.sweep.split(","):
        it, w = (int(v) for v in s.split("x"))
        ids, _, c, v = ctx.beam_search(0, qn, dvs.SearchParams(it, w, 10, w))
        out[s] = (round(float(np.mean([len(set(ids[i, :c[i]].tolist()) & set(gt[i].tolist())) / 10
                                       for i in range(len(qn))])), 4), float(v.mean()))
    # entry region vs query region: distance of queries to the mean row
    eo = ctx.entry_order(0)[:64]
    out["entry_rows"] = eo[:4].tolist()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
