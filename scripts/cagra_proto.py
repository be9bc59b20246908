#!/usr/bin/env python
"""Prototype (torch) of a CAGRA-style graph optimisation on top of a kNN-32
graph: rank-based detour pruning to `keep` forward edges + reverse edges,
then recall of the reference's beam search on each graph."""
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


def optimize(adj, keep):
    """adj: (n, d) int64 cuda, rows sorted by distance.  -> (n, d) int64."""
    n, d = adj.shape
    dev = adj.device
    det = torch.empty((n, d), dtype=torch.int32, device=dev)
    ar = torch.arange(d, device=dev)
    for b in range(0, n, 1 << 15):
        e = min(n, b + (1 << 15))
        a = adj[b:e]                       # (m, d): u_j
        nn = adj[a]                        # (m, d i, d r): N(u_i)
        # rank of u_j in N(u_i) (d if absent)
        eq = nn[:, :, :, None] == a[:, None, None, :]          # (m, i, r, j)
        hit = eq.any(2)
        rank = torch.where(hit, eq.int().argmax(2), torch.full_like(hit, d, dtype=torch.int64))  # (m, i, j)
        # u_i detours u_j: i < j and rank_{u_i}(u_j) < j
        cond = (ar[:, None] < ar[None, :]) & (rank < ar[None, None, :])
        det[b:e] = cond.sum(1).int()
    key = det.long() * d + ar[None, :]
    order = torch.sort(key, 1).indices
    fwd = torch.gather(adj, 1, order[:, :keep])            # pruned forward, by (detours, rank)
    # reverse edges: u gets v for every kept v -> u, preferring small rank
    src = torch.arange(n, device=dev)[:, None].expand(n, keep).reshape(-1)
    dst = fwd.reshape(-1)
    rk = torch.gather(order, 1, torch.arange(keep, device=dev)[None, :].expand(n, keep)).reshape(-1)
    k2 = (dst << 37) | (rk << 32) | src
    k2 = torch.sort(k2).values
    dsts = k2 >> 37
    cnt = torch.bincount(dsts, minlength=n)
    start = torch.cumsum(cnt, 0) - cnt
    idx = torch.arange(k2.numel(), device=dev) - start[dsts]
    rev = torch.full((n, d - keep), -1, dtype=torch.int64, device=dev)
    m = idx < (d - keep)
    rev[dsts[m], idx[m]] = k2[m] & 0xFFFFFFFF
    out = torch.empty((n, d), dtype=torch.int64, device=dev)
    # final: forward kept, then reverse (dedup), then the rest of the forward list by rank
    for b in range(0, n, 1 << 18):
        e = min(n, b + (1 << 18))
        cand = torch.cat([fwd[b:e], rev[b:e], torch.gather(adj[b:e], 1, order[b:e, keep:])], 1)
        # dedup keeping first occurrence, drop -1
        srt, pos = torch.sort(cand, dim=1, stable=True)
        dup = torch.zeros_like(srt, dtype=torch.bool)
        dup[:, 1:] = srt[:, 1:] == srt[:, :-1]
        dup |= srt < 0
        bad = torch.zeros_like(dup)
        bad.scatter_(1, pos, dup)
        score = torch.where(bad, torch.full_like(cand, 10 ** 6), torch.arange(cand.shape[1], device=dev)[None, :].expand_as(cand))
        sel = torch.sort(score, 1).indices[:, :d]
        out[b:e] = torch.gather(cand, 1, sel)
    return out


def recall(ctx, vec, adj, q, gt, sweeps):
    n = vec.shape[0]
    x = vec.cpu().numpy()
    a = adj.cpu().numpy().astype(np.uint32)
    ctx.reset()
    ctx.load_partition(0, dvs.GraphIndex(x, np.arange(n, dtype=np.uint32), a.shape[1], a, None))
    out = {}
    for it, w in sweeps:
        ids, _, c, v = ctx.beam_search(0, q, dvs.SearchParams(it, w, 10, w))
        out[f"{it}x{w}"] = (round(float(np.mean([len(set(ids[i, :c[i]].tolist()) & set(gt[i].tolist())) / 10
                                                 for i in range(len(q))])), 4), float(v.mean()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=96)
    ap.add_argument("--probe", type=int, default=8)
    ap.add_argument("--keep", type=int, default=16)
    ap.add_argument("--exact", action="store_true")
    args = ap.parse_args()
    ctx = dvs.Context(0)
    xt = ivf.sift_like_device(args.n, args.dim, 16, seed=1)
    ivf.build_graph_ivf(ctx, xt, probe=args.probe, dim=args.dim, log=log)
    del xt
    pv, pa, _, _, n = ctx.partition_view_device(0)
    vec = ivf.device_view(pv, (n, args.dim), torch.float32, "cuda").clone()
    adj = ivf.device_view(pa, (n, 32), torch.int32, "cuda").long().clone()
    q = ivf.sift_like_queries_device(2000, args.dim, 16, 1, 2)
    gt = ivf.brute_force_topk(ctx, vec, ivf.row_norms(ctx, vec), q, 10)[0].cpu().numpy()
    qn = q.cpu().numpy()
    sweeps = [(6, 64), (10, 64), (8, 96)]
    res = {"n": n, "ivf": recall(ctx, vec, adj, qn, gt, sweeps)}
    res["ivf_cagra"] = recall(ctx, vec, optimize(adj, args.keep), qn, gt, sweeps)
    if args.exact:
        ex = torch.from_numpy(ctx.build_graph(vec.cpu().numpy(), 32).astype(np.int64)).cuda()
        res["exact"] = recall(ctx, vec, ex, qn, gt, sweeps)
        res["exact_cagra"] = recall(ctx, vec, optimize(ex, args.keep), qn, gt, sweeps)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
