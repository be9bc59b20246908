#!/usr/bin/env python
"""Prototype: does a CAGRA-style optimisation from an intermediate kNN-64
graph (instead of kNN-32) buy fewer visited vectors at recall 0.95?  Exact
kNN at n=2M (torch matmul, integer data -> exact fp32), both graphs pruned to
degree 32 with the same rule (rank-based detours over the intermediate
graph, keep forward, reverse by forward rank), recall / visited sweep."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_02278_b200 as dvs  # noqa: E402
from paper_2512_02278_b200 import ivf  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False


def knn(x, k):
    n = x.shape[0]
    xn = (x * x).sum(1)
    out = torch.empty((n, k), dtype=torch.int64, device=x.device)
    for b in range(0, n, 512):
        e = min(n, b + 512)
        d = xn[b:e, None] + xn[None, :] - 2.0 * (x[b:e] @ x.T)
        d[torch.arange(e - b), torch.arange(b, e)] = float("inf")
        key = (d.round().to(torch.int64) << 32) | torch.arange(n, device=x.device)[None, :]
        out[b:e] = torch.topk(key, k, dim=1, largest=False).values & 0xFFFFFFFF
    return out


def optimize(adj, keep, dout):
    """rank-based detour pruning on adj (n, din) -> (n, dout)."""
    n, d = adj.shape
    dev = adj.device
    det = torch.empty((n, d), dtype=torch.int32, device=dev)
    ar = torch.arange(d, device=dev)
    lower = ar[:, None] < ar[None, :]
    for b in range(0, n, 1 << 12):
        e = min(n, b + (1 << 12))
        a = adj[b:e]
        nn = adj[a]
        eq = nn[:, :, :, None] == a[:, None, None, :]
        rank = torch.where(eq.any(2), eq.to(torch.int8).argmax(2), d)
        det[b:e] = (lower[None] & (rank < ar[None, None, :])).sum(1).to(torch.int32)
    order = torch.sort(det.to(torch.int64) * d + ar[None, :], 1).indices
    fwd = torch.gather(adj, 1, order[:, :keep])
    nrev = dout - keep
    dst = fwd.reshape(-1)
    src = torch.arange(n, device=dev).repeat_interleave(keep)
    rk = order[:, :keep].reshape(-1)
    key = torch.sort((dst << 37) | (rk << 32) | src).values
    dsts = key >> 37
    cnt = torch.bincount(dsts, minlength=n)
    start = torch.cumsum(cnt, 0) - cnt
    idx = torch.arange(key.numel(), device=dev) - start[dsts]
    m = idx < nrev
    rev = torch.full((n, nrev), -1, dtype=torch.int64, device=dev)
    rev[dsts[m], idx[m]] = key[m] & 0xFFFFFFFF
    out = torch.empty((n, dout), dtype=torch.int64, device=dev)
    for b in range(0, n, 1 << 16):
        e = min(n, b + (1 << 16))
        cand = torch.cat([fwd[b:e], rev[b:e], torch.gather(adj[b:e], 1, order[b:e, keep:])], 1)
        srt, pos = torch.sort(cand, dim=1, stable=True)
        dup = torch.zeros_like(srt, dtype=torch.bool)
        dup[:, 1:] = srt[:, 1:] == srt[:, :-1]
        dup |= srt < 0
        bad = torch.zeros_like(dup)
        bad.scatter_(1, pos, dup)
        score = torch.where(bad, 10 ** 6, torch.arange(cand.shape[1], device=dev)[None, :].expand_as(cand))
        sel = torch.sort(score, 1).indices[:, :dout]
        out[b:e] = torch.gather(cand, 1, sel)
    return out


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    ctx = dvs.Context(0)
    x = ivf.sift_like_device(n, 96, 16, seed=1)
    q = ivf.sift_like_queries_device(2000, 96, 16, 1, 2)
    g64 = knn(x, 64)
    gt = ivf.brute_force_topk(ctx, x, ivf.row_norms(ctx, x), q, 10)[0].cpu().numpy()
    xh = x.cpu().numpy()
    res = {}
    for name, adj in [("knn32_opt12", optimize(g64[:, :32].contiguous(), 12, 32)),
                      ("knn64_opt16", optimize(g64, 16, 32)), ("knn64_opt12", optimize(g64, 12, 32)),
                      ("knn64_opt20", optimize(g64, 20, 32))]:
        a = adj.cpu().numpy().astype(np.uint32)
        ctx.reset()
        ctx.load_partition(0, dvs.GraphIndex(xh, np.arange(n, dtype=np.uint32), 32, a, None))
        out = {}
        for it, w in [(12, 16), (16, 16), (20, 16), (8, 32), (10, 32)]:
            ids, _, c, v = ctx.beam_search(0, q.cpu().numpy(), dvs.SearchParams(it, w, 10, w, accum="f32"))
            r = np.mean([len(set(ids[i, :c[i]].tolist()) & set(gt[i].tolist())) / 10 for i in range(2000)])
            out[f"{it}x{w}"] = (round(float(r), 4), round(float(v.mean())))
        res[name] = out
        print(name, out, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
