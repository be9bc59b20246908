"""Synthetic workloads for bench.py -- setup only, never timed.

  sift_like   integer-valued low-rank data in [0, 255]: x = A z + 0.1 eps,
              z ~ N(0, I_r), A ~ N(0, 1/r), scaled by 40 around 128 and
              rounded (SIFT vectors are bytes).  Integer data keeps every
              fp32 squared-L2 sum exact (< 2^24 at d=128), so the GPU graph
              builder and the fp32 search mode are bit-identical to the
              reference's fp64 arithmetic on it.
  kmeans      Lloyd on a subsample (numpy) -- centroids only feed routing;
              kmeans_train itself is out of scope.
  build_index partition_database via K5 (assign top-1, exact) and one exact
              kNN graph per cluster via K6; returns an api.BuiltIndex.
"""
from __future__ import annotations

import numpy as np

from .api import BuiltIndex, Context, GraphIndex, compute_entry_order


def sift_like(n: int, dim: int = 128, rank: int = 16, seed: int = 1, scale: float = 40.0,
              chunk: int = 1 << 18) -> np.ndarray:
    rng = np.random.default_rng(seed)
    a = rng.normal(0.0, 1.0 / np.sqrt(rank), size=(rank, dim)).astype(np.float32)
    out = np.empty((n, dim), np.float32)
    for b in range(0, n, chunk):
        e = min(n, b + chunk)
        z = rng.standard_normal(size=(e - b, rank), dtype=np.float32)
        x = z @ a + 0.1 * rng.standard_normal(size=(e - b, dim), dtype=np.float32)
        out[b:e] = np.clip(np.rint(x * scale + 128.0), 0, 255)
    return out


def sift_like_queries(n: int, dim: int = 128, rank: int = 16, data_seed: int = 1,
                      seed: int = 2, scale: float = 40.0) -> np.ndarray:
    """Fresh points from the same subspace A as sift_like(..., seed=data_seed)."""
    rng = np.random.default_rng(data_seed)
    a = rng.normal(0.0, 1.0 / np.sqrt(rank), size=(rank, dim)).astype(np.float32)
    rq = np.random.default_rng(seed)
    z = rq.standard_normal(size=(n, rank), dtype=np.float32)
    x = z @ a + 0.1 * rq.standard_normal(size=(n, dim), dtype=np.float32)
    return np.clip(np.rint(x * scale + 128.0), 0, 255).astype(np.float32)


def kmeans(data: np.ndarray, clusters: int, iters: int = 10, seed: int = 42,
           sample: int = 100_000) -> np.ndarray:
    rng = np.random.default_rng(seed)
    idx = rng.choice(data.shape[0], size=min(sample, data.shape[0]), replace=False)
    x = data[np.sort(idx)].astype(np.float64)
    c = x[rng.choice(x.shape[0], size=clusters, replace=False)].copy()
    for _ in range(iters):
        d = (x * x).sum(1)[:, None] + (c * c).sum(1)[None, :] - 2.0 * x @ c.T
        lab = d.argmin(1)
        for j in range(clusters):
            m = lab == j
            if m.any():
                c[j] = x[m].mean(0)
    return c.astype(np.float32)


def build_index(ctx: Context, data: np.ndarray, clusters: int, out_degree: int = 32,
                ranks: int = 1, seed: int = 42) -> BuiltIndex:
    """BuiltIndex like build_index (index.cpp:43-72) with GPU partition + graphs."""
    if clusters == 1:
        cents = data.mean(0, dtype=np.float64).astype(np.float32)[None, :]
        labels = np.zeros(data.shape[0], np.uint32)
    else:
        cents = kmeans(data, clusters, seed=seed)
        ctx.reset()
        ctx.set_centroids(cents, None, 1)
        labels = np.concatenate([ctx.assign_top_c(data[b:b + (1 << 20)], 1)[:, 0]
                                 for b in range(0, data.shape[0], 1 << 20)])
    graphs = []
    for c in range(clusters):
        ids = np.nonzero(labels == c)[0].astype(np.uint32)
        part = np.ascontiguousarray(data[ids])
        adj = ctx.build_graph(part, out_degree)
        graphs.append(GraphIndex(part, ids, out_degree, adj, compute_entry_order(part)))
    placement = (np.arange(clusters) % ranks).astype(np.uint32)
    return BuiltIndex(cents, placement, ranks, out_degree, graphs)


def brute_force_gt(data: np.ndarray, queries: np.ndarray, k: int, device: str = "cuda:0",
                   ctx=None):
    """Exact top-k ids for recall@k (topk.cpp:12-30, ties by lower id): the
    library's GPU brute force (dvsg_brute_force_topk) when k <= 32."""
    if k <= 32:
        from .api import Context
        cx = ctx or Context(int(device.split(":")[1]) if ":" in device else 0)
        return cx.brute_force_topk(data, queries, k)[0]
    import torch
    x = torch.from_numpy(data).to(device)
    xn = (x.double() ** 2).sum(1).float()
    out = []
    for b in range(0, queries.shape[0], 256):
        q = torch.from_numpy(queries[b:b + 256]).to(device)
        d = (q.double() ** 2).sum(1, keepdim=True).float() + xn[None, :] - 2.0 * (q @ x.T)
        # (dist, id) order: exact ints, so scale dist and add id as a tiebreak
        key = d.double().round() * float(1 << 24) + torch.arange(x.shape[0], device=device).double()
        out.append(torch.topk(key, k, dim=1, largest=False).indices.cpu().numpy())
    return np.concatenate(out).astype(np.uint32)


def recall_at_k(ids: np.ndarray, counts: np.ndarray, truth: np.ndarray, k: int) -> float:
    """recall_at_k, topk.cpp:32-49, averaged over queries."""
    tot = 0.0
    for q in range(truth.shape[0]):
        tot += len(set(ids[q, :int(counts[q])].tolist()) & set(truth[q, :k].tolist())) / k
    return tot / truth.shape[0]
