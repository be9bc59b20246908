"""Device-resident construction of 10M-100M-row indexes (setup, never timed).

The reference builds a partition's graph with an exact O(n^2) kNN
(`build_graph`, /root/reference/proj/src/graph_index.cpp:46-97): ~10^16
distance pairs at 100M rows.  Here the graph is a *cluster-restricted* kNN
graph built without leaving HBM, from the library's K7 range top-m kernel
(csrc/ivf_build.cu) and torch for the bookkeeping (sorts, block tables):

  1. two-level k-means on a strided sample: C1 coarse centroids, then
     C ~ n / cluster_size fine centroids split over the coarse cells in
     proportion to their sample counts (assignments: K7 with m = 1; means:
     dvsg_segment_means_device, in-order fp64 sums -> deterministic);
  2. every row -> nearest coarse centroid, then nearest fine centroid of that
     coarse cell (K7 over a row_map view, no gathered copy);
  3. rows stored in fine-cluster order (stable: ties by generation index) --
     the index's local ids are this order;
  4. each fine cluster's `probe` nearest fine centroids (K7 centroid x
     centroid);
  5. row v's adjacency = its `degree` nearest rows by (squared L2, id) among
     the members of its cluster's probe list, self excluded (K7, exact within
     that candidate set on integer-valued data), written straight into the
     context's adjacency array;
  6. commit: device validation + the exact device compute_entry_order
     (graph_index.cpp:21-44).

Every step is deterministic (no float atomics), so two processes that
generate the same data build bit-identical graphs -- the reference arm of
bench.py relies on that.  The graph is approximate w.r.t. the exact kNN graph
(rows whose true neighbours fall outside the probe list get the nearest
candidates inside it); search parity does not depend on that, because the GPU
and the reference search the same graph.
"""
from __future__ import annotations

import os
import time
from typing import Optional

import numpy as np

from . import _lib

TR = 128  # K7 rows per block


class _CAI:
    """Zero-copy torch view of a device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(int(s) for s in shape),
                                         "typestr": typestr, "version": 3, "strides": None}


def device_view(ptr: int, shape, dtype, device):
    import torch
    ts = {torch.float32: "<f4", torch.int32: "<i4", torch.int64: "<i8", torch.uint8: "|u1"}[dtype]
    return torch.as_tensor(_CAI(ptr, shape, ts), device=device)


def _sync():
    import torch
    torch.cuda.synchronize()


def segment_blocks(off, list_of_seg=None):
    """K7 block table over segments [off[s], off[s+1]) in blocks of <= 128
    rows; block b of segment s gets list id list_of_seg[s] (default s) and
    writes its rows at their own index.  -> int32 (nb, 4) tensor."""
    import torch
    off = off.to(torch.int64)
    sizes = off[1:] - off[:-1]
    nb = (sizes + TR - 1) // TR
    total = int(nb.sum())
    seg = torch.repeat_interleave(torch.arange(sizes.numel(), device=off.device), nb)
    first = torch.cumsum(nb, 0) - nb
    j = torch.arange(total, device=off.device) - first[seg]
    row0 = off[seg] + TR * j
    nrows = torch.minimum(torch.full_like(row0, TR), off[seg + 1] - row0)
    lst = seg if list_of_seg is None else list_of_seg.to(torch.int64)[seg]
    return torch.stack([row0, nrows, lst, row0], 1).to(torch.int32).contiguous(), total


def range_topk(ctx, rows, rnorm, cols, cnorm, blocks, list_off, ranges, m, flags=0, row_map=None,
               out_ids=None, out_dists=None, out_stride=None, out_rows=None, rows_bf16=None, cols_bf16=None):
    """K7 over torch tensors (all on the context's device).  With bf16 copies
    of rows and cols (to_bf16) it runs on the tensor cores (ivf_tc.cu)."""
    import torch
    dpad = rows.shape[1]
    stride = out_stride or m
    if out_ids is None:
        nout = out_rows if out_rows is not None else rows.shape[0] if row_map is None else row_map.numel()
        out_ids = torch.empty((nout, stride), dtype=torch.int32, device=rows.device)
    if os.environ.get("DVSG_IVF_CHECK", "0") == "1":
        _check_k7(rows, cols, blocks, list_off, ranges, m, flags, row_map, out_ids, stride)
    _sync()
    if rows_bf16 is not None and cols_bf16 is not None:
        ctx.range_topk_bf16_device(rows_bf16.data_ptr(), rnorm.data_ptr(), cols_bf16.data_ptr(), cnorm.data_ptr(),
                                   rows_bf16.shape[1], 0 if row_map is None else row_map.data_ptr(),
                                   blocks.data_ptr(), blocks.shape[0], list_off.data_ptr(), ranges.data_ptr(), m,
                                   flags, out_ids.data_ptr(), 0 if out_dists is None else out_dists.data_ptr(),
                                   stride)
    else:
        ctx.range_topk_device(rows.data_ptr(), rnorm.data_ptr(), cols.data_ptr(), cnorm.data_ptr(), dpad,
                              0 if row_map is None else row_map.data_ptr(), blocks.data_ptr(), blocks.shape[0],
                              list_off.data_ptr(), ranges.data_ptr(), m, flags, out_ids.data_ptr(),
                              0 if out_dists is None else out_dists.data_ptr(), stride)
    return out_ids


def to_bf16(ctx, x):
    """n x dpad float32 -> n x kpad bf16 (kpad = dpad rounded up to 16; as
    int16 storage), exact for integers in [-256, 256]."""
    import torch
    n, dpad = x.shape
    kpad = (dpad + 15) // 16 * 16
    out = torch.empty((n, kpad), dtype=torch.int16, device=x.device)
    _sync()
    ctx.to_bf16_device(x.data_ptr(), n, dpad, kpad, out.data_ptr())
    return out


def _check_k7(rows, cols, blocks, list_off, ranges, m, flags, row_map, out_ids, stride):
    """Host-side bounds checks of a K7 launch (DVSG_IVF_CHECK=1)."""
    b = blocks.long()
    nlog = rows.shape[0] if row_map is None else row_map.numel()
    assert int(b[:, 1].max()) <= TR and int(b[:, 1].min()) >= 0
    assert int((b[:, 0] + b[:, 1]).max()) <= nlog, "block rows past the row view"
    assert int(b[:, 2].max()) < list_off.numel() - 1, "list id past list_off"
    lo = list_off.long()
    assert bool((lo[1:] >= lo[:-1]).all()) and int(lo[-1]) <= ranges.shape[0], "list_off past ranges"
    r = ranges.long()
    assert bool((r[:, 0] <= r[:, 1]).all()) and int(r[:, 1].max()) <= cols.shape[0], "range past cols"
    if row_map is not None:
        assert int(row_map.long().max()) < rows.shape[0], "row_map past rows"
    if flags & 8:
        assert int(row_map.long().max()) < out_ids.shape[0]
    else:
        assert int((b[:, 3] + b[:, 1]).max()) <= out_ids.shape[0], "output rows past out_ids"
    assert out_ids.shape[1] == stride and m <= stride


def row_norms(ctx, x):
    import torch
    out = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    _sync()
    ctx.row_norms_device(x.data_ptr(), x.shape[0], x.shape[1], out.data_ptr())
    return out


def _single_list(ncols, device):
    import torch
    return (torch.tensor([0, 1], dtype=torch.int32, device=device),
            torch.tensor([[0, ncols]], dtype=torch.int32, device=device))


def assign_nearest(ctx, x, xn, cents, row_map=None, off=None, cell_off=None):
    """Nearest centroid (m = 1) of every row of x (or of x[row_map]).  With
    off/cell_off: rows [off[j], off[j+1]) (of the row_map order) only see
    centroids [cell_off[j], cell_off[j+1])."""
    import torch
    cn = row_norms(ctx, cents)
    n = x.shape[0] if row_map is None else row_map.numel()
    if off is None:
        off = torch.tensor([0, n], dtype=torch.int64, device=x.device)
        lo, rg = _single_list(cents.shape[0], x.device)
        blocks, _ = segment_blocks(off, torch.zeros(1, dtype=torch.int64, device=x.device))
    else:
        lo = torch.arange(off.numel(), dtype=torch.int32, device=x.device)
        rg = torch.stack([cell_off[:-1], cell_off[1:]], 1).to(torch.int32).contiguous()
        blocks, _ = segment_blocks(off)
    out = range_topk(ctx, x, xn, cents, cn, blocks, lo, rg, 1, row_map=row_map, out_rows=n)
    return out[:, 0].to(torch.int64)


def _sorted_segments(labels, nseg):
    import torch
    order = torch.sort(labels, stable=True).indices
    counts = torch.bincount(labels, minlength=nseg)
    off = torch.zeros(nseg + 1, dtype=torch.int64, device=labels.device)
    off[1:] = torch.cumsum(counts, 0)
    return order, off


def _means(ctx, x, order, off, cents):
    o32 = order.to(_torch().int32).contiguous()
    offc = off.contiguous()
    _sync()
    ctx.segment_means_device(x.data_ptr(), x.shape[1], o32.data_ptr(), offc.data_ptr(), offc.numel() - 1,
                             cents.data_ptr())


def _torch():
    import torch
    return torch


def kmeans2(ctx, x, xn, n_fine: int, n_coarse: int = 256, sample: int = 4 << 20, iters: int = 6,
            log=None):
    """Two-level k-means on a strided sample -> (coarse (C1 x dpad), fine
    (C x dpad), fine offset per coarse cell (C1 + 1))."""
    torch = _torch()
    n = x.shape[0]
    dev = x.device
    ns = min(n, sample)
    sidx = (torch.arange(ns, device=dev, dtype=torch.int64) * n) // ns
    s = x[sidx].contiguous()
    sn = xn[sidx].contiguous()
    c1 = min(n_coarse, ns)
    coarse = s[torch.linspace(0, ns - 1, c1, device=dev).round().long()].clone()
    for _ in range(iters):
        lab = assign_nearest(ctx, s, sn, coarse)
        order, off = _sorted_segments(lab, c1)
        _means(ctx, s, order, off, coarse)
    lab = assign_nearest(ctx, s, sn, coarse)
    order, off = _sorted_segments(lab, c1)
    cnt = (off[1:] - off[:-1]).double()
    per = torch.clamp(torch.round(cnt * n_fine / ns), min=1).long()
    foff = torch.zeros(c1 + 1, dtype=torch.int64, device=dev)
    foff[1:] = torch.cumsum(per, 0)
    nf = int(foff[-1])
    # init: evenly spaced members of each coarse cell (its coarse centroid if empty)
    cell = torch.repeat_interleave(torch.arange(c1, device=dev), per)
    j = torch.arange(nf, device=dev) - foff[cell]
    size = (off[cell + 1] - off[cell])
    pos = off[cell] + torch.where(size > 0, (j * size) // per[cell], torch.zeros_like(j))
    fine = torch.where((size > 0)[:, None], s[order[torch.clamp(pos, max=ns - 1)]], coarse[cell]).contiguous()
    s_sorted = s[order].contiguous()
    sn_sorted = sn[order].contiguous()
    for _ in range(iters):
        flab = assign_nearest(ctx, s_sorted, sn_sorted, fine, off=off, cell_off=foff)
        forder, ffoff = _sorted_segments(flab, nf)
        _means(ctx, s_sorted, forder, ffoff, fine)
    if log:
        log(f"[ivf] k-means: {c1} coarse x {nf} fine centroids from a {ns}-row sample")
    return coarse, fine, foff


def build_graph_ivf(ctx, x, degree: int = 32, cluster_size: int = 1024, probe: int = 8,
                    n_coarse: int = 32, sample: int = 4 << 20, iters: int = 6, cluster: int = 0,
                    dim: Optional[int] = None, shortlist: int = 32, optimize: bool = False,
                    keep: Optional[int] = None, tensor_cores: bool = False, log=None) -> dict:
    """Build one partition from the n x dpad float32 CUDA tensor `x` (rows in
    generation order) into `ctx`: rows stored in fine-cluster order, per-row
    probed kNN graph (K7 passes), optional CAGRA-style optimisation, device
    entry order.  `x`'s storage is released once the rows are stored.
    -> {"perm": generation index of each stored row (int64 tensor), ...}"""
    torch = _torch()
    t0 = time.time()
    n, dpad = x.shape
    dev = x.device
    dim = dim or dpad  # x holds dpad columns (zero pad)
    if (dim + 3) // 4 * 4 != dpad:
        raise ValueError(f"build_graph_ivf: x has {dpad} columns, dim {dim} pads to {(dim + 3) // 4 * 4}")
    xn = row_norms(ctx, x)
    n_fine = max(1, int(round(n / cluster_size)))
    coarse, fine, foff = kmeans2(ctx, x, xn, n_fine, n_coarse, sample, iters, log)
    nf = fine.shape[0]
    t1 = time.time()
    # every row: coarse cell, then the nearest fine centroid of that cell
    clab = assign_nearest(ctx, x, xn, coarse)
    corder, coff = _sorted_segments(clab, coarse.shape[0])
    corder32 = corder.to(torch.int32).contiguous()
    flab_sorted = assign_nearest(ctx, x, xn, fine, row_map=corder32, off=coff, cell_off=foff)
    del clab
    flab = torch.empty_like(flab_sorted)
    flab[corder] = flab_sorted
    del flab_sorted, corder32, corder
    perm, off = _sorted_segments(flab, nf)          # stable: ties by generation index
    del flab
    t2 = time.time()
    # the index rows, in cluster order, written straight into the context
    pv, pa, _, _ = ctx.partition_alloc_device(cluster, n, dim, degree)
    vec = device_view(pv, (n, dpad), torch.float32, dev)
    for b in range(0, n, 1 << 23):
        e = min(n, b + (1 << 23))
        vec[b:e] = x[perm[b:e]]
    del xn
    _sync()
    x.untyped_storage().resize_(0)                  # the generation-order copy is no longer needed
    torch.cuda.empty_cache()
    t3 = time.time()
    vn = row_norms(ctx, vec)
    fn = row_norms(ctx, fine)
    # per-row probe lists: the `probe` nearest fine centroids of each row, among
    # the `shortlist` nearest centroids of its own cluster's centroid
    q = min(shortlist, nf)
    p = min(probe, q)
    one = torch.zeros(1, dtype=torch.int64, device=dev)
    nbr = range_topk(ctx, fine, fn, fine, fn, segment_blocks(
        torch.tensor([0, nf], dtype=torch.int64, device=dev), one)[0],
        *_single_list(nf, dev), q).to(torch.int64)
    cb = fine[nbr.reshape(-1)].contiguous()
    cbn = fn[nbr.reshape(-1)].contiguous()
    blocks, nb = segment_blocks(off)
    lo = torch.arange(nf + 1, device=dev, dtype=torch.int32)       # list c = range c
    rg = torch.stack([torch.arange(nf, device=dev) * q, torch.arange(1, nf + 1, device=dev) * q], 1)
    rg = rg.to(torch.int32).contiguous()
    pidx = range_topk(ctx, vec, vn, cb, cbn, blocks, lo, rg, p)
    probes = nbr.reshape(-1)[pidx.to(torch.int64)]   # K7 returns columns of cb
    del cb, cbn, pidx
    # P passes: pass j groups the rows by their j-th probe cluster (row_map
    # view) and merges that cluster's members into the row's running top-32
    adj = device_view(pa, (n, degree), torch.int32, dev)
    dists = torch.empty((n, degree), dtype=torch.float32, device=dev)
    vb = to_bf16(ctx, vec) if tensor_cores and dpad <= 256 else None  # K7 on tcgen05 (ivf_tc.cu)
    lo1 = torch.arange(nf + 1, dtype=torch.int32, device=dev)
    rg1 = torch.stack([off[:-1], off[1:]], 1).to(torch.int32).contiguous()
    for j in range(p):
        lab = probes[:, j].contiguous()
        order, poff = _sorted_segments(lab, nf)
        order32 = order.to(torch.int32).contiguous()
        bl, _ = segment_blocks(poff)
        fl = _lib.RANGE_EXCLUDE_SELF | _lib.RANGE_OUT_PHYSICAL | (_lib.RANGE_MERGE if j else 0) | \
            (_lib.RANGE_BUILD_PAD if j == p - 1 else 0)
        range_topk(ctx, vec, vn, vec, vn, bl, lo1, rg1, degree, flags=fl, row_map=order32,
                   out_ids=adj, out_dists=dists, out_stride=degree, rows_bf16=vb, cols_bf16=vb)
        del order, order32, bl
    t4 = time.time()
    cand = float((off[probes + 1] - off[probes]).sum(1).double().mean())
    del probes
    del dists, vb
    if optimize:  # CAGRA-style rank pruning + reverse edges (csrc/graph_opt.cu)
        torch.cuda.empty_cache()
        _sync()
        ctx.optimize_graph_device(pa, n, degree, keep or degree // 2)
    t5 = time.time()
    _sync()
    ctx.partition_commit_device(_lib.COMMIT_ENTRY_ORDER | _lib.COMMIT_IOTA_IDS)
    t6 = time.time()
    info = {"n": n, "fine_clusters": nf, "coarse_clusters": int(coarse.shape[0]), "probe": p,
            "knn_kernel": "K7 tcgen05 (bf16, TMEM)" if tensor_cores and dpad <= 256 else "K7 CUDA-core fp32",
            "shortlist": q, "candidates_per_row": cand, "blocks": nb, "optimized": bool(optimize),
            "seconds": {"kmeans": t1 - t0, "assign_sort": t2 - t1, "store": t3 - t2, "knn": t4 - t3,
                        "optimize": t5 - t4, "commit_entry_order": t6 - t5, "total": t6 - t0},
            "perm": perm}
    if log:
        log(f"[ivf] graph: n={n} C={nf} probe={p}/{q} ~{cand:.0f} candidates/row, "
            f"{info['seconds']['total']:.1f}s ({', '.join(f'{k} {v:.1f}' for k, v in info['seconds'].items())})")
    return info


def brute_force_topk(ctx, db, dbn, queries, k: int, splits: int = 0, db_bf16=None):
    """Exact top-k (dist, id) of each query row over all db rows (topk.cpp:12-30;
    exact on integer-valued data): K7 over column splits, then a per-query merge.
    -> (ids int64 nq x k, dists float32 nq x k) tensors."""
    torch = _torch()
    dev = db.device
    n = db.shape[0]
    nq = queries.shape[0]
    qb = (nq + TR - 1) // TR
    if not splits:
        splits = max(1, min(n // 4096 + 1, (8 * 148 + qb - 1) // qb))
    cut = torch.linspace(0, n, splits + 1, device=dev).round().long()
    rg = torch.stack([cut[:-1], cut[1:]], 1).to(torch.int32).contiguous()
    lo = torch.arange(splits + 1, dtype=torch.int32, device=dev)
    qoff = torch.tensor([0, nq], dtype=torch.int64, device=dev)
    qblocks, nbq = segment_blocks(qoff, torch.zeros(1, dtype=torch.int64, device=dev))
    bl = qblocks.repeat(splits, 1)
    sidx = torch.repeat_interleave(torch.arange(splits, device=dev, dtype=torch.int32), nbq)
    bl[:, 2] = sidx
    bl[:, 3] = bl[:, 0] + sidx * nq
    qn = row_norms(ctx, queries)
    ids = torch.empty((splits * nq, k), dtype=torch.int32, device=dev)
    dists = torch.empty((splits * nq, k), dtype=torch.float32, device=dev)
    qb = to_bf16(ctx, queries) if db_bf16 is not None else None
    range_topk(ctx, queries, qn, db, dbn, bl.contiguous(), lo, rg, k, out_ids=ids, out_dists=dists,
               rows_bf16=qb, cols_bf16=db_bf16)
    ids = ids.view(splits, nq, k).permute(1, 0, 2).reshape(nq, splits * k).to(torch.int64)
    dists = dists.view(splits, nq, k).permute(1, 0, 2).reshape(nq, splits * k)
    valid = ids >= 0
    key = (dists.contiguous().view(torch.int32).to(torch.int64) << 32) | (ids & 0xFFFFFFFF)
    key = torch.where(valid, key, torch.full_like(key, torch.iinfo(torch.int64).max))
    top = torch.sort(key, dim=1).values[:, :k]
    out_ids = (top & 0xFFFFFFFF)
    out_d = (top >> 32).to(torch.int32).view(torch.float32)
    return out_ids, out_d


def sift_like_device(n: int, dim: int, rank: int = 16, seed: int = 1, scale: float = 40.0,
                     device="cuda:0", dpad: Optional[int] = None, chunk: int = 1 << 22, out=None):
    """SIFT-/Deep-like integer-valued data generated on the GPU (torch Philox,
    deterministic for a seed): x = round(40 (A z + 0.1 eps) + 128) clipped to
    [0, 255], z ~ N(0, I_rank), A ~ N(0, 1/rank) -- the generator of
    synth.sift_like, without a 38 GB host round trip.  Rows padded to dpad."""
    import torch
    dpad = dpad or ((dim + 3) & ~3)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    a = torch.randn((rank, dim), generator=g, device=device, dtype=torch.float32) / float(np.sqrt(rank))
    if out is None:
        out = torch.zeros((n, dpad), dtype=torch.float32, device=device)
    for b in range(0, n, chunk):
        e = min(n, b + chunk)
        z = torch.randn((e - b, rank), generator=g, device=device, dtype=torch.float32)
        eps = torch.randn((e - b, dim), generator=g, device=device, dtype=torch.float32)
        xb = torch.addmm(eps, z, a, beta=0.1, alpha=1.0)  # z a + 0.1 eps
        out[b:e, :dim] = torch.clamp(torch.round(xb * scale + 128.0), 0.0, 255.0)
    return out


def sift_like_queries_device(nq: int, dim: int, rank: int = 16, data_seed: int = 1, seed: int = 2,
                             scale: float = 40.0, device="cuda:0", dpad: Optional[int] = None):
    """Fresh points from the same subspace A as sift_like_device(seed=data_seed)."""
    import torch
    dpad = dpad or dim
    g = torch.Generator(device=device)
    g.manual_seed(int(data_seed))
    a = torch.randn((rank, dim), generator=g, device=device, dtype=torch.float32) / float(np.sqrt(rank))
    gq = torch.Generator(device=device)
    gq.manual_seed(int(seed))
    z = torch.randn((nq, rank), generator=gq, device=device, dtype=torch.float32)
    eps = torch.randn((nq, dim), generator=gq, device=device, dtype=torch.float32)
    out = torch.zeros((nq, dpad), dtype=torch.float32, device=device)
    out[:, :dim] = torch.clamp(torch.round(torch.addmm(eps, z, a, beta=0.1) * scale + 128.0), 0.0, 255.0)
    return out


def embedding_like_device(n: int, dim: int = 768, rank: int = 32, seed: int = 3, noise: float = 0.05,
                          device="cuda:0", chunk: int = 1 << 21, out=None, basis_seed: Optional[int] = None):
    """Text-embedding-like float data for BASELINE configs[3]:
    x = z B + noise * eps with z ~ N(0, I_rank), B ~ N(0, 1) (rank x dim), rows
    L2-normalised.  Float-valued: the search runs in a parity mode (f32c/f64).
    `basis_seed` (default `seed`) fixes B, so queries can share the data's B."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed if basis_seed is None else basis_seed))
    b = torch.randn((rank, dim), generator=g, device=device, dtype=torch.float32)
    if basis_seed is not None:
        g.manual_seed(int(seed))
    if out is None:
        out = torch.empty((n, dim), dtype=torch.float32, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        z = torch.randn((e - s, rank), generator=g, device=device, dtype=torch.float32)
        eps = torch.randn((e - s, dim), generator=g, device=device, dtype=torch.float32)
        xb = torch.addmm(eps, z, b, beta=noise, alpha=1.0)
        out[s:e] = xb / torch.linalg.vector_norm(xb, dim=1, keepdim=True)
    return out


def topk_ip_device(db, queries, k: int, chunk: int = 0):
    """Exact-order top-k by (f32(-dot), id) over all rows -- the inner-product
    restatement of brute_force_topk (topk.cpp:12-30) for ground truth at
    k > 32.  dot in fp64 per chunk (torch), then rounded to f32 like the
    search's distances.  -> int64 ids (nq x k)."""
    import torch
    n = db.shape[0]
    chunk = chunk or max(4096, (1 << 27) // max(1, queries.shape[0]))  # ~1 GB per int64 temporary
    best = None
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        d = -(queries.double() @ db[s:e].double().T)
        key = (d.float().contiguous().view(torch.int32).to(torch.int64))
        # order-preserving map of the f32 bit pattern, then id as the tie-break
        key = torch.where(key < 0, ~key & 0xFFFFFFFF, key | 0x80000000)
        key = (key << 32) | torch.arange(s, e, device=db.device, dtype=torch.int64)[None, :]
        key = key ^ (1 << 63)  # int64 compare on the unsigned key
        cand = torch.topk(key, min(k, e - s), dim=1, largest=False).values
        best = cand if best is None else torch.topk(torch.cat([best, cand], 1), k, dim=1, largest=False).values
    return (best ^ (1 << 63)) & 0xFFFFFFFF
