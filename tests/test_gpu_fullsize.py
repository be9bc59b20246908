"""Size-independent properties at the full BASELINE cfg1 size (1M x 128,
kNN-32 graph, beam 64, I=6), where the CPU oracle cannot finish in seconds:

* every result list ascending by (dist, global id), ids unique and inside the
  partition, count = min(k, pool) = k, distances equal to a direct fp64
  squared_l2 of the returned rows (distance.cpp:19-27),
* visited within the reference's bound entry + I*w*d_g (test_graph_index.cpp:149),
* determinism (two runs bit-identical) and f32 mode == f64 parity mode on
  integer-valued data,
* node-sharded search (bulk exchange, 4 emulated ranks) == unsharded,
* a bounded sample still bit-identical to the reference's own C++
  (oracle/_ref), which is what bench.py checks on 34k queries.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2512_02278_b200 as dvs  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg1(ctx):
    import torch

    import bench
    args = bench.parse(["--workload", "cfg1", "--nq", "4000"])
    ctx.reset()
    ctx._single_key = None
    w = bench.build_cfg1(args, 0, ctx, torch.device("cuda", 0))  # loads the index into ctx
    data, adj = w.host
    g = dvs.GraphIndex(data, np.arange(data.shape[0], dtype=np.uint32), 32, adj, None)
    return data, w.queries.cpu().numpy(), g


def test_fullsize_properties(ctx, cfg1):
    data, queries, g = cfg1
    I, w, k, E = 6, 64, 10, 64
    ids, dists, counts, visited = ctx.beam_search(0, queries, dvs.SearchParams(I, w, k, E, accum="f32"))
    assert (counts == k).all()
    assert (visited <= E + I * w * 32).all() and (visited >= E).all()
    for q in range(0, len(queries), 37):
        row_ids = ids[q]
        assert len(set(row_ids.tolist())) == k and row_ids.max() < data.shape[0]
        keys = list(zip(dists[q].tolist(), row_ids.tolist()))
        assert keys == sorted(keys)
        diff = data[row_ids].astype(np.float64) - queries[q].astype(np.float64)
        assert np.array_equal(dists[q], (diff * diff).sum(1).astype(np.float32))
    again = ctx.beam_search(0, queries, dvs.SearchParams(I, w, k, E, accum="f32"))
    for a, b in zip(again, (ids, dists, counts, visited)):
        assert np.array_equal(a, b)
    exact = ctx.beam_search(0, queries, dvs.SearchParams(I, w, k, E, accum="f64"))
    for a, b in zip(exact, (ids, dists, counts, visited)):
        assert np.array_equal(a, b)
    sharded = ctx.beam_search_sharded_emulated(4, queries[:2000], dvs.SearchParams(I, w, k, E, accum="f32"))
    for a, b in zip(sharded, (ids[:2000], dists[:2000], counts[:2000], visited[:2000])):
        assert np.array_equal(a, b)


def test_fullsize_sample_matches_reference(ctx, cfg1, ref):
    data, queries, g = cfg1
    I, w, k, E = 6, 64, 10, 64
    sub = queries[:200]
    ids, dists, counts, visited = ctx.beam_search(0, sub, dvs.SearchParams(I, w, k, E, accum="f64"))
    rg = ref.graph_from_arrays(data, g.global_ids, g.adjacency)  # entry order recomputed by the reference
    want = rg.beam_search(sub, I, w, k, E)
    assert np.array_equal(counts, want[2]) and np.array_equal(visited, want[3])
    for q in range(len(sub)):
        n = int(counts[q])
        assert np.array_equal(ids[q, :n], want[0][q, :n])
        assert np.array_equal(dists[q, :n], want[1][q, :n])


def test_cfg3_fullsize_properties(ctx):
    """The bench's cfg3 index (100M x 96, GPU-built graph) at full size:
    result order / uniqueness / exact fp64 distances of the returned rows,
    the visited bound, determinism, f32 == f64 on integer data and the
    node-sharded search (4 emulated ranks) == unsharded."""
    import torch

    import bench
    args = bench.parse(["--nq", "20000", "--recall-sample", "500"])
    ctx.reset()
    ctx._single_key = None
    w = bench.build_cfg3(args, 0, ctx, torch.device("cuda", 0))
    I, wd, k, E = args.iterations, args.beam, args.k, args.entry
    q = w.queries.cpu().numpy()
    ids, dists, counts, visited = ctx.beam_search(0, q, dvs.SearchParams(I, wd, k, E, accum="f32"))
    assert (counts == k).all()
    assert (visited <= E + I * wd * 32).all() and (visited >= E).all()
    rows = np.arange(0, len(q), 97)
    vec = w.vec[torch.from_numpy(ids[rows].astype(np.int64).reshape(-1)).cuda()].cpu().numpy()
    vec = vec.reshape(len(rows), k, -1)[:, :, :args.dim]
    for j, r in enumerate(rows):
        assert len(set(ids[r].tolist())) == k and int(ids[r].max()) < args.n
        keys = list(zip(dists[r].tolist(), ids[r].tolist()))
        assert keys == sorted(keys)
        diff = vec[j].astype(np.float64) - q[r].astype(np.float64)
        assert np.array_equal(dists[r], (diff * diff).sum(1).astype(np.float32))
    rec = bench.recall_at_k(ids[:w.gt.shape[0]], counts[:w.gt.shape[0]], w.gt, k)
    assert rec >= 0.95
    again = ctx.beam_search(0, q, dvs.SearchParams(I, wd, k, E, accum="f32"))
    exact = ctx.beam_search(0, q[:5000], dvs.SearchParams(I, wd, k, E, accum="f64"))
    for a, b, c in zip(again, exact, (ids, dists, counts, visited)):
        assert np.array_equal(a, c) and np.array_equal(b, c[:5000])
    sharded = ctx.beam_search_sharded_emulated(4, q[:2000], dvs.SearchParams(I, wd, k, E, accum="f32"))
    for a, c in zip(sharded, (ids, dists, counts, visited)):
        assert np.array_equal(a, c[:2000])
    del w
    ctx.reset()
    torch.cuda.empty_cache()
