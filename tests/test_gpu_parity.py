"""GPU parity: the sm_100a path through the C-ABI against the oracle and the
reference's golden fixtures.  Bar: integer/index outputs bit-exact (ids,
counts, visited); distances bit-exact in f64 mode and on integer data.  The
f32 mode is exact on integer data and is upgraded to a parity mode (f64, or
f32c for inner product / wide rows) on float data; at scale the float-data
bar is north_star's (>= 99.9% identical id lists, 1e-4 relative)."""
import os

import numpy as np
import pytest

import paper_2512_02278_b200 as dvs
from conftest import sift_like

pytestmark = pytest.mark.gpu


def _graph(v, adj, gids=None, eo=None):
    gids = np.arange(v.shape[0], dtype=np.uint32) if gids is None else gids
    return dvs.GraphIndex(v, gids, adj.shape[1], adj, eo)


def _search(ctx, v, adj, q, p, gids=None, eo=None):
    ctx.reset()
    ctx._single_key = None
    ctx.load_partition(0, _graph(v, adj, gids, eo))
    return ctx.beam_search(0, q, p)


def _assert_same(got, want, exact_dists=True, tag=""):
    gi, gd, gc, gv = got
    wi, wd, wc, wv = want
    assert np.array_equal(gc, wc), tag
    assert np.array_equal(gv, wv), tag
    for q in range(len(wc)):
        n = int(wc[q])
        assert np.array_equal(gi[q, :n], wi[q, :n]), (tag, q)
        if exact_dists:
            assert np.array_equal(gd[q, :n], wd[q, :n]), (tag, q)
        else:
            np.testing.assert_allclose(gd[q, :n], wd[q, :n], rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("fixture", ["g1_uniform.npz", "g2_siftlike.npz"])
@pytest.mark.parametrize("accum", ["f64", "f32"])
def test_search_matches_reference_golden(ctx, golden, fixture, accum):
    g = golden(fixture)
    v, adj, q = g["vectors"], g["adjacency"], g["queries"]
    gids = g["gids"] if "gids" in g.files else None
    for i, (I, w, k, E) in enumerate(g["params"]):
        p = dvs.SearchParams(int(I), int(w), int(k), int(E), accum=accum)
        got = _search(ctx, v, adj, q, p, gids)
        want = (g[f"ids{i}"], g[f"dists{i}"], g[f"counts{i}"], g[f"visited{i}"])
        # f64 always; f32 is exact on integer data (g2) and upgraded to a parity
        # mode on float data (g1), so every case is bit-exact
        _assert_same(got, want, True, (fixture, i, accum))


def test_entry_order_on_upload_matches_reference(ctx, golden):
    g = golden("g1_uniform.npz")
    ctx.reset()
    ctx.load_partition(7, _graph(g["vectors"], g["adjacency"], g["gids"]))
    assert np.array_equal(ctx.entry_order(7), g["entry_order"])


@pytest.mark.parametrize("n,dim,dg,I,w,k,E", [
    (3000, 128, 32, 6, 64, 10, 64),   # cfg1 shape (VPL=1)
    (2500, 96, 32, 6, 32, 10, 32),    # cfg3 dim (24 active lanes)
    (1200, 200, 16, 4, 16, 20, 8),    # dpad=200, VPL=2
    (900, 768, 32, 3, 16, 100, 16),   # cfg4 dim (VPL=6), k=100
    (800, 13, 7, 5, 5, 7, 3),         # ragged dim (dpad=16) and odd degree
    (50, 4, 8, 8, 64, 10, 64),        # tiny partition, entry > n
])
def test_search_matches_oracle_fresh(ctx, oracle, n, dim, dg, I, w, k, E):
    v = oracle.random_dataset(n, dim, 1000 + n)
    adj = oracle.build_graph(v, dg)
    eo = oracle.compute_entry_order(v)
    q = oracle.random_dataset(64, dim, 2000 + n)
    gids = (7 + 5 * np.arange(n)).astype(np.uint32)
    want = oracle.beam_search(v, gids, adj, eo, q, I, w, k, E)
    got = _search(ctx, v, adj, q, dvs.SearchParams(I, w, k, E, accum="f64"), gids)
    _assert_same(got, want, True, (n, dim))


@pytest.mark.parametrize("gid_order", ["increasing", "shuffled"])
@pytest.mark.parametrize("I,w,k,E", [(6, 16, 10, 16), (2, 4, 10, 4), (3, 8, 50, 8), (1, 2, 5, 2)])
def test_pool_truncation_exact_under_ties(ctx, oracle, gid_order, I, w, k, E):
    """Tiny-integer coordinates (many equal distances): the pool kept at
    max(I*w, k) (increasing gids) or at the reference cap (shuffled gids)
    gives the reference's ids, dists and visited counters."""
    n, dim = 1500, 6
    rng = np.random.default_rng(5)
    v = rng.integers(0, 4, size=(n, dim)).astype(np.float32)
    adj = oracle.build_graph(v, 12)
    eo = oracle.compute_entry_order(v)
    q = rng.integers(0, 4, size=(80, dim)).astype(np.float32)
    gids = (3 + 2 * np.arange(n)).astype(np.uint32)
    if gid_order == "shuffled":
        gids = rng.permutation(gids).astype(np.uint32)
    want = oracle.beam_search(v, gids, adj, eo, q, I, w, k, E)
    for accum in ("f64", "f32"):
        got = _search(ctx, v, adj, q, dvs.SearchParams(I, w, k, E, accum=accum), gids)
        _assert_same(got, want, True, (gid_order, accum))
    ctx.reset()
    ctx._single_key = None
    ctx.load_partition(0, _graph(v, adj, gids, eo))
    got = ctx.beam_search_sharded_emulated(3, q, dvs.SearchParams(I, w, k, E, accum="f32"))
    _assert_same(got, want, True, (gid_order, "bulk sharded"))


@pytest.mark.parametrize("small_min", ["128", "0"])
def test_small_visited_table_growth_exact(ctx, oracle, monkeypatch, small_min):
    """Visited tables that start at half size and grow (exact rehash) when
    the load could pass 3/4 -- forced on small partitions -- give the
    reference's results and visited counters."""
    monkeypatch.setenv("DVSG_HASH_SMALL_MIN", small_min)
    n, dim = 6000, 16
    v = sift_like(n, dim, 6, 71)
    adj = oracle.build_graph(v, 24)
    eo = oracle.compute_entry_order(v)
    q = sift_like(48, dim, 6, 72)
    gids = np.arange(n, dtype=np.uint32)
    for (I, w, k, E) in [(6, 64, 10, 64), (3, 128, 20, 300), (2, 8, 5, 8)]:
        want = oracle.beam_search(v, gids, adj, eo, q, I, w, k, E)
        got = _search(ctx, v, adj, q, dvs.SearchParams(I, w, k, E, accum="f32"), gids)
        _assert_same(got, want, True, ("small table", small_min, I, w))


def test_global_hash_path_matches_oracle(ctx, oracle):
    # bound = min(n, E + I*w*dg) > 16384 -> the visited hash lives in global memory
    n, dim = 20000, 8
    v = oracle.random_dataset(n, dim, 77)
    adj = oracle.build_graph(v, 32)
    eo = oracle.compute_entry_order(v)
    q = oracle.random_dataset(32, dim, 78)
    gids = np.arange(n, dtype=np.uint32)
    want = oracle.beam_search(v, gids, adj, eo, q, 6, 128, 100, 128)
    got = _search(ctx, v, adj, q, dvs.SearchParams(6, 128, 100, 128))
    _assert_same(got, want, True, "global-hash")


def test_inner_product_matches_oracle(ctx, oracle):
    v = oracle.random_dataset(2000, 64, 5)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    adj = oracle.build_graph(v, 16)
    eo = oracle.compute_entry_order(v)
    q = oracle.random_dataset(64, 64, 6)
    gids = np.arange(2000, dtype=np.uint32)
    want = oracle.beam_search(v, gids, adj, eo, q, 6, 32, 10, 32, metric=1)
    got = _search(ctx, v, adj, q, dvs.SearchParams(6, 32, 10, 32, metric="ip"))
    _assert_same(got, want, True, "ip")


# ---- reference KATs through the GPU (test_graph_index.cpp) ------------------

def test_kat_complete_graph_equals_brute_force(ctx, oracle):
    v = oracle.random_dataset(9, 5, 53)  # :100-120
    g = dvs.build_graph(v, 12, ctx=ctx)
    q = oracle.random_dataset(10, 5, 54)
    p = dvs.SearchParams(1, 1, 5, 1)
    bi, bd = oracle.brute_force_topk(v, q, 5)
    for t in range(10):
        hits = dvs.beam_search(g, q[t], p, ctx=ctx)
        assert [h.id for h in hits] == bi[t].tolist()
        assert [h.dist for h in hits] == bd[t].tolist()


def test_kat_stored_vector_rank_one(ctx, oracle):
    v = oracle.random_dataset(500, 8, 55)  # :122-134
    g = dvs.build_graph(v, 32, ctx=ctx)
    hits = dvs.beam_search(g, v[123], dvs.SearchParams(4, 4, 3, 4), ctx=ctx)
    assert hits and hits[0].id == 123 and hits[0].dist == 0.0


def test_kat_visited_bounds(ctx, oracle):
    v = oracle.random_dataset(2000, 6, 56)  # :136-152
    g = dvs.build_graph(v, 32, ctx=ctx)
    p = dvs.SearchParams(6, 6, 10, 6)
    q = oracle.random_dataset(5, 6, 57)
    for t in range(5):
        vis = dvs.visited_count(g, q[t], p, ctx=ctx)
        assert 6 <= vis <= 6 * 6 * 32 + 6
    v = oracle.random_dataset(10, 3, 58)  # :154-166
    g = dvs.build_graph(v, 16, ctx=ctx)
    assert dvs.visited_count(g, np.zeros(3, np.float32), dvs.SearchParams(5, 5, 5, 3), ctx=ctx) <= 10


def test_kat_single_vector_partition(ctx):
    g = dvs.build_graph(np.array([[1, 2, 3]], np.float32), 3, global_ids=[42], ctx=ctx)
    assert g.adjacency.shape == (1, 3)
    hits = dvs.beam_search(g, np.zeros(3, np.float32), dvs.SearchParams(2, 2, 5, 1), ctx=ctx)
    assert len(hits) == 1 and hits[0].id == 42


def test_kat_deterministic_and_inside_partition(ctx, oracle):
    v = oracle.random_dataset(250, 6, 62)  # :202-227
    globals_ = (1000 + 3 * np.arange(250)).astype(np.uint32)
    g = dvs.build_graph(v, 8, global_ids=globals_, ctx=ctx)
    p = dvs.SearchParams(3, 4, 12, 4)
    q = np.array([0.1, 0.2, 0.3, 0.4, 0.5, 0.6], np.float32)
    a = dvs.beam_search_stats(g, q, p, 1, ctx=ctx)
    b = dvs.beam_search_stats(g, q, p, 99, ctx=ctx)
    assert a.visited == b.visited and a.hits == b.hits
    ids = [h.id for h in a.hits]
    assert set(ids) <= set(globals_.tolist()) and len(set(ids)) == len(ids)
    keys = [(h.dist, h.id) for h in a.hits]
    assert keys == sorted(keys)


def test_kat_recall_never_drops_with_iterations(ctx, oracle):
    v = oracle.random_dataset(400, 8, 60)  # :180-200
    g = dvs.build_graph(v, 8, ctx=ctx)
    q = oracle.random_dataset(5, 8, 61)
    truth, _ = oracle.brute_force_topk(v, q, 10)
    for t in range(5):
        prev = -1
        for iters in range(1, 9):
            hits = dvs.beam_search(g, q[t], dvs.SearchParams(iters, 2, 10, 2), ctx=ctx)
            r = len({h.id for h in hits} & set(truth[t].tolist())) / 10
            assert r >= prev
            prev = r


def test_kat_errors(ctx, oracle):
    v = oracle.random_dataset(10, 2, 63)  # :229-242
    g = dvs.build_graph(v, 3, ctx=ctx)
    with pytest.raises(dvs.InvalidArgument):
        dvs.beam_search(g, np.zeros(2, np.float32), dvs.SearchParams(iterations=0), ctx=ctx)
    with pytest.raises(dvs.InvalidArgument):
        dvs.beam_search(g, np.zeros(2, np.float32), dvs.SearchParams(iterations=1, k=0), ctx=ctx)
    with pytest.raises(dvs.InvalidArgument):
        dvs.beam_search(g, np.zeros(3, np.float32), dvs.SearchParams(iterations=1), ctx=ctx)
    with pytest.raises(dvs.InvalidArgument):
        dvs.build_graph(np.zeros((0, 4), np.float32), 4, ctx=ctx)


# ---- graph build (K6) -----------------------------------------------------------

@pytest.mark.parametrize("n,dim,dg", [(200, 8, 8), (3000, 32, 32), (31, 4, 32), (2, 2, 4), (1, 3, 3)])
def test_build_graph_matches_reference(ctx, oracle, n, dim, dg):
    # integer-valued data: fp32 distances exact -> rows bit-identical to build_graph
    v = sift_like(n, dim, 4, n)
    want = oracle.build_graph(v, dg)
    got = ctx.build_graph(v, dg)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,dim,dg", [(3000, 37, 32), (2500, 96, 16), (700, 128, 24), (5, 7, 8), (1, 3, 3),
                                      (33, 5, 32)])
def test_build_graph_float_data_exact(ctx, ref, oracle, n, dim, dg):
    """K6 exact mode (fp32 candidates + fp64 re-rank + certificate + fp64
    fallback): rows bit-identical to the compiled reference's build_graph on
    float data, incl. tiny partitions (cyclic rows) and a lone node."""
    rng = np.random.default_rng(n + dim)
    v = rng.normal(size=(n, dim)).astype(np.float32)
    _, want, _ = ref.build_graph(v, dg)
    got = ctx.build_graph(v, dg)
    assert ctx.last_knn_info()[0] == 1
    assert np.array_equal(got, want), np.argwhere(np.any(got != want, axis=1))[:5]
    assert np.array_equal(got, oracle.build_graph(v, dg))


def test_build_graph_float_ties_and_fallback(ctx, ref):
    """Exact ties (duplicated rows) and near-ties (points on a sphere around a
    centre row: distances equal up to rounding) that the certificate must
    hand to the fp64 fallback; rows still equal the reference's."""
    rng = np.random.default_rng(9)
    v = rng.normal(size=(1500, 24)).astype(np.float32)
    v[100:120] = v[7]
    ring = rng.normal(size=(60, 24))
    ring = ring / np.linalg.norm(ring, axis=1, keepdims=True) * 0.5
    v[200] = 0.0
    v[201:261] = ring.astype(np.float32)
    for dg in (8, 32):
        _, want, _ = ref.build_graph(v, dg)
        assert np.array_equal(ctx.build_graph(v, dg), want), dg
        mode, fb = ctx.last_knn_info()
        assert mode == 1 and fb >= 1, (mode, fb)  # the sphere centre went to the fp64 scan


def test_brute_force_float_data_exact(ctx, ref):
    """brute_force_topk (topk.cpp:12-30) on float data, k = 10 and 32: ids and
    fp32 distances bit-identical to the reference, incl. duplicated rows."""
    rng = np.random.default_rng(4)
    v = rng.normal(size=(20000, 64)).astype(np.float32)
    v[500:510] = v[3]
    q = rng.normal(size=(300, 64)).astype(np.float32)
    q[0] = v[3]
    for k in (10, 32):
        wi, wd = ref.brute_force_topk(v, q, k)
        gi, gd = ctx.brute_force_topk(v, q, k)
        assert ctx.last_knn_info()[0] == 1
        assert np.array_equal(gi, wi) and np.array_equal(gd, wd), k


def test_build_graph_golden(ctx, golden):
    g = golden("g2_siftlike.npz")
    assert np.array_equal(ctx.build_graph(g["vectors"], 32), g["adjacency"])


# ---- routing / merge / pipeline ------------------------------------------------

def test_combine_matches_reference_golden(ctx, golden):
    g = golden("g4_combine.npz")
    for i in range(int(g["ncases"])):
        hits = [[dvs.ScoredId(int(a), float(b)) for a, b in zip(g[f"c{i}_ids"][j][:c], g[f"c{i}_dists"][j][:c])]
                for j, c in enumerate(g[f"c{i}_counts"])]
        out = dvs.combine_results(hits, int(g[f"c{i}_k"]), ctx=ctx)
        assert [h.id for h in out] == g[f"c{i}_oi"].tolist()
        assert [h.dist for h in out] == g[f"c{i}_od"].tolist()


def test_combine_rejects_unsorted_partial(ctx):
    bad = [[dvs.ScoredId(1, 2.0), dvs.ScoredId(2, 1.0)]]
    with pytest.raises(dvs.InternalError, match="not sorted"):
        dvs.combine_results(bad, 3, ctx=ctx)


def test_assign_matches_reference(ctx, oracle, golden):
    q = oracle.random_dataset(25, 8, 45, -1000, 1000)  # test_kmeans.cpp:156-189
    c = oracle.random_dataset(16, 8, 46, -1000, 1000)
    assert np.array_equal(dvs.assign_top_c(c, q, 16, ctx=ctx), oracle.assign_top_c(c, q, 16))
    cents = np.array([[0, 0], [10, 0]], np.float32)  # tie -> lower id
    assert dvs.assign_top_c(cents, np.array([[5, 0]], np.float32), 1, ctx=ctx).tolist() == [[0]]
    with pytest.raises(dvs.InvalidArgument):
        dvs.assign_top_c(cents, np.array([[5, 0]], np.float32), 3, ctx=ctx)


@pytest.mark.parametrize("clusters,dim,c", [(128, 8, 4), (300, 37, 9), (1000, 128, 32), (513, 96, 1)])
def test_assign_large_c_tiled_matches_reference(ctx, oracle, clusters, dim, c):
    """Large-C K5 (register-tiled fp64 with the reference's accumulation
    order + per-lane top-c selection) equals assign_top_c, ties by lower id
    (duplicated centroids force exact distance ties)."""
    cents = oracle.random_dataset(clusters, dim, 400 + clusters, -100, 100)
    cents[clusters // 2:clusters // 2 + 5] = cents[3]
    q = oracle.random_dataset(333, dim, 500 + clusters, -100, 100)
    q[7] = cents[3]
    want = oracle.assign_top_c(cents, q, c)
    got = dvs.assign_top_c(cents, q, c, ctx=ctx)
    assert np.array_equal(got, want)


def test_pipeline_pinned_and_pageable_schedules_agree(ctx, golden):
    """dvsg_run_pipeline picks its copy schedule from the host buffers
    (pinned: all H2D first; pageable: interleaved); both equal the golden."""
    import torch
    from fnsy import G3_FNSY
    res = golden("g3_mixture.npz")
    dvs.load_index(G3_FNSY, ctx=ctx)
    q = res["queries"]
    nq, dim = q.shape
    k = 10
    pq = torch.empty((nq, dim), dtype=torch.float32).pin_memory().numpy()
    pq[:] = q
    out = {"ids": torch.empty((nq, k), dtype=torch.int32).pin_memory().numpy().view(np.uint32),
           "dists": torch.empty((nq, k), dtype=torch.float32).pin_memory().numpy(),
           "counts": torch.empty((nq,), dtype=torch.int32).pin_memory().numpy().view(np.uint32),
           "vectors": torch.empty((nq, k, dim), dtype=torch.float32).pin_memory().numpy()}
    p = dvs.SearchParams(6, 16, 10, 16)
    pinned = ctx.run_pipeline(pq, p, 2, 4, batch_index=1, out=out)
    pageable = ctx.run_pipeline(q.copy(), p, 2, 4, batch_index=1)
    for a, b in ((pinned.ids, pageable.ids), (pinned.dists, pageable.dists), (pinned.counts, pageable.counts),
                 (pinned.hit_vectors, pageable.hit_vectors)):
        assert np.array_equal(a, b)
    assert np.array_equal(pinned.counts, res["counts_f2"])
    assert pinned.visited_total == pageable.visited_total == int(res["visited_f2"])


def test_pipeline_matches_reference_golden(ctx, golden):
    from fnsy import G3_FNSY
    res = golden("g3_mixture.npz")
    dvs.load_index(G3_FNSY, ctx=ctx)
    q = res["queries"]
    for fo in (1, 2, 3):
        r = ctx.run_pipeline(q, dvs.SearchParams(6, 16, 10, 16), fo, 4, batch_index=1)
        assert np.array_equal(r.counts, res[f"counts_f{fo}"])
        for i in range(len(q)):
            n = int(r.counts[i])
            assert np.array_equal(r.ids[i, :n], res[f"ids_f{fo}"][i, :n])
            assert np.array_equal(r.dists[i, :n], res[f"dists_f{fo}"][i, :n])
            assert np.array_equal(r.hit_vectors[i, :n], res[f"vectors_f{fo}"][i, :n])
        assert r.visited_total == int(res[f"visited_f{fo}"])
    with pytest.raises(dvs.InvalidArgument, match="fanout"):
        ctx.run_pipeline(q, dvs.SearchParams(6, 16, 10, 16), 9, 4)
    with pytest.raises(dvs.InvalidArgument, match="ranks"):
        ctx.run_pipeline(q, dvs.SearchParams(6, 16, 10, 16), 2, 8)


def test_device_entry_points_and_distributed_pipeline_single_rank(ctx, golden):
    """assign/combine/gather device entry points and the cluster-sharded
    pipeline's route -> search -> return -> combine path (one NCCL rank)
    reproduce the reference's run_pipeline golden."""
    import socket
    import torch
    import torch.distributed as dist
    from fnsy import G3_FNSY
    from paper_2512_02278_b200.dist import run_pipeline_distributed
    res = golden("g3_mixture.npz")
    dvs.load_index(G3_FNSY, ctx=ctx)
    q = res["queries"]
    dev = torch.device("cuda", 0)
    d_q = torch.from_numpy(q).to(dev)
    out = torch.empty((len(q), 3), dtype=torch.int32, device=dev)
    ctx.assign_top_c_device(d_q.data_ptr(), len(q), q.shape[1], 3, out.data_ptr())
    ctx.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ctx.assign_top_c(q, 3))
    own_pg = not dist.is_initialized()
    if own_pg:
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=dev)
    try:
        _distributed_pipeline_checks(ctx, res, q, d_q, dev)
    finally:
        if own_pg:
            dist.destroy_process_group()


def _distributed_pipeline_checks(ctx, res, q, d_q, dev):
    import torch
    from paper_2512_02278_b200.dist import run_pipeline_distributed
    placement = torch.zeros(8, dtype=torch.int64, device=dev)
    for fo in (1, 2, 3):
        ids, dists, counts, vecs, vt = run_pipeline_distributed(ctx, d_q, dvs.SearchParams(6, 16, 10, 16), fo,
                                                                placement, 1)
        ctx.synchronize()
        cnt = counts.cpu().numpy().view(np.uint32)
        assert np.array_equal(cnt, res[f"counts_f{fo}"])
        gi, gd, gv = ids.cpu().numpy().view(np.uint32), dists.cpu().numpy(), vecs.cpu().numpy()
        for i in range(len(q)):
            n = int(cnt[i])
            assert np.array_equal(gi[i, :n], res[f"ids_f{fo}"][i, :n])
            assert np.array_equal(gd[i, :n], res[f"dists_f{fo}"][i, :n])
            assert np.array_equal(gv[i, :n], res[f"vectors_f{fo}"][i, :n])
        assert vt == int(res[f"visited_f{fo}"])


def test_load_index_rank_filter(ctx):
    from fnsy import G3_FNSY, read_fnsy
    idx = read_fnsy(G3_FNSY)
    dvs.load_index(G3_FNSY, ctx=ctx, rank=1)
    info = ctx.info()
    want = [c for c in range(8) if idx.cluster_to_rank[c] == 1]
    assert info["cluster_ids"].tolist() == want


def test_load_index_format_errors(ctx, tmp_path):
    from fnsy import G3_FNSY
    raw = open(G3_FNSY, "rb").read()
    bad = tmp_path / "bad.fnsy"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(dvs.FormatError, match="bad magic"):
        dvs.load_index(str(bad), ctx=ctx)
    bad.write_bytes(raw[:-7])
    with pytest.raises(dvs.FormatError, match="truncated"):
        dvs.load_index(str(bad), ctx=ctx)


# ---- node-sharded search (ranks emulated in one launch) ------------------------

@pytest.mark.parametrize("exchange", ["bulk", "fused"])
@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_sharded_emulated_matches_unsharded(ctx, oracle, nranks, exchange):
    n, dim = 3000, 32
    v = sift_like(n, dim, 6, 91)
    adj = oracle.build_graph(v, 32)
    eo = oracle.compute_entry_order(v)
    q = sift_like(96, dim, 6, 92)
    gids = (5 + 2 * np.arange(n)).astype(np.uint32)
    p = dvs.SearchParams(6, 32, 10, 32, accum="f32")
    want = oracle.beam_search(v, gids, adj, eo, q, 6, 32, 10, 32)
    ctx.reset()
    ctx._single_key = None
    ctx.load_partition(0, _graph(v, adj, gids, eo))
    ctx.set_shard_exchange(exchange)
    try:
        got = ctx.beam_search_sharded_emulated(nranks, q, p)
    finally:
        ctx.set_shard_exchange("bulk")
    _assert_same(got, want, True, f"sharded {exchange} R={nranks}")


def test_sharded_bulk_waves_and_shapes(ctx, oracle, monkeypatch):
    """Bulk exchange split into many small waves (DVSG_XG_WAVE), odd dim,
    ragged rank split, tiny partition (entry_count > n), IP metric, f64."""
    monkeypatch.setenv("DVSG_XG_WAVE", "7")
    for (n, dim, nq, R, w, k, E, metric, accum) in [(2500, 37, 61, 3, 16, 10, 16, "l2", "f32"),
                                                      (900, 12, 3, 8, 8, 5, 8, "l2", "f32"),  # ranks without queries
                                                      (40, 8, 23, 4, 8, 20, 64, "l2", "f64"),
                                                      (1800, 24, 50, 2, 32, 5, 32, "ip", "f32")]:
        v = sift_like(n, dim, 6, 301 + n)
        adj = oracle.build_graph(v, 16)
        eo = oracle.compute_entry_order(v)
        q = sift_like(nq, dim, 6, 302 + n)
        gids = (7 + 3 * np.arange(n)).astype(np.uint32)
        p = dvs.SearchParams(5, w, k, E, metric=metric, accum=accum)
        ctx.reset()
        ctx._single_key = None
        ctx.load_partition(0, _graph(v, adj, gids, eo))
        want = ctx.beam_search(0, q, p)
        got = ctx.beam_search_sharded_emulated(R, q, p)
        _assert_same(got, want, True, ("bulk waves", n, dim, R, metric))


@pytest.mark.parametrize("exchange", ["bulk", "fused", "nccl"])
def test_sharded_multi_gpu_api_single_rank(oracle, exchange):
    """The real multi-GPU entry points (shard_init / IPC export + connect /
    NCCL connect / prepare / search_sharded_device) at one rank: every code
    path of the device-side exchange runs, results equal the reference."""
    import torch
    n, dim = 2500, 24
    v = sift_like(n, dim, 6, 501)
    adj = oracle.build_graph(v, 16)
    eo = oracle.compute_entry_order(v)
    q = sift_like(70, dim, 6, 502)
    gids = np.arange(n, dtype=np.uint32)
    I, w, k, E = 5, 24, 10, 24
    want = oracle.beam_search(v, gids, adj, eo, q, I, w, k, E)
    cx = dvs.Context(0)
    try:
        cx.set_shard_exchange(exchange)
        cx.shard_init(1, 0, v, n, adj, eo)
        cx.shard_connect([cx.shard_export()])
        if exchange == "nccl":
            cx.nccl_connect(cx.nccl_unique_id())
        cx.shard_prepare()
        dev = torch.device("cuda", 0)
        d_q = torch.from_numpy(q).to(dev)
        ids = torch.empty((len(q), k), dtype=torch.int32, device=dev)
        dists = torch.empty((len(q), k), dtype=torch.float32, device=dev)
        cnt = torch.empty((len(q),), dtype=torch.int32, device=dev)
        vis = torch.empty((len(q),), dtype=torch.int64, device=dev)
        cx.search_sharded_device(d_q.data_ptr(), len(q), dim, dvs.SearchParams(I, w, k, E, accum="f32"),
                                 ids.data_ptr(), dists.data_ptr(), cnt.data_ptr(), vis.data_ptr())
        cx.synchronize()
        got = (ids.cpu().numpy().view(np.uint32), dists.cpu().numpy(), cnt.cpu().numpy().view(np.uint32),
               vis.cpu().numpy().view(np.uint64))
        _assert_same(got, want, True, exchange)
    finally:
        cx.close()


def test_sharded_emulated_golden(ctx, golden):
    g = golden("g1_uniform.npz")
    v, adj, q = g["vectors"], g["adjacency"], g["queries"]
    ctx.reset()
    ctx._single_key = None
    ctx.load_partition(0, _graph(v, adj, g["gids"]))
    for i, (I, w, k, E) in enumerate(g["params"]):
        p = dvs.SearchParams(int(I), int(w), int(k), int(E), accum="f64")
        got = ctx.beam_search_sharded_emulated(4, q, p)
        want = (g[f"ids{i}"], g[f"dists{i}"], g[f"counts{i}"], g[f"visited{i}"])
        _assert_same(got, want, True, ("sharded golden", i))


def test_pipeline_rejects_non_finite_query(ctx, golden):
    from fnsy import G3_FNSY
    res = golden("g3_mixture.npz")
    dvs.load_index(G3_FNSY, ctx=ctx)
    q = res["queries"].copy()
    q[57, 3] = np.nan  # dataset.cpp:18-33
    with pytest.raises(dvs.InvalidArgument, match="non-finite"):
        ctx.run_pipeline(q, dvs.SearchParams(6, 16, 10, 16), 2, 4, batch_index=1)


def test_pipeline_microbatched_matches_golden(ctx, golden):
    # 200 golden queries tiled to 60k: several pipelined microbatches, same answers
    from fnsy import G3_FNSY
    res = golden("g3_mixture.npz")
    dvs.load_index(G3_FNSY, ctx=ctx)
    reps = 300
    q = np.tile(res["queries"], (reps, 1))
    r = ctx.run_pipeline(q, dvs.SearchParams(6, 16, 10, 16), 2, 4, batch_index=1)
    assert np.array_equal(r.counts, np.tile(res["counts_f2"], reps))
    assert np.array_equal(r.ids, np.tile(res["ids_f2"], (reps, 1)))
    assert np.array_equal(r.hit_vectors, np.tile(res["vectors_f2"], (reps, 1, 1)))
    assert r.visited_total == reps * int(res["visited_f2"])


# ---- BASELINE config shapes at parity-test scale (configs[2..4]) ---------------

def test_cfg4_shape_ip768_k100_beam256(ctx, oracle):
    # text-embedding-like: 768-d, L2-normalised, inner product, top-100, beam 256
    # (pool cap 3072 > 2048 -> the large final-sort path; visited bound > 16k)
    n, dim = 4000, 768
    rng = np.random.default_rng(4)
    basis = rng.normal(size=(32, dim)).astype(np.float32)
    v = (rng.normal(size=(n, 32)).astype(np.float32) @ basis)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    q = (rng.normal(size=(24, 32)).astype(np.float32) @ basis)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    adj = oracle.build_graph(v, 32)
    eo = oracle.compute_entry_order(v)
    gids = np.arange(n, dtype=np.uint32)
    want = oracle.beam_search(v, gids, adj, eo, q, 6, 256, 100, 256, metric=1)
    got = _search(ctx, v, adj, q, dvs.SearchParams(6, 256, 100, 256, metric="ip", accum="f64"))
    _assert_same(got, want, True, "cfg4-shape f64")
    # f32 requested on float data runs in the compensated mode (f32c): the
    # north_star bar is >= 99.9% identical id lists, i.e. all 24 here
    got32 = _search(ctx, v, adj, q, dvs.SearchParams(6, 256, 100, 256, metric="ip", accum="f32"))
    same = sum(np.array_equal(got32[0][j, :got32[2][j]], want[0][j, :want[2][j]]) for j in range(len(q)))
    assert same >= int(np.ceil(0.999 * len(q)))
    np.testing.assert_allclose(got32[1][:, :10], want[1][:, :10], rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_f64_float_data_10k_queries_768d(ctx, oracle, metric):
    """The f64 mode on float data at scale: 10k queries at 768-d against the
    oracle's sequential fp64 (distance.cpp:19-27 order).  L2 is exact by
    construction (finish_dist) and must match every row; inner product (no
    reference) keeps north_star's bar (>= 99.9% identical id lists, 1e-4)."""
    n, dim, nq = 20000, 768, 10000
    rng = np.random.default_rng(8)
    basis = rng.normal(size=(32, dim)).astype(np.float32)
    v = rng.normal(size=(n, 32)).astype(np.float32) @ basis + 0.05 * rng.normal(size=(n, dim)).astype(np.float32)
    q = rng.normal(size=(nq, 32)).astype(np.float32) @ basis + 0.05 * rng.normal(size=(nq, dim)).astype(np.float32)
    if metric == "ip":
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        q /= np.linalg.norm(q, axis=1, keepdims=True)
    adj = ctx.build_graph(v, 32)  # any graph will do: both sides search the same one
    eo = oracle.compute_entry_order(v)
    gids = np.arange(n, dtype=np.uint32)
    want = oracle.beam_search(v, gids, adj, eo, q, 6, 32, 10, 32, metric=1 if metric == "ip" else 0,
                              nthreads=16)
    got = _search(ctx, v, adj, q, dvs.SearchParams(6, 32, 10, 32, metric=metric, accum="f64"), eo=eo)
    same = sum(np.array_equal(got[0][j, :got[2][j]], want[0][j, :want[2][j]]) for j in range(nq))
    dist_same = int(np.sum(np.all(got[1] == want[1], axis=1)))
    print(f"f64 {metric} 768-d: {same}/{nq} id lists and {dist_same}/{nq} distance rows bit-identical")
    assert same >= int(np.ceil(0.999 * nq))
    np.testing.assert_allclose(got[1], want[1], rtol=1e-4, atol=1e-6)
    vis_same = int(np.sum(got[3] == want[3]))
    print(f"  visited counters equal on {vis_same}/{nq} queries")
    assert vis_same >= int(np.ceil(0.999 * nq))
    if metric == "l2":  # exact by construction (finish_dist): every row, every distance
        assert same == nq and dist_same == nq and vis_same == nq


def test_f64_tree_sum_rounding_boundary(ctx, oracle):
    """A distance whose tree-ordered fp64 sum and the reference's sequential
    sum round to different floats: terms 1, 2^-24 (lane 0) and four 2^-54
    (lane 1).  Sequentially each 2^-54 is absorbed and the sum stays at the
    midpoint 1 + 2^-24 (-> 1.0, ties to even); the tree adds 2^-52 at once and
    lands above it (-> 1 + 2^-23).  finish_dist must detect the boundary and
    return the reference's 1.0."""
    rng = np.random.default_rng(3)
    v = (3.0 + rng.random((40, 8))).astype(np.float32)
    v[0] = np.array([1.0, 2.0 ** -12, 0, 0, 2.0 ** -27, 2.0 ** -27, 2.0 ** -27, 2.0 ** -27], np.float32)
    q = np.zeros((2, 8), np.float32)
    q[1, 1] = 2.0 ** -12  # a second boundary case: 1 + 4 x 2^-54 sequential -> 1.0
    adj = oracle.build_graph(v, 8)
    eo = oracle.compute_entry_order(v)
    gids = np.arange(len(v), dtype=np.uint32)
    # entry_count = n: every row is scored in the entry phase
    want = oracle.beam_search(v, gids, adj, eo, q, 1, 8, 5, len(v), metric=0)
    got = _search(ctx, v, adj, q, dvs.SearchParams(1, 8, 5, len(v), accum="f64"), eo=eo)
    assert want[1][0, 0] == np.float32(1.0) and want[0][0, 0] == 0
    _assert_same(got, want, True, "f64 boundary")


def test_cfg3_shape_d96_beam_sweep(ctx, oracle):
    # Deep-like 96-d, top-10, the cfg5 beam sweep 32..256
    n, dim = 6000, 96
    v = oracle.random_dataset(n, dim, 96)
    adj = oracle.build_graph(v, 32)
    eo = oracle.compute_entry_order(v)
    q = oracle.random_dataset(32, dim, 97)
    gids = np.arange(n, dtype=np.uint32)
    for w in (32, 64, 128, 256):
        want = oracle.beam_search(v, gids, adj, eo, q, 6, w, 10, w)
        got = _search(ctx, v, adj, q, dvs.SearchParams(6, w, 10, w, accum="f64"))
        _assert_same(got, want, True, f"cfg3-shape w={w}")


@pytest.mark.parametrize("dg", [1, 2, 3, 33])
def test_odd_degrees_match_oracle(ctx, oracle, dg):
    # exercises the multiply-high row index (dg == 1 special case, non-pow2 degrees)
    n, dim = 700, 16
    v = oracle.random_dataset(n, dim, 300 + dg)
    adj = oracle.build_graph(v, dg)
    eo = oracle.compute_entry_order(v)
    q = oracle.random_dataset(40, dim, 400 + dg)
    gids = np.arange(n, dtype=np.uint32)
    want = oracle.beam_search(v, gids, adj, eo, q, 8, 24, 10, 8)
    got = _search(ctx, v, adj, q, dvs.SearchParams(8, 24, 10, 8, accum="f64"))
    _assert_same(got, want, True, f"dg={dg}")


def test_brute_force_topk_matches_reference(ctx, golden, oracle):
    g = golden("g2_siftlike.npz")  # truth from the reference's brute_force_topk
    ids, d = ctx.brute_force_topk(g["vectors"], g["queries"], 10)
    assert np.array_equal(ids, g["truth_ids"]) and np.array_equal(d, g["truth_dists"])
    v = sift_like(5000, 48, 4, 77)  # many exact ties: (dist, id) order
    q = sift_like(50, 48, 4, 78)
    wi, wd = oracle.brute_force_topk(v, q, 32)
    gi, gd = ctx.brute_force_topk(v, q, 32)
    assert np.array_equal(gi, wi) and np.array_equal(gd, wd)
    with pytest.raises(dvs.InvalidArgument):
        ctx.brute_force_topk(v[:5], q, 6)


@pytest.mark.parametrize("metric,dim", [("l2", 768), ("ip", 768), ("l2", 96)])
def test_compensated_f32_matches_reference_on_float_data(ctx, oracle, metric, dim):
    # accum "f32c": TwoSum / FMA-TwoProd pairs instead of fp64.  Not a parity
    # mode: ids must agree with the reference on >= 99.9% of queries and
    # distances within 1e-6 relative (tighter than the north_star 1e-4).
    n = 2000
    v = oracle.random_dataset(n, dim, 91)
    if metric == "ip":
        v /= np.linalg.norm(v, axis=1, keepdims=True)
    adj = oracle.build_graph(v, 24)
    eo = oracle.compute_entry_order(v)
    q = oracle.random_dataset(256, dim, 92)
    gids = np.arange(n, dtype=np.uint32)
    want = oracle.beam_search(v, gids, adj, eo, q, 4, 32, 10, 32, metric=1 if metric == "ip" else 0)
    gi, gd, gc, gv = _search(ctx, v, adj, q, dvs.SearchParams(4, 32, 10, 32, metric=metric, accum="f32c"), gids)
    wi, wd, wc, wv = want
    same = sum(int(gc[i]) == int(wc[i]) and np.array_equal(gi[i, :wc[i]], wi[i, :wc[i]]) for i in range(len(q)))
    assert same >= 0.999 * len(q), (same, len(q))
    for i in range(len(q)):
        np.testing.assert_allclose(gd[i, :wc[i]], wd[i, :wc[i]], rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("exchange", ["bulk", "fused"])
@pytest.mark.parametrize("metric,dim", [("l2", 768), ("ip", 96)])
def test_compensated_f32_sharded_equals_unsharded(ctx, oracle, exchange, metric, dim):
    # same pair arithmetic in K1 and in both sharded kernels: bit-identical
    n = 1500
    v = oracle.random_dataset(n, dim, 95)
    if metric == "ip":
        v /= np.linalg.norm(v, axis=1, keepdims=True)
    adj = oracle.build_graph(v, 16)
    eo = oracle.compute_entry_order(v)
    q = oracle.random_dataset(64, dim, 96)
    p = dvs.SearchParams(4, 16, 10, 16, metric=metric, accum="f32c")
    want = _search(ctx, v, adj, q, p, None, eo)
    ctx.set_shard_exchange(exchange)
    try:
        got = ctx.beam_search_sharded_emulated(3, q, p)
    finally:
        ctx.set_shard_exchange("bulk")
    _assert_same(got, want, True, f"f32c sharded {exchange} {metric}")


@pytest.mark.parametrize("dim", [300, 512, 640, 1024])
@pytest.mark.parametrize("accum", ["f64", "f32"])
def test_wide_rows_match_oracle(ctx, oracle, dim, accum):
    """Wide-row K1 (VPL 3-8: 4 or 2 rows in flight per warp at 2 CTAs/SM,
    FULL and padded rows) against the oracle.  f64 on float data: exact by
    construction (rounding-boundary guard); f32 on byte data: exact sums."""
    rng = np.random.default_rng(dim)
    n, nq = 3000, 200
    if accum == "f64":
        v = rng.normal(size=(n, dim)).astype(np.float32)
        q = rng.normal(size=(nq, dim)).astype(np.float32)
    else:
        v = rng.integers(0, 16, size=(n, dim)).astype(np.float32)  # partial sums stay below 2^24
        q = rng.integers(0, 16, size=(nq, dim)).astype(np.float32)
    adj = oracle.build_graph(v, 16)
    eo = oracle.compute_entry_order(v)
    gids = np.arange(n, dtype=np.uint32)
    want = oracle.beam_search(v, gids, adj, eo, q, 5, 48, 10, 48)
    got = _search(ctx, v, adj, q, dvs.SearchParams(5, 48, 10, 48, accum=accum), eo=eo)
    _assert_same(got, want, True, f"dim={dim} {accum}")


@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_wide_rows_f64_exact(ctx, oracle, nranks):
    """Node-sharded scorer on wide rows (768-d: 4 rows in flight per warp) in
    the f64 mode on float data: identical to K1 and to the oracle."""
    rng = np.random.default_rng(77 + nranks)
    n, nq, dim = 3000, 120, 768
    v = rng.normal(size=(n, dim)).astype(np.float32)
    q = rng.normal(size=(nq, dim)).astype(np.float32)
    adj = oracle.build_graph(v, 16)
    eo = oracle.compute_entry_order(v)
    p = dvs.SearchParams(5, 32, 10, 32, accum="f64")
    k1 = _search(ctx, v, adj, q, p, eo=eo)
    for mode in ("bulk", "fused"):
        ctx.set_shard_exchange(mode)
        got = ctx.beam_search_sharded_emulated(nranks, q, p)
        _assert_same(got, k1, True, f"sharded {mode} R={nranks}")
    ctx.set_shard_exchange("bulk")
    want = oracle.beam_search(v, np.arange(n, dtype=np.uint32), adj, eo, q, 5, 32, 10, 32)
    _assert_same(k1, want, True, "k1 vs oracle")


def test_brute_force_float_tiny_and_k_equals_n(ctx, ref):
    """Exact-mode brute force where every row is a candidate (n <= 32, k = n)
    and where k is the last valid size."""
    rng = np.random.default_rng(12)
    for n, k in ((5, 5), (32, 32), (33, 32), (40, 1)):
        v = rng.normal(size=(n, 9)).astype(np.float32)
        q = rng.normal(size=(7, 9)).astype(np.float32)
        wi, wd = ref.brute_force_topk(v, q, k)
        gi, gd = ctx.brute_force_topk(v, q, k)
        assert ctx.last_knn_info()[0] == 1
        assert np.array_equal(gi, wi) and np.array_equal(gd, wd), (n, k)
