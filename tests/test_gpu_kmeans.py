"""GPU kmeans_train / partition_database / build_index (kmeans.cpp:189-300,
index.cpp:43-72) against the reference's own C++ (oracle/_ref): centroids,
iteration counts and WCSS bit-identical on integer-valued data, identical
labels, identical BuiltIndex arrays, the same errors."""
import numpy as np
import pytest

import paper_2512_02278_b200 as dvs
from conftest import sift_like

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,dim,clusters,iters,seed", [(3000, 16, 24, 10, 42), (5000, 32, 64, 25, 7),
                                                       (800, 8, 100, 5, 3)])
def test_kmeans_train_matches_reference(ctx, ref, n, dim, clusters, iters, seed):
    x = sift_like(n, dim, 6, seed)
    want, wit, wwcss = ref.kmeans_train_stats(x, clusters, iters, seed)
    got, st = dvs.kmeans_train(x, clusters, iters, seed, ctx=ctx, stats=True)
    assert st.iterations == wit
    assert np.array_equal(got, want)
    assert np.array_equal(st.wcss, wwcss)


def test_kmeans_train_float_data(ctx, ref):
    rng = np.random.default_rng(5)
    x = (rng.normal(size=(4000, 24)) * 3.7).astype(np.float32)
    want, wit, _ = ref.kmeans_train_stats(x, 32, 15, 11)
    got, st = dvs.kmeans_train(x, 32, 15, 11, ctx=ctx, stats=True)
    assert st.iterations == wit
    np.testing.assert_array_equal(got, want)  # observed bit-identical (see kmeans.cu header)


def test_kmeans_train_repairs_and_errors(ctx, ref):
    # many duplicates: k-means++ runs out of mass and empty clusters get repaired
    base = sift_like(12, 8, 4, 2)
    x = np.repeat(base, 30, axis=0)
    want = ref.kmeans_train(x, 12, 8, 9)
    assert np.array_equal(dvs.kmeans_train(x, 12, 8, 9, ctx=ctx), want)
    # fewer distinct points than clusters: both refuse
    with pytest.raises(Exception):
        ref.kmeans_train(x[:60], 13, 8, 9)
    with pytest.raises(dvs.InvalidArgument):
        dvs.kmeans_train(x[:60], 13, 8, 9, ctx=ctx)
    with pytest.raises(dvs.InvalidArgument):
        dvs.kmeans_train(x, 0, 8, 9, ctx=ctx)
    with pytest.raises(dvs.InvalidArgument):
        dvs.kmeans_train(x, 4, 0, 9, ctx=ctx)


def test_partition_database_matches_reference(ctx, ref):
    x = sift_like(6000, 24, 8, 13)
    cents = ref.kmeans_train(x, 40, 10, 42)
    want = ref.partition_labels(x, cents)
    parts = dvs.partition_database(x, cents, ctx=ctx)
    got = np.zeros(x.shape[0], np.uint32)
    for c, ids in enumerate(parts):
        assert (np.diff(ids.astype(np.int64)) > 0).all()  # row order inside a cluster
        got[ids] = c
    assert np.array_equal(got, want)


def test_build_index_matches_reference(ctx, ref):
    x = sift_like(4000, 16, 6, 17)
    want = ref.build_index(x, 8, 16, 2, 2, 12, 42).dump()
    got = dvs.build_index(x, 8, 16, ranks=2, kmeans_iters=12, seed=42, ctx=ctx)
    assert np.array_equal(got.centroids, want["centroids"])
    assert np.array_equal(got.cluster_to_rank, want["cluster_to_rank"])
    for g, (vec, adj, gids, eo) in zip(got.graphs, want["graphs"]):
        assert np.array_equal(g.global_ids, gids)
        assert np.array_equal(g.vectors, vec)
        assert np.array_equal(np.asarray(g.adjacency).reshape(adj.shape), adj)
        assert np.array_equal(g.entry_order, eo)
