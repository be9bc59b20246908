"""K5 on the tensor cores (route_kernels.cu "K5 on the tensor cores"):
TF32 tcgen05 candidates (K7, kind::tf32) + exact fp64 re-rank + per-query
certificate + exact fallback.  Bar: bit-identical to the reference's
assign_top_c (kmeans.cpp:243-280) -- the compiled reference (oracle/_ref)
and the plain-C oracle at test sizes, and the exact fp64 tile path
(prefix of a c > 24 assignment, which stays on that path) at 200k x 4096."""
import numpy as np
import pytest
import torch

import paper_2512_02278_b200 as dvs
from conftest import sift_like

pytestmark = pytest.mark.gpu


def _assign(ctx, cents, q, c):
    out = dvs.assign_top_c(cents, q, c, ctx=ctx)
    return out, ctx.last_assign_info()


@pytest.mark.parametrize("clusters,dim,c,kind", [
    (256, 8, 1, "uniform"), (1024, 128, 8, "sift"), (4096, 96, 10, "gauss"),
    (300, 37, 24, "uniform"), (777, 100, 3, "sift"), (2048, 64, 16, "offset")])
def test_tc_assign_matches_reference(ctx, oracle, ref, clusters, dim, c, kind):
    rng = np.random.default_rng(clusters + dim)
    nq = 3000
    if kind == "sift":
        x = sift_like(clusters + nq, dim, 16, clusters)
        cents, q = x[:clusters], x[clusters:]
    elif kind == "gauss":
        cents = rng.normal(size=(clusters, dim)).astype(np.float32)
        q = rng.normal(size=(nq, dim)).astype(np.float32)
    elif kind == "offset":  # far from the origin: the centring matters
        cents = (1e3 + rng.normal(size=(clusters, dim))).astype(np.float32)
        q = (1e3 + rng.normal(size=(nq, dim))).astype(np.float32)
    else:
        cents = oracle.random_dataset(clusters, dim, 7, -100, 100)
        q = oracle.random_dataset(nq, dim, 8, -100, 100)
    got, (path, fb) = _assign(ctx, cents, q, c)
    assert path == 2
    want = ref.assign_top_c(cents, q, c)
    assert np.array_equal(got, want), (np.argwhere(got != want)[:5], fb)
    assert np.array_equal(got, oracle.assign_top_c(cents, q, c))
    assert fb <= nq // 10, fb  # the certificate accepts the bulk of ordinary queries


def test_tc_assign_ties_and_fallback(ctx, ref):
    """Duplicated centroids (exact distance ties, broken by the lower id) and
    queries equidistant from 40 centroids (more near-ties than candidates:
    the certificate must reject them and the exact kernel must finish them)."""
    rng = np.random.default_rng(5)
    dim, clusters = 32, 512
    cents = rng.integers(-50, 50, size=(clusters, dim)).astype(np.float32)
    cents[100:110] = cents[3]
    # 40 centroids on a sphere around p: their squared distances to p agree
    # to float rounding, so 32 candidates cannot certify a top-24
    p = np.zeros(dim, np.float32)
    ring = rng.normal(size=(40, dim))
    ring = ring / np.linalg.norm(ring, axis=1, keepdims=True) * 10.0
    cents[200:240] = (p + ring).astype(np.float32)
    q = rng.integers(-50, 50, size=(500, dim)).astype(np.float32)
    q[0] = cents[3]
    q[1:20] = p
    for c in (1, 5, 24):
        got, (path, fb) = _assign(ctx, cents, q, c)
        assert path == 2
        assert np.array_equal(got, ref.assign_top_c(cents, q, c)), c
        if c == 24:
            assert fb >= 19, fb  # the 19 ring-centre queries went to the exact kernel


def test_tc_assign_matches_exact_tiles_at_scale(ctx):
    """200k queries x 4096 centroids x 96-d: the tensor-core top-8 equals the
    first 8 of the exact fp64 tile path's top-25 (c > 24 stays on the tiles;
    the reference's top-c is a prefix of its top-c' for c < c')."""
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(3)
    cents = torch.randn(4096, 96, device=dev, generator=g).cpu().numpy()
    q = torch.randn(200_000, 96, device=dev, generator=g).cpu().numpy()
    got, (path, fb) = _assign(ctx, cents, q, 8)
    assert path == 2
    full = dvs.assign_top_c(cents, q, 25, ctx=ctx)
    assert ctx.last_assign_info()[0] == 1
    assert np.array_equal(got, full[:, :8]), np.argwhere(got != full[:, :8])[:5]
    assert fb < 2000, fb


def test_tc_kmeans_and_partition_match_reference(ctx, ref):
    """kmeans_train / partition_database at C >= 256 run their nearest-centre
    passes through the tensor-core K5 and still reproduce the reference."""
    x = sift_like(20_000, 32, 8, 11)
    want, wit, wwcss = ref.kmeans_train_stats(x, 300, 3, 5)
    got, st = dvs.kmeans_train(x, 300, 3, 5, ctx=ctx, stats=True)
    assert np.array_equal(got, want)
    assert st.iterations == wit
    lab = np.full(x.shape[0], -1, np.int64)
    for ci, ids in enumerate(dvs.partition_database(x, got, ctx=ctx)):
        lab[ids] = ci
    assert np.array_equal(lab, ref.partition_labels(x, want).astype(np.int64))
