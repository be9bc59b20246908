"""The device-initiated cluster exchange (cluster_xchg.cu, SURVEY 8e design A)
against the one-GPU run_pipeline (simulator.cpp:250-337): two rank contexts
on one device, each with its own partitions and arena, driven by two host
threads exactly as two processes would drive two GPUs.  Ids, dists, counts,
hit vectors and visited_total must be identical."""
import threading

import numpy as np
import pytest

import paper_2512_02278_b200 as dvs
from conftest import sift_like

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _run_ranks(ctxs, batches, p, fanout, steps=2):
    out = [None] * len(ctxs)
    errs = []

    def work(r):
        try:
            q = torch.from_numpy(batches[r]).cuda()
            from paper_2512_02278_b200.dist import run_pipeline_cluster
            for _ in range(steps):  # both cursor parities
                res = run_pipeline_cluster(ctxs[r], q, p, fanout)
                ctxs[r].synchronize()
                ctxs[r].cluster_comm_check()
            out[r] = [t.cpu().numpy() for t in res]
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(len(ctxs))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    return out


@pytest.mark.parametrize("ranks,clusters,fanout", [(1, 4, 2), (2, 6, 3), (3, 7, 2)])
def test_cluster_exchange_equals_run_pipeline(ctx, ranks, clusters, fanout):
    x = sift_like(6000, 24, 6, 31)
    q = sift_like(600, 24, 6, 32)
    p = dvs.SearchParams(6, 24, 10, 24, accum="f32")
    idx = dvs.build_index(x, clusters, 16, ranks=ranks, kmeans_iters=10, seed=42, ctx=ctx)
    want = dvs.run_pipeline(idx, q, p, fanout, ranks, ctx=ctx)
    ctxs = [dvs.Context(0) for _ in range(ranks)]
    for r, c in enumerate(ctxs):
        c.load_index(idx, rank=r)
        c.cluster_comm_init(ranks, r, 600, fanout, 10, True)
    arenas = [c.cluster_comm_arena() for c in ctxs]
    for c in ctxs:
        c.cluster_comm_connect_local(arenas)
    cuts = np.linspace(0, len(q), ranks + 1).astype(int)
    batches = [np.ascontiguousarray(q[cuts[r]:cuts[r + 1]]) for r in range(ranks)]
    got = _run_ranks(ctxs, batches, p, fanout)
    ids = np.concatenate([g[0] for g in got]).view(np.uint32)
    dists = np.concatenate([g[1] for g in got])
    counts = np.concatenate([g[2] for g in got]).view(np.uint32)
    vecs = np.concatenate([g[3] for g in got])
    assert np.array_equal(counts, want.counts)
    for i in range(len(q)):
        n = int(counts[i])
        assert np.array_equal(ids[i, :n], want.ids[i, :n]), i
        assert np.array_equal(dists[i, :n], want.dists[i, :n]), i
        assert np.array_equal(vecs[i, :n], want.hit_vectors[i, :n]), i
    assert sum(int(g[4][0]) for g in got) == want.visited_total
    for c in ctxs:
        c.close()


def test_cluster_exchange_capacity_error(ctx):
    x = sift_like(2000, 16, 6, 33)
    idx = dvs.build_index(x, 2, 8, ranks=1, kmeans_iters=5, seed=1, ctx=ctx)
    c = dvs.Context(0)
    c.load_index(idx, rank=0)
    c.cluster_comm_init(1, 0, 10, 1, 10, False)
    c.cluster_comm_connect_local([c.cluster_comm_arena()])
    q = torch.from_numpy(sift_like(20, 16, 6, 34)).cuda()
    from paper_2512_02278_b200.dist import run_pipeline_cluster
    with pytest.raises(dvs.InvalidArgument):  # 20 queries > max_queries 10
        run_pipeline_cluster(c, q, dvs.SearchParams(4, 8, 10, 8), 1, with_vectors=False)
    c.close()
