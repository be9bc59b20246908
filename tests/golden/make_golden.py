"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs only in the build container, where /root/reference exists and
`make -C oracle` has compiled the reference's own sources into
oracle/_ref/libdvsref.so.  Every array stored here was produced by the
reference's code path (build_graph, compute_entry_order, beam_search_stats,
kmeans_train/build_index, save_index, run_pipeline, assign_top_c,
brute_force_topk, combine_results); the inputs come from the reference's
seeded generators (tests/support/synthetic.hpp) as restated in
oracle/dvs_oracle.c.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle, Ref  # noqa: E402

PARAMS = [(6, 64, 10, 64), (6, 6, 10, 6), (4, 16, 25, 8), (2, 3, 50, 1), (8, 12, 5, 200)]


def sift_like(n, dim, rank, seed):
    """Integer-valued low-rank data in [0, 255] (SURVEY 8d "SIFT-like")."""
    rng = np.random.default_rng(seed)
    a = rng.normal(0.0, 1.0 / np.sqrt(rank), size=(rank, dim))
    z = rng.normal(size=(n, rank))
    x = z @ a + 0.1 * rng.normal(size=(n, dim))
    return np.clip(np.rint(x * 40.0 + 128.0), 0, 255).astype(np.float32)


def main():
    o, r = Oracle(), Ref()

    # --- G1: uniform random partition with non-dense global ids --------------
    v = o.random_dataset(2000, 16, 101)
    gids = (1000 + 3 * np.arange(2000)).astype(np.uint32)
    g, adj, eo = r.build_graph(v, 32, gids)
    q = o.random_dataset(200, 16, 102)
    out = dict(vectors=v, gids=gids, adjacency=adj, entry_order=eo, queries=q,
               params=np.array(PARAMS, np.int32))
    for i, (I, w, k, E) in enumerate(PARAMS):
        ids, d, c, vis = g.beam_search(q, I, w, k, E)
        out[f"ids{i}"], out[f"dists{i}"], out[f"counts{i}"], out[f"visited{i}"] = ids, d, c, vis
    np.savez_compressed(os.path.join(HERE, "g1_uniform.npz"), **out)

    # --- G2: SIFT-like integer data, d=32 ------------------------------------
    v = sift_like(3000, 32, 8, 201)
    g, adj, eo = r.build_graph(v, 32)
    q = sift_like(200, 32, 8, 202)
    out = dict(vectors=v, adjacency=adj, entry_order=eo, queries=q,
               params=np.array(PARAMS[:3], np.int32))
    for i, (I, w, k, E) in enumerate(PARAMS[:3]):
        ids, d, c, vis = g.beam_search(q, I, w, k, E)
        out[f"ids{i}"], out[f"dists{i}"], out[f"counts{i}"], out[f"visited{i}"] = ids, d, c, vis
    tid, td = r.brute_force_topk(v, q, 10)
    out["truth_ids"], out["truth_dists"] = tid, td
    np.savez_compressed(os.path.join(HERE, "g2_siftlike.npz"), **out)

    # --- G3: mixture, reference build_index (kmeans C=8, 4 ranks) + FNSY ------
    means, pts, _ = o.gaussian_mixture(3000, 24, 16, 3.0, 1.0, 7)
    qs = o.mixture_queries(means, 200, 1.0, 8)
    idx = r.build_index(pts, 8, 16, 4, 4, 10, 42)
    fnsy = os.path.join(HERE, "g3_mixture.fnsy")
    idx.save(fnsy)
    res = {}
    for fo in (1, 2, 3):
        ids, d, c, vecs, vt = idx.run_pipeline(qs, 6, 16, 10, 16, fo, 4, 4, batch_index=1)
        res[f"ids_f{fo}"], res[f"dists_f{fo}"], res[f"counts_f{fo}"] = ids, d, c
        res[f"vectors_f{fo}"], res[f"visited_f{fo}"] = vecs, np.uint64(vt)
    dump = idx.dump()
    res["assign3"] = r.assign_top_c(dump["centroids"], qs, 3)
    res["entry_orders"] = np.concatenate([gr[3] for gr in dump["graphs"]])
    np.savez_compressed(os.path.join(HERE, "g3_mixture.npz"), queries=qs, **res)

    # --- G4: combine_results KATs from the reference --------------------------
    rng = np.random.default_rng(5)
    cases = []
    for t in range(40):
        nparts = int(rng.integers(1, 5))
        stride = int(rng.integers(1, 12))
        k = int(rng.integers(1, 15))
        ids = rng.integers(0, 30, size=(nparts, stride)).astype(np.uint32)
        dists = np.round(rng.random((nparts, stride)) * 4, 1).astype(np.float32)
        counts = rng.integers(0, stride + 1, size=nparts).astype(np.uint32)
        for j in range(nparts):  # sort each partial by (dist, id)
            n = counts[j]
            order = np.lexsort((ids[j, :n], dists[j, :n]))
            ids[j, :n], dists[j, :n] = ids[j, :n][order], dists[j, :n][order]
        oi, od = r.combine_results(ids, dists, counts, k)
        cases.append((ids, dists, counts, k, oi, od))
    np.savez_compressed(os.path.join(HERE, "g4_combine.npz"),
                        **{f"c{i}_{n}": x for i, cs in enumerate(cases)
                           for n, x in zip(("ids", "dists", "counts", "k", "oi", "od"), cs)},
                        ncases=np.int32(len(cases)))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
