"""ctypes bindings of the TEST-ONLY checkers (see dvs_oracle.h).

  Oracle   -- liboracle.so, the plain-C restatement (always buildable)
  Ref      -- _ref/libdvsref.so, the reference's own sources compiled in place

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  ``ensure_built()`` compiles liboracle.so with gcc when it is
missing (e.g. on a fresh GPU box); _ref needs /root/reference and is built by
``make -C oracle`` in the build container only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_uint32, c_uint64, c_void_p
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdvsref.so")


def ensure_built() -> None:
    src = os.path.join(HERE, "dvs_oracle.c")
    if not os.path.isfile(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def _p(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class dvso_graph(ctypes.Structure):
    _fields_ = [("vectors", c_void_p), ("global_ids", c_void_p), ("adjacency", c_void_p),
                ("entry_order", c_void_p), ("n", c_uint64), ("dim", c_int), ("out_degree", c_int)]


class dvso_params(ctypes.Structure):
    _fields_ = [("iterations", c_int), ("beam_width", c_int), ("k", c_int),
                ("entry_count", c_int), ("metric", c_int)]


class dvso_index(ctypes.Structure):
    _fields_ = [("clusters", c_int), ("dim", c_int), ("out_degree", c_int),
                ("centroids", c_void_p), ("cluster_to_rank", c_void_p), ("ranks", c_int),
                ("graphs", POINTER(dvso_graph))]


class Oracle:
    """The C restatement."""

    def __init__(self):
        ensure_built()
        self.lib = ctypes.CDLL(ORACLE_SO)
        self.lib.dvso_last_error.restype = c_char_p
        self.lib.dvso_squared_l2.restype = c_float
        self.lib.dvso_squared_l2.argtypes = [c_void_p, c_void_p, c_int]
        self.lib.dvso_dot.restype = c_double
        self.lib.dvso_dot.argtypes = [c_void_p, c_void_p, c_int]
        self.lib.dvso_squared_l2_expanded.restype = c_float
        self.lib.dvso_squared_l2_expanded.argtypes = [c_void_p, c_void_p, c_int]
        self.lib.dvso_random_dataset.argtypes = [c_uint64, c_int, c_uint64, c_double, c_double, c_void_p]
        self.lib.dvso_gaussian_mixture.argtypes = [c_uint64, c_int, c_int, c_double, c_double,
                                                   c_uint64, c_void_p, c_void_p, c_void_p]
        self.lib.dvso_mixture_queries.argtypes = [c_void_p, c_int, c_int, c_uint64, c_double,
                                                  c_uint64, c_void_p]
        self.lib.dvso_compute_entry_order.argtypes = [c_void_p, c_uint64, c_int, c_void_p]
        self.lib.dvso_build_graph.argtypes = [c_void_p, c_uint64, c_int, c_int, c_void_p, c_int]
        self.lib.dvso_beam_search_batch.argtypes = [POINTER(dvso_graph), c_void_p, c_uint64,
                                                    POINTER(dvso_params), c_int, c_void_p,
                                                    c_void_p, c_void_p, c_void_p]
        self.lib.dvso_combine_results.argtypes = [c_int, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                                  c_void_p, c_void_p, c_void_p]
        self.lib.dvso_assign_top_c.argtypes = [c_void_p, c_int, c_int, c_void_p, c_uint64, c_int, c_void_p]
        self.lib.dvso_partition_database.argtypes = [c_void_p, c_uint64, c_int, c_void_p, c_int, c_void_p]
        self.lib.dvso_brute_force_topk_batch.argtypes = [c_void_p, c_uint64, c_int, c_void_p, c_uint64,
                                                         c_int, c_int, c_void_p, c_void_p]
        self.lib.dvso_run_pipeline.argtypes = [POINTER(dvso_index), c_void_p, c_uint64,
                                               POINTER(dvso_params), c_int, c_int, c_int, c_int,
                                               c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, self.lib.dvso_last_error().decode())

    # synthetic.hpp
    def random_dataset(self, n, dim, seed, lo=-1.0, hi=1.0) -> np.ndarray:
        out = np.zeros((n, dim), np.float32)
        self.lib.dvso_random_dataset(n, dim, seed, lo, hi, _p(out))
        return out

    def gaussian_mixture(self, n, dim, components, mean_scale, stddev, seed):
        means = np.zeros((components, dim), np.float32)
        pts = np.zeros((n, dim), np.float32)
        labels = np.zeros(n, np.int32)
        self.lib.dvso_gaussian_mixture(n, dim, components, mean_scale, stddev, seed, _p(means),
                                       _p(pts), _p(labels))
        return means, pts, labels

    def mixture_queries(self, means, n, stddev, seed) -> np.ndarray:
        means = np.ascontiguousarray(means, np.float32)
        out = np.zeros((n, means.shape[1]), np.float32)
        self.lib.dvso_mixture_queries(_p(means), means.shape[0], means.shape[1], n, stddev, seed, _p(out))
        return out

    def squared_l2(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.dvso_squared_l2(_p(a), _p(b), a.shape[0])

    def compute_entry_order(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros(v.shape[0], np.uint32)
        self._check(self.lib.dvso_compute_entry_order(_p(v), v.shape[0], v.shape[1], _p(out)))
        return out

    def build_graph(self, v, out_degree, nthreads=8) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float32)
        adj = np.zeros((v.shape[0], out_degree), np.uint32)
        self._check(self.lib.dvso_build_graph(_p(v), v.shape[0], v.shape[1], out_degree, _p(adj), nthreads))
        return adj

    @staticmethod
    def _graph(vectors, gids, adjacency, entry_order):
        keep = [np.ascontiguousarray(vectors, np.float32), np.ascontiguousarray(gids, np.uint32),
                np.ascontiguousarray(adjacency, np.uint32), np.ascontiguousarray(entry_order, np.uint32)]
        g = dvso_graph(keep[0].ctypes.data, keep[1].ctypes.data, keep[2].ctypes.data,
                       keep[3].ctypes.data, keep[0].shape[0], keep[0].shape[1],
                       int(keep[2].size // max(keep[0].shape[0], 1)))
        return g, keep

    def beam_search(self, vectors, gids, adjacency, entry_order, queries, iterations, beam_width,
                    k, entry_count, metric=0, nthreads=8):
        g, keep = self._graph(vectors, gids, adjacency, entry_order)
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, keep[0].shape[1])
        nq = q.shape[0]
        p = dvso_params(iterations, beam_width, k, entry_count, metric)
        ids = np.zeros((nq, max(k, 1)), np.uint32)
        dists = np.zeros((nq, max(k, 1)), np.float32)
        counts = np.zeros(nq, np.uint32)
        vis = np.zeros(nq, np.uint64)
        self._check(self.lib.dvso_beam_search_batch(ctypes.byref(g), _p(q), nq, ctypes.byref(p),
                                                    nthreads, _p(ids), _p(dists), _p(counts), _p(vis)))
        return ids, dists, counts, vis

    def combine_results(self, ids, dists, counts, k):
        """one query: ids/dists nparts x stride, counts nparts"""
        ids = np.ascontiguousarray(ids, np.uint32)
        dists = np.ascontiguousarray(dists, np.float32)
        counts = np.ascontiguousarray(counts, np.uint32)
        oi = np.zeros(max(k, 1), np.uint32)
        od = np.zeros(max(k, 1), np.float32)
        oc = c_uint32(0)
        self._check(self.lib.dvso_combine_results(ids.shape[0], _p(ids), _p(dists), _p(counts),
                                                  ids.shape[1], k, _p(oi), _p(od), ctypes.byref(oc)))
        return oi[:oc.value], od[:oc.value]

    def assign_top_c(self, cents, queries, c):
        cents = np.ascontiguousarray(cents, np.float32)
        q = np.ascontiguousarray(queries, np.float32)
        out = np.zeros((q.shape[0], c), np.uint32)
        self._check(self.lib.dvso_assign_top_c(_p(cents), cents.shape[0], cents.shape[1], _p(q),
                                               q.shape[0], c, _p(out)))
        return out

    def partition_database(self, db, cents):
        db = np.ascontiguousarray(db, np.float32)
        cents = np.ascontiguousarray(cents, np.float32)
        out = np.zeros(db.shape[0], np.uint32)
        self._check(self.lib.dvso_partition_database(_p(db), db.shape[0], db.shape[1], _p(cents),
                                                      cents.shape[0], _p(out)))
        return out

    def brute_force_topk(self, db, queries, k, nthreads=8):
        db = np.ascontiguousarray(db, np.float32)
        q = np.ascontiguousarray(queries, np.float32)
        ids = np.zeros((q.shape[0], k), np.uint32)
        d = np.zeros((q.shape[0], k), np.float32)
        self._check(self.lib.dvso_brute_force_topk_batch(_p(db), db.shape[0], db.shape[1], _p(q),
                                                         q.shape[0], k, nthreads, _p(ids), _p(d)))
        return ids, d

    def run_pipeline(self, index, queries, iterations, beam_width, k, entry_count, fanout, ranks,
                     batch_index=0, metric=0, nthreads=8, with_vectors=True):
        """index: api.BuiltIndex-like (centroids, cluster_to_rank, ranks, out_degree, graphs)."""
        keeps = []
        graphs = (dvso_graph * len(index.graphs))()
        for i, g in enumerate(index.graphs):
            eo = g.entry_order if g.entry_order is not None else self.compute_entry_order(g.vectors)
            gg, keep = self._graph(g.vectors, g.global_ids, g.adjacency, eo)
            graphs[i] = gg
            keeps.append(keep)
        cents = np.ascontiguousarray(index.centroids, np.float32)
        ctr = np.ascontiguousarray(index.cluster_to_rank, np.uint32)
        idx = dvso_index(cents.shape[0], cents.shape[1], int(index.out_degree), cents.ctypes.data,
                         ctr.ctypes.data, int(index.ranks), graphs)
        q = np.ascontiguousarray(queries, np.float32)
        nq, dim = q.shape
        p = dvso_params(iterations, beam_width, k, entry_count, metric)
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float32)
        counts = np.zeros(nq, np.uint32)
        vecs = np.zeros((nq, k, dim), np.float32) if with_vectors else None
        vt = c_uint64(0)
        self._check(self.lib.dvso_run_pipeline(ctypes.byref(idx), _p(q), nq, ctypes.byref(p), fanout,
                                               ranks, batch_index, nthreads, _p(ids), _p(dists),
                                               _p(counts), _p(vecs), ctypes.byref(vt)))
        return ids, dists, counts, vecs, int(vt.value)


class Ref:
    """The reference's own C++ (unmodified sources) via oracle/ref_capi.cpp."""

    def __init__(self):
        if not os.path.isfile(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = ctypes.CDLL(REF_SO)
        self.lib = L
        L.dvsref_last_error.restype = c_char_p
        L.dvsref_build_graph.restype = c_void_p
        L.dvsref_build_graph.argtypes = [c_void_p, c_uint64, c_int, c_void_p, c_int]
        L.dvsref_graph_from_arrays.restype = c_void_p
        L.dvsref_graph_from_arrays.argtypes = [c_void_p, c_uint64, c_int, c_void_p, c_int, c_void_p]
        L.dvsref_graph_free.argtypes = [c_void_p]
        L.dvsref_graph_size.restype = c_uint64
        L.dvsref_graph_size.argtypes = [c_void_p]
        L.dvsref_graph_arrays.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p]
        L.dvsref_compute_entry_order.argtypes = [c_void_p, c_uint64, c_int, c_void_p]
        L.dvsref_beam_search.argtypes = [c_void_p, c_void_p, c_uint64, c_int, c_int, c_int, c_int,
                                         c_int, c_void_p, c_void_p, c_void_p, c_void_p]
        L.dvsref_check_timeline.argtypes = [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_void_p, c_char_p, c_int]
        L.dvsref_combine_results.argtypes = [c_int, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                             c_void_p, c_void_p, c_void_p]
        L.dvsref_assign_top_c.argtypes = [c_void_p, c_int, c_int, c_void_p, c_uint64, c_int, c_void_p]
        L.dvsref_brute_force_topk.argtypes = [c_void_p, c_uint64, c_int, c_void_p, c_uint64, c_int,
                                              c_int, c_void_p, c_void_p]
        L.dvsref_kmeans_train.argtypes = [c_void_p, c_uint64, c_int, c_int, c_int, c_uint64, c_void_p]
        L.dvsref_build_index.restype = c_void_p
        L.dvsref_build_index.argtypes = [c_void_p, c_uint64, c_int, c_int, c_int, c_int, c_int, c_int,
                                         c_uint64]
        L.dvsref_index_from_arrays.restype = c_void_p
        L.dvsref_index_from_arrays.argtypes = [c_int, c_int, c_int, c_void_p, c_void_p, c_int,
                                               c_void_p, c_void_p, c_void_p, c_void_p]
        L.dvsref_index_free.argtypes = [c_void_p]
        L.dvsref_index_save.argtypes = [c_void_p, c_char_p]
        L.dvsref_index_load.restype = c_void_p
        L.dvsref_index_load.argtypes = [c_char_p]
        L.dvsref_index_info.argtypes = [c_void_p, POINTER(c_int), POINTER(c_int), POINTER(c_int),
                                        POINTER(c_int), c_void_p]
        L.dvsref_index_dump.argtypes = [c_void_p] + [c_void_p] * 6
        L.dvsref_run_pipeline.argtypes = [c_void_p, c_void_p, c_uint64, c_int, c_int, c_int, c_int,
                                          c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                                          c_void_p, c_void_p, c_void_p]

    def err(self):
        return self.lib.dvsref_last_error().decode()

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.err())

    def build_graph(self, v, out_degree, gids=None):
        v = np.ascontiguousarray(v, np.float32)
        g = None if gids is None else np.ascontiguousarray(gids, np.uint32)
        h = self.lib.dvsref_build_graph(_p(v), v.shape[0], v.shape[1], _p(g), out_degree)
        if not h:
            raise OracleError(2, self.err())
        n = v.shape[0]
        adj = np.zeros((n, out_degree), np.uint32)
        eo = np.zeros(n, np.uint32)
        self.lib.dvsref_graph_arrays(h, _p(adj), _p(eo), None)
        return RefGraph(self, h, v.shape[1]), adj, eo

    def check_timeline(self, intervals):
        """simulator.cpp:170-217 on intervals with the reference's lane /
        stage names -> None or the reference's message."""
        lanes = {"compute": 0, "comm": 1}
        stages = {"kmeans": 0, "dispatch": 1, "search": 2, "combine": 3}
        n = len(intervals)
        cols = [np.array([f(iv) for iv in intervals], dt) for f, dt in (
            (lambda iv: iv["rank"], np.int32), (lambda iv: lanes[iv["lane"]], np.int32),
            (lambda iv: stages[iv["stage"]], np.int32), (lambda iv: iv["microbatch"], np.int32),
            (lambda iv: iv["start"], np.float64), (lambda iv: iv["end"], np.float64))]
        msg = ctypes.create_string_buffer(512)
        r = self.lib.dvsref_check_timeline(n, *[_p(c) for c in cols], msg, 512)
        return None if r == 0 else msg.value.decode()

    def graph_from_arrays(self, v, gids, adjacency):
        v = np.ascontiguousarray(v, np.float32)
        gids = np.ascontiguousarray(gids, np.uint32)
        adj = np.ascontiguousarray(adjacency, np.uint32)
        h = self.lib.dvsref_graph_from_arrays(_p(v), v.shape[0], v.shape[1], _p(gids),
                                              adj.size // v.shape[0], _p(adj))
        if not h:
            raise OracleError(2, self.err())
        return RefGraph(self, h, v.shape[1])

    def compute_entry_order(self, v):
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros(v.shape[0], np.uint32)
        self._check(self.lib.dvsref_compute_entry_order(_p(v), v.shape[0], v.shape[1], _p(out)))
        return out

    def combine_results(self, ids, dists, counts, k):
        ids = np.ascontiguousarray(ids, np.uint32)
        dists = np.ascontiguousarray(dists, np.float32)
        counts = np.ascontiguousarray(counts, np.uint32)
        oi = np.zeros(max(k, 1), np.uint32)
        od = np.zeros(max(k, 1), np.float32)
        oc = c_uint32(0)
        self._check(self.lib.dvsref_combine_results(ids.shape[0], _p(ids), _p(dists), _p(counts),
                                                    ids.shape[1], k, _p(oi), _p(od), ctypes.byref(oc)))
        return oi[:oc.value], od[:oc.value]

    def assign_top_c(self, cents, queries, c):
        cents = np.ascontiguousarray(cents, np.float32)
        q = np.ascontiguousarray(queries, np.float32)
        out = np.zeros((q.shape[0], c), np.uint32)
        self._check(self.lib.dvsref_assign_top_c(_p(cents), cents.shape[0], cents.shape[1], _p(q),
                                                 q.shape[0], c, _p(out)))
        return out

    def brute_force_topk(self, db, queries, k, nthreads=8):
        db = np.ascontiguousarray(db, np.float32)
        q = np.ascontiguousarray(queries, np.float32)
        ids = np.zeros((q.shape[0], k), np.uint32)
        d = np.zeros((q.shape[0], k), np.float32)
        self._check(self.lib.dvsref_brute_force_topk(_p(db), db.shape[0], db.shape[1], _p(q),
                                                     q.shape[0], k, nthreads, _p(ids), _p(d)))
        return ids, d

    def kmeans_train(self, db, clusters, max_iters, seed):
        db = np.ascontiguousarray(db, np.float32)
        out = np.zeros((clusters, db.shape[1]), np.float32)
        self._check(self.lib.dvsref_kmeans_train(_p(db), db.shape[0], db.shape[1], clusters,
                                                 max_iters, seed, _p(out)))
        return out

    def kmeans_train_stats(self, db, clusters, max_iters, seed):
        """-> (centroids, iterations, wcss per iteration) -- KmeansStats (kmeans.hpp:27-30)."""
        db = np.ascontiguousarray(db, np.float32)
        out = np.zeros((clusters, db.shape[1]), np.float32)
        it = c_int(0)
        wcss = np.zeros(max(max_iters, 1), np.float64)
        self.lib.dvsref_kmeans_train_stats.argtypes = [c_void_p, c_uint64, c_int, c_int, c_int, c_uint64,
                                                        c_void_p, POINTER(c_int), c_void_p]
        self._check(self.lib.dvsref_kmeans_train_stats(_p(db), db.shape[0], db.shape[1], clusters, max_iters,
                                                       seed, _p(out), ctypes.byref(it), _p(wcss)))
        return out, it.value, wcss[:it.value]

    def partition_labels(self, db, cents):
        """partition_database (kmeans.cpp:282-300) as a label per row."""
        db = np.ascontiguousarray(db, np.float32)
        cents = np.ascontiguousarray(cents, np.float32)
        lab = np.zeros(db.shape[0], np.uint32)
        self.lib.dvsref_partition_database.argtypes = [c_void_p, c_uint64, c_int, c_void_p, c_int, c_void_p]
        self._check(self.lib.dvsref_partition_database(_p(db), db.shape[0], db.shape[1], _p(cents),
                                                       cents.shape[0], _p(lab)))
        return lab

    def build_index(self, db, clusters, out_degree, ranks, ranks_per_node, kmeans_iters, seed):
        db = np.ascontiguousarray(db, np.float32)
        h = self.lib.dvsref_build_index(_p(db), db.shape[0], db.shape[1], clusters, out_degree,
                                        ranks, ranks_per_node, kmeans_iters, seed)
        if not h:
            raise OracleError(2, self.err())
        return RefIndex(self, h)

    def index_from_arrays(self, centroids, cluster_to_rank, ranks, out_degree, graphs):
        """graphs: list of (vectors, adjacency, gids)."""
        cents = np.ascontiguousarray(centroids, np.float32)
        ctr = np.ascontiguousarray(cluster_to_rank, np.uint32)
        sizes = [g[0].shape[0] for g in graphs]
        offs = np.zeros(len(graphs) + 1, np.uint64)
        offs[1:] = np.cumsum(sizes)
        def cat(parts, dt):  # no concatenated copy of a single (possibly 50 GB) graph
            return np.ascontiguousarray(parts[0] if len(parts) == 1 else np.concatenate(parts), dt)
        vec = cat([g[0] for g in graphs], np.float32)
        adj = cat([np.asarray(g[1]).reshape(-1) for g in graphs], np.uint32)
        gids = cat([g[2] for g in graphs], np.uint32)
        h = self.lib.dvsref_index_from_arrays(cents.shape[0], cents.shape[1], out_degree, _p(cents),
                                              _p(ctr), ranks, _p(offs), _p(vec), _p(adj), _p(gids))
        if not h:
            raise OracleError(2, self.err())
        return RefIndex(self, h)

    def load_index(self, path):
        h = self.lib.dvsref_index_load(str(path).encode())
        if not h:
            raise OracleError(3, self.err())
        return RefIndex(self, h)


class RefGraph:
    def __init__(self, ref: Ref, h, dim):
        self.ref, self.h, self.dim = ref, h, dim

    def __del__(self):
        try:
            self.ref.lib.dvsref_graph_free(self.h)
        except Exception:
            pass

    def beam_search(self, queries, iterations, beam_width, k, entry_count, nthreads=8):
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        nq = q.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float32)
        counts = np.zeros(nq, np.uint32)
        vis = np.zeros(nq, np.uint64)
        self.ref._check(self.ref.lib.dvsref_beam_search(self.h, _p(q), nq, iterations, beam_width, k,
                                                        entry_count, nthreads, _p(ids), _p(dists),
                                                        _p(counts), _p(vis)))
        return ids, dists, counts, vis


class RefIndex:
    def __init__(self, ref: Ref, h):
        self.ref, self.h = ref, h

    def __del__(self):
        try:
            self.ref.lib.dvsref_index_free(self.h)
        except Exception:
            pass

    def info(self):
        c, d, dg, r = c_int(), c_int(), c_int(), c_int()
        self.ref.lib.dvsref_index_info(self.h, ctypes.byref(c), ctypes.byref(d), ctypes.byref(dg),
                                       ctypes.byref(r), None)
        sizes = np.zeros(c.value, np.uint64)
        self.ref.lib.dvsref_index_info(self.h, ctypes.byref(c), ctypes.byref(d), ctypes.byref(dg),
                                       ctypes.byref(r), _p(sizes))
        return c.value, d.value, dg.value, r.value, sizes

    def dump(self):
        """-> dict(centroids, cluster_to_rank, ranks, out_degree, graphs=[(vec, adj, gids, entry)])"""
        C, d, dg, r, sizes = self.info()
        total = int(sizes.sum())
        cents = np.zeros((C, d), np.float32)
        plc = np.zeros(C, np.uint32)
        vec = np.zeros((total, d), np.float32)
        adj = np.zeros((total, dg), np.uint32)
        gids = np.zeros(total, np.uint32)
        eo = np.zeros(total, np.uint32)
        self.ref.lib.dvsref_index_dump(self.h, _p(cents), _p(plc), _p(vec), _p(adj), _p(gids), _p(eo))
        graphs = []
        off = 0
        for s in sizes.astype(np.int64):
            graphs.append((vec[off:off + s], adj[off:off + s], gids[off:off + s], eo[off:off + s]))
            off += s
        return dict(centroids=cents, cluster_to_rank=plc, ranks=r, out_degree=dg, graphs=graphs)

    def save(self, path):
        self.ref._check(self.ref.lib.dvsref_index_save(self.h, str(path).encode()))

    def run_pipeline(self, queries, iterations, beam_width, k, entry_count, fanout, ranks,
                     ranks_per_node=None, batch_index=0, nthreads=8, with_vectors=True):
        q = np.ascontiguousarray(queries, np.float32)
        nq, dim = q.shape
        rpn = ranks_per_node or ranks
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float32)
        counts = np.zeros(nq, np.uint32)
        vecs = np.zeros((nq, k, dim), np.float32) if with_vectors else None
        vt = c_uint64(0)
        self.ref._check(self.ref.lib.dvsref_run_pipeline(self.h, _p(q), nq, iterations, beam_width, k,
                                                         entry_count, fanout, ranks, rpn, batch_index,
                                                         nthreads, _p(ids), _p(dists), _p(counts),
                                                         _p(vecs), ctypes.byref(vt)))
        return ids, dists, counts, vecs, int(vt.value)


def have_ref() -> bool:
    return os.path.isfile(REF_SO)
