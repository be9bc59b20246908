"""Host-side mirror of the reference's search API over the C-ABI (include/dvsg.h).

Names, argument meaning and error behaviour follow
/root/reference/proj/include/dvs/*.hpp so that callers (and the parity tests)
read like the reference's own code:

  SearchParams            graph_index.hpp:27-32
  GraphIndex              graph_index.hpp:13-25
  SearchResult            graph_index.hpp:47-50
  beam_search_stats       graph_index.hpp:58-59     (batched: beam_search_batch)
  beam_search             graph_index.hpp:61-62
  visited_count           graph_index.hpp:64-65
  compute_entry_order     graph_index.hpp:45
  build_graph             graph_index.hpp:40-42
  combine_results         simulator.hpp:66-67
  assign_top_c            kmeans.hpp:41
  place_clusters / route  router.hpp:53-57
  BuiltIndex / run_pipeline (functional part)  index.hpp:14-23, simulator.hpp:98-102
  load_index / save_index index_file.hpp:13-14

std::invalid_argument -> InvalidArgument (a ValueError), format_error ->
FormatError, internal_error / CUDA failures -> InternalError.

Every compute call runs on the GPU through libdvsg.so; numpy only holds host
buffers.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import (ACCUM_F32, ACCUM_F32C, ACCUM_F64, METRIC_IP, METRIC_L2, FormatError, InternalError,
                   InvalidArgument, check, lib)

__all__ = [
    "SearchParams", "GraphIndex", "SearchResult", "ScoredId", "BuiltIndex", "PipelineResult",
    "Context", "default_context", "beam_search_stats", "beam_search", "visited_count",
    "beam_search_batch", "compute_entry_order", "build_graph", "combine_results",
    "assign_top_c", "place_clusters", "route", "run_pipeline", "load_index", "save_index",
    "check_timeline", "InvalidArgument", "FormatError", "InternalError", "kmeans_train",
    "partition_database", "build_index", "KmeansStats",
]


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _f32(a, ndim=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    if ndim is not None and a.ndim != ndim:
        raise InvalidArgument(f"expected a {ndim}-d float array, got shape {a.shape}")
    return a


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


@dataclass
class SearchParams:
    """graph_index.hpp:27-32 (+ metric / accumulation of the B200 kernel)."""

    iterations: int = 6
    beam_width: int = 6
    k: int = 10
    entry_count: int = 6
    metric: str = "l2"   # "l2" (squared_l2) | "ip" (-dot; parity unpinned)
    accum: str = "f64"   # "f64" parity mode | "f32" fast mode | "f32c" compensated f32

    def to_c(self) -> _lib.dvsg_search_params:
        metric = {"l2": METRIC_L2, "ip": METRIC_IP}.get(self.metric)
        accum = {"f64": ACCUM_F64, "f32": ACCUM_F32, "f32c": ACCUM_F32C}.get(self.accum)
        if metric is None:
            raise InvalidArgument(f"SearchParams: unknown metric {self.metric!r}")
        if accum is None:
            raise InvalidArgument(f"SearchParams: unknown accum {self.accum!r}")
        return _lib.dvsg_search_params(int(self.iterations), int(self.beam_width), int(self.k),
                                       int(self.entry_count), metric, accum)


@dataclass(frozen=True)
class ScoredId:
    """dataset.hpp:33-46: ordering is (dist, id)."""

    id: int
    dist: float


@dataclass
class GraphIndex:
    """graph_index.hpp:13-25.  adjacency is n x out_degree of local ids."""

    vectors: np.ndarray
    global_ids: np.ndarray
    out_degree: int
    adjacency: np.ndarray
    entry_order: Optional[np.ndarray] = None

    def size(self) -> int:
        return int(self.vectors.shape[0])

    def neighbors(self, local: int) -> np.ndarray:
        return self.adjacency[local]


@dataclass
class SearchResult:
    """graph_index.hpp:47-50."""

    hits: List[ScoredId]
    visited: int


@dataclass
class BuiltIndex:
    """index.hpp:14-23: centroids + placement + one GraphIndex per cluster."""

    centroids: np.ndarray              # clusters x dim
    cluster_to_rank: np.ndarray        # clusters
    ranks: int
    out_degree: int
    graphs: List[GraphIndex] = field(default_factory=list)

    def dim(self) -> int:
        return int(self.centroids.shape[1])

    def clusters(self) -> int:
        return int(self.centroids.shape[0])

    def total_vectors(self) -> int:
        return sum(g.size() for g in self.graphs)


@dataclass
class PipelineResult:
    """simulator.hpp:86-93 (functional fields)."""

    ids: np.ndarray       # nq x k (ragged by counts)
    dists: np.ndarray     # nq x k
    counts: np.ndarray    # nq
    hit_vectors: Optional[np.ndarray]  # nq x k x dim
    visited_total: int

    @property
    def hits(self) -> List[List[ScoredId]]:
        return [[ScoredId(int(self.ids[q, i]), float(self.dists[q, i]))
                 for i in range(int(self.counts[q]))] for q in range(len(self.counts))]


class Context:
    """One CUDA device with its resident index (dvsg_ctx)."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        check(lib.dvsg_create(int(device), ctypes.byref(h)))
        self._h = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.dvsg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return int(lib.dvsg_stream(self._h) or 0)

    def synchronize(self) -> None:
        check(lib.dvsg_synchronize(self._h))

    def kernel_launches(self) -> int:
        return int(lib.dvsg_kernel_launches(self._h))

    # ---- index -------------------------------------------------------------
    def reset(self) -> None:
        check(lib.dvsg_index_reset(self._h))

    def set_centroids(self, centroids, cluster_to_rank=None, ranks: int = 1) -> None:
        c = _f32(centroids, 2)
        ctr = None if cluster_to_rank is None else _u32(cluster_to_rank)
        check(lib.dvsg_set_centroids(self._h, _ptr(c), c.shape[0], c.shape[1], _ptr(ctr), int(ranks)))

    def load_partition(self, cluster: int, g: GraphIndex) -> None:
        v = _f32(g.vectors, 2)
        adj = _u32(g.adjacency).reshape(v.shape[0], -1) if v.shape[0] else _u32(g.adjacency)
        gids = None if g.global_ids is None else _u32(g.global_ids)
        eo = None if g.entry_order is None else _u32(g.entry_order)
        check(lib.dvsg_load_partition(self._h, int(cluster), v.shape[0], v.shape[1] if v.ndim == 2 else 0,
                                      int(g.out_degree), _ptr(v), _ptr(adj), _ptr(gids), _ptr(eo)))

    def load_index(self, index: BuiltIndex, rank: int = -1) -> None:
        """Upload a BuiltIndex (all clusters, or those placed on `rank`)."""
        self.reset()
        for c, g in enumerate(index.graphs):
            if rank < 0 or int(index.cluster_to_rank[c]) == rank:
                self.load_partition(c, g)
        self.set_centroids(index.centroids, index.cluster_to_rank, index.ranks)

    def load_index_file(self, path: str, rank: int = -1) -> None:
        check(lib.dvsg_load_index_file(self._h, str(path).encode(), int(rank)))

    def info(self):
        np_, dim, dg, cl = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(lib.dvsg_index_info(self._h, ctypes.byref(np_), ctypes.byref(dim), ctypes.byref(dg),
                                  ctypes.byref(cl), None, None))
        ids = np.zeros(np_.value, np.uint32)
        sizes = np.zeros(np_.value, np.uint64)
        check(lib.dvsg_index_info(self._h, None, None, None, None, _ptr(ids), _ptr(sizes)))
        return {"partitions": np_.value, "dim": dim.value, "out_degree": dg.value,
                "clusters": cl.value, "cluster_ids": ids, "sizes": sizes}

    def entry_order(self, cluster: int) -> np.ndarray:
        n = int(self.info()["sizes"][list(self.info()["cluster_ids"]).index(cluster)])
        out = np.zeros(n, np.uint32)
        check(lib.dvsg_get_entry_order(self._h, int(cluster), _ptr(out)))
        return out

    # ---- search ------------------------------------------------------------
    def beam_search(self, cluster: int, queries, p: SearchParams
                    ) -> Tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
        """Batched beam_search_stats -> (ids nq x k, dists nq x k, counts, visited)."""
        q = _f32(queries)
        if q.ndim == 1:
            q = q.reshape(1, -1)
        nq, dim = q.shape
        cp = p.to_c()
        k = max(int(p.k), 1)
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float32)
        counts = np.zeros(nq, np.uint32)
        visited = np.zeros(nq, np.uint64)
        check(lib.dvsg_beam_search(self._h, int(cluster), _ptr(q), nq, dim, ctypes.byref(cp),
                                   _ptr(ids), _ptr(dists), _ptr(counts), _ptr(visited)))
        return ids, dists, counts, visited

    def beam_search_sharded_emulated(self, nranks: int, queries, p: SearchParams):
        """Node-sharded search with `nranks` ranks emulated on this device over
        the resident whole-graph partition -> (ids, dists, counts, visited)."""
        q = _f32(queries)
        if q.ndim == 1:
            q = q.reshape(1, -1)
        nq, dim = q.shape
        cp = p.to_c()
        k = max(int(p.k), 1)
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float32)
        counts = np.zeros(nq, np.uint32)
        visited = np.zeros(nq, np.uint64)
        check(lib.dvsg_beam_search_sharded_emulated(self._h, int(nranks), _ptr(q), nq, dim, ctypes.byref(cp),
                                                    _ptr(ids), _ptr(dists), _ptr(counts), _ptr(visited)))
        return ids, dists, counts, visited

    # ---- node-sharded multi-GPU (one process per GPU) --------------------------
    def shard_init(self, nranks: int, rank: int, shard_vectors, n_total: int, adjacency,
                   entry_order, global_ids=None) -> None:
        v = _f32(shard_vectors, 2)
        adj = _u32(adjacency)
        eo = _u32(entry_order)
        gids = None if global_ids is None else _u32(global_ids)
        check(lib.dvsg_shard_init(self._h, int(nranks), int(rank), int(n_total), v.shape[1],
                                  int(adj.shape[1]), _ptr(v), _ptr(adj), _ptr(gids), _ptr(eo)))

    def shard_init_resident(self, nranks: int, rank: int) -> None:
        """dvsg_shard_init_resident: keep this rank's rows of the resident partition."""
        check(lib.dvsg_shard_init_resident(self._h, int(nranks), int(rank)))

    def shard_export(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        check(lib.dvsg_shard_export(self._h, buf))
        return buf.raw

    def shard_connect(self, handles) -> None:
        blob = b"".join(handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        check(lib.dvsg_shard_connect(self._h, buf))

    def set_shard_exchange(self, mode: str) -> None:
        """'bulk' (bulk-synchronous phases over NVLink peer stores,
        xchg_kernel.cu; default), 'fused' (per-CTA round trips,
        shard_kernel.cu) or 'nccl' (the bulk protocol with host-driven
        ncclSend/ncclRecv -- the measured baseline); all exact."""
        check(lib.dvsg_set_shard_exchange(self._h, {"bulk": 0, "fused": 1, "nccl": 2}[mode]))

    def nccl_unique_id(self) -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(lib.dvsg_nccl_unique_id(self._h, buf))
        return buf.raw

    def nccl_connect(self, uid: bytes) -> None:
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        check(lib.dvsg_nccl_connect(self._h, buf))

    def shard_prepare(self) -> None:
        check(lib.dvsg_shard_prepare(self._h))

    def search_sharded_device(self, d_queries: int, nq: int, dim: int, p: SearchParams, d_ids: int,
                              d_dists: int, d_counts: int, d_visited: int) -> None:
        cp = p.to_c()
        check(lib.dvsg_search_sharded_device(self._h, ctypes.c_void_p(d_queries), int(nq), int(dim),
                                             ctypes.byref(cp), ctypes.c_void_p(d_ids),
                                             ctypes.c_void_p(d_dists), ctypes.c_void_p(d_counts),
                                             ctypes.c_void_p(d_visited)))

    def last_assign_info(self):
        """(path, fallbacks) of the last assign: path 0 warp, 1 fp64 tiles,
        2 tensor cores; fallbacks = queries the certificate sent to the exact
        kernel (path 2 only)."""
        path, fb = ctypes.c_int(), ctypes.c_uint64()
        check(lib.dvsg_last_assign_info(self._h, ctypes.byref(path), ctypes.byref(fb)))
        return int(path.value), int(fb.value)

    def set_vector_storage(self, mode: str) -> None:
        """"f32" (default) or "u8": K1 gathers a byte copy of the resident rows
        (every coordinate must be an integer in [0, 255]; results unchanged)."""
        m = {"f32": 0, "u8": 1}.get(mode)
        if m is None:
            raise InvalidArgument(f"set_vector_storage: unknown mode {mode!r}")
        check(lib.dvsg_set_vector_storage(self._h, m))

    def last_knn_info(self):
        """(exact_mode, fallbacks) of the last build_graph / brute_force_topk:
        0 fp32 tiles, 1 fp32 candidates + fp64 re-rank + certificate."""
        mode, fb = ctypes.c_int(), ctypes.c_uint64()
        check(lib.dvsg_last_knn_info(self._h, ctypes.byref(mode), ctypes.byref(fb)))
        return int(mode.value), int(fb.value)

    def assign_top_c(self, queries, c: int) -> np.ndarray:
        q = _f32(queries, 2)
        out = np.zeros((q.shape[0], max(int(c), 1)), np.uint32)
        check(lib.dvsg_assign_top_c(self._h, _ptr(q), q.shape[0], q.shape[1], int(c), _ptr(out)))
        return out

    def combine_results(self, ids, dists, counts, k: int):
        """ids/dists: nq x nparts x stride, counts nq x nparts."""
        ids = _u32(ids)
        dists = _f32(dists)
        counts = _u32(counts)
        nq, nparts, stride = ids.shape
        oi = np.zeros((nq, max(int(k), 1)), np.uint32)
        od = np.zeros((nq, max(int(k), 1)), np.float32)
        oc = np.zeros(nq, np.uint32)
        check(lib.dvsg_combine_results(self._h, nq, nparts, _ptr(ids), _ptr(dists), _ptr(counts),
                                       stride, int(k), _ptr(oi), _ptr(od), _ptr(oc)))
        return oi, od, oc

    def run_pipeline(self, queries, p: SearchParams, fanout: int, ranks: int,
                     batch_index: int = 0, with_vectors: bool = True,
                     out: Optional[dict] = None) -> PipelineResult:
        """Host buffers in and out (H2D/D2H inside).  `out` may hold
        preallocated (e.g. pinned) arrays: ids, dists, counts, vectors."""
        q = _f32(queries, 2)
        nq, dim = q.shape
        cp = p.to_c()
        k = max(int(p.k), 1)
        out = out or {}
        ids = out.get("ids")
        ids = np.zeros((nq, k), np.uint32) if ids is None else ids
        dists = out.get("dists")
        dists = np.zeros((nq, k), np.float32) if dists is None else dists
        counts = out.get("counts")
        counts = np.zeros(nq, np.uint32) if counts is None else counts
        vecs = out.get("vectors")
        if vecs is None and with_vectors:
            vecs = np.zeros((nq, k, dim), np.float32)
        if not with_vectors:
            vecs = None
        for a, shape, dt in ((ids, (nq, k), np.uint32), (dists, (nq, k), np.float32),
                             (counts, (nq,), np.uint32)):
            if a.shape != shape or a.dtype != dt or not a.flags.c_contiguous:
                raise InvalidArgument("run_pipeline: bad output buffer")
        vt = ctypes.c_uint64(0)
        check(lib.dvsg_run_pipeline(self._h, _ptr(q), nq, dim, ctypes.byref(cp), int(fanout),
                                    int(ranks), int(batch_index), _ptr(ids), _ptr(dists),
                                    _ptr(counts), _ptr(vecs), ctypes.byref(vt)))
        return PipelineResult(ids, dists, counts, vecs, int(vt.value))

    def build_graph(self, vectors, out_degree: int) -> np.ndarray:
        v = _f32(vectors, 2)
        adj = np.zeros((v.shape[0], int(out_degree)), np.uint32)
        check(lib.dvsg_build_graph(self._h, _ptr(v), v.shape[0], v.shape[1], int(out_degree), _ptr(adj)))
        return adj

    def last_search_stats(self):
        u, v, e = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.dvsg_last_search_stats(self._h, ctypes.byref(u), ctypes.byref(v), ctypes.byref(e)))
        return {"units": u.value, "visited": v.value, "expanded": e.value}

    def run_pipeline_device(self, d_queries: int, nq: int, dim: int, p: SearchParams, fanout: int,
                            d_ids: int, d_dists: int, d_counts: int, d_vectors: int = 0,
                            d_visited: int = 0) -> None:
        """Asynchronous on self.stream; all arguments are device addresses."""
        cp = p.to_c()
        check(lib.dvsg_run_pipeline_device(self._h, ctypes.c_void_p(d_queries), int(nq), int(dim),
                                           ctypes.byref(cp), int(fanout), ctypes.c_void_p(d_ids),
                                           ctypes.c_void_p(d_dists), ctypes.c_void_p(d_counts),
                                           ctypes.c_void_p(d_vectors or None),
                                           ctypes.c_void_p(d_visited or None)))

    # ---- device-pointer building blocks (asynchronous on self.stream) ------------
    def search_units_device(self, d_queries: int, nq: int, dim: int, d_unit_query: int,
                            d_unit_cluster: int, nunits: int, p: SearchParams, d_ids: int,
                            d_dists: int, d_counts: int, d_visited: int) -> None:
        cp = p.to_c()
        v = ctypes.c_void_p
        check(lib.dvsg_search_units_device(self._h, v(d_queries), int(nq), int(dim), v(d_unit_query),
                                           v(d_unit_cluster), int(nunits), ctypes.byref(cp), v(d_ids),
                                           v(d_dists), v(d_counts), v(d_visited)))

    def assign_top_c_device(self, d_queries: int, nq: int, dim: int, c: int, d_out: int) -> None:
        check(lib.dvsg_assign_top_c_device(self._h, ctypes.c_void_p(d_queries), int(nq), int(dim), int(c),
                                           ctypes.c_void_p(d_out)))

    def combine_results_device(self, nq: int, nparts: int, d_ids: int, d_dists: int, d_counts: int,
                               stride: int, k: int, d_out_ids: int, d_out_dists: int, d_out_count: int) -> None:
        v = ctypes.c_void_p
        check(lib.dvsg_combine_results_device(self._h, int(nq), int(nparts), v(d_ids), v(d_dists), v(d_counts),
                                              int(stride), int(k), v(d_out_ids), v(d_out_dists), v(d_out_count)))

    def gather_vectors_device(self, d_ids: int, d_counts: int, n: int, k: int, d_out: int) -> None:
        v = ctypes.c_void_p
        check(lib.dvsg_gather_vectors_device(self._h, v(d_ids), v(d_counts), int(n), int(k), v(d_out)))

    def brute_force_topk(self, db, queries, k: int):
        """topk.cpp:12-30 on the GPU -> (ids nq x k, dists nq x k)."""
        d = _f32(db, 2)
        q = _f32(queries, 2)
        if q.shape[1] != d.shape[1]:
            raise InvalidArgument("brute_force_topk: dimension mismatch")
        ids = np.zeros((q.shape[0], max(int(k), 1)), np.uint32)
        dists = np.zeros((q.shape[0], max(int(k), 1)), np.float32)
        check(lib.dvsg_brute_force_topk(self._h, _ptr(d), d.shape[0], d.shape[1], _ptr(q), q.shape[0],
                                        int(k), _ptr(ids), _ptr(dists)))
        return ids, dists

    # ---- timing --------------------------------------------------------------
    # ---- large-index construction (device pointers, synchronous) -----------
    def row_norms_device(self, d_x: int, n: int, dpad: int, d_out: int) -> None:
        check(lib.dvsg_row_norms_device(self._h, d_x, n, dpad, d_out))

    def range_topk_device(self, d_rows: int, d_row_norms: int, d_cols: int, d_col_norms: int, dpad: int,
                          d_row_map: int, d_blocks: int, nblocks: int, d_list_off: int, d_ranges: int,
                          m: int, flags: int, d_out_ids: int, d_out_dists: int, out_stride: int) -> None:
        check(lib.dvsg_range_topk_device(self._h, d_rows, d_row_norms, d_cols, d_col_norms, dpad,
                                         d_row_map or None, d_blocks or None, nblocks, d_list_off or None,
                                         d_ranges or None, m, flags, d_out_ids, d_out_dists or None,
                                         out_stride))

    def to_bf16_device(self, d_x: int, n: int, dpad: int, kpad: int, d_out: int) -> None:
        check(lib.dvsg_to_bf16_device(self._h, d_x, n, dpad, kpad, d_out))

    def range_topk_bf16_device(self, d_rows: int, d_row_norms: int, d_cols: int, d_col_norms: int, kpad: int,
                               d_row_map: int, d_blocks: int, nblocks: int, d_list_off: int, d_ranges: int,
                               m: int, flags: int, d_out_ids: int, d_out_dists: int, out_stride: int) -> None:
        check(lib.dvsg_range_topk_bf16_device(self._h, d_rows, d_row_norms, d_cols, d_col_norms, kpad,
                                              d_row_map or None, d_blocks or None, nblocks, d_list_off or None,
                                              d_ranges or None, m, flags, d_out_ids, d_out_dists or None,
                                              out_stride))

    def segment_means_device(self, d_x: int, dpad: int, d_idx: int, d_off: int, nseg: int,
                             d_cents: int) -> None:
        check(lib.dvsg_segment_means_device(self._h, d_x, dpad, d_idx or None, d_off, nseg, d_cents))

    def compute_entry_order_device(self, d_x: int, n: int, dim: int, dpad: int, d_out: int) -> None:
        check(lib.dvsg_compute_entry_order_device(self._h, d_x, n, dim, dpad, d_out))

    def partition_alloc_device(self, cluster: int, n: int, dim: int, out_degree: int):
        """-> (d_vectors, d_adjacency, d_global_ids, d_entry_order) pointers into the
        context's index arrays (dvsg_partition_alloc_device)."""
        v, a, g, e = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        check(lib.dvsg_partition_alloc_device(self._h, int(cluster), int(n), int(dim), int(out_degree),
                                              ctypes.byref(v), ctypes.byref(a), ctypes.byref(g),
                                              ctypes.byref(e)))
        return int(v.value or 0), int(a.value or 0), int(g.value or 0), int(e.value or 0)

    def partition_commit_device(self, flags: int) -> None:
        check(lib.dvsg_partition_commit_device(self._h, int(flags)))

    def partition_view_device(self, cluster: int):
        """-> (d_vectors, d_adjacency, d_global_ids, d_entry_order, n) of a resident partition."""
        v, a, g, e, n = (ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(),
                         ctypes.c_uint64())
        check(lib.dvsg_partition_view_device(self._h, int(cluster), ctypes.byref(v), ctypes.byref(a),
                                             ctypes.byref(g), ctypes.byref(e), ctypes.byref(n)))
        return int(v.value or 0), int(a.value or 0), int(g.value or 0), int(e.value or 0), int(n.value)

    def optimize_graph_device(self, d_adjacency: int, n: int, out_degree: int, keep: int) -> None:
        check(lib.dvsg_optimize_graph_device(self._h, d_adjacency, int(n), int(out_degree), int(keep)))

    # ---- cluster-sharded run_pipeline, device-initiated exchange -------------
    def cluster_comm_init(self, nranks: int, rank: int, max_queries: int, max_fanout: int, k: int,
                          with_vectors: bool = True) -> None:
        check(lib.dvsg_cluster_comm_init(self._h, int(nranks), int(rank), int(max_queries), int(max_fanout),
                                         int(k), int(bool(with_vectors))))

    def cluster_comm_export(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        check(lib.dvsg_cluster_comm_export(self._h, buf))
        return buf.raw

    def cluster_comm_connect(self, handles) -> None:
        blob = b"".join(handles)
        check(lib.dvsg_cluster_comm_connect(self._h, ctypes.c_char_p(blob)))

    def cluster_comm_arena(self) -> int:
        return int(lib.dvsg_cluster_comm_arena(self._h) or 0)

    def cluster_comm_connect_local(self, arenas) -> None:
        arr = (ctypes.c_void_p * len(arenas))(*[int(a) for a in arenas])
        check(lib.dvsg_cluster_comm_connect_local(self._h, arr))

    def run_pipeline_cluster_device(self, d_queries: int, nq: int, dim: int, p: SearchParams, fanout: int,
                                    d_ids: int, d_dists: int, d_counts: int, d_vectors: int = 0,
                                    d_visited_total: int = 0) -> None:
        cp = p.to_c()
        check(lib.dvsg_run_pipeline_cluster_device(self._h, ctypes.c_void_p(d_queries), int(nq), int(dim),
                                                   ctypes.byref(cp), int(fanout), ctypes.c_void_p(d_ids),
                                                   ctypes.c_void_p(d_dists), ctypes.c_void_p(d_counts),
                                                   ctypes.c_void_p(d_vectors or None),
                                                   ctypes.c_void_p(d_visited_total or None)))

    def cluster_comm_check(self) -> None:
        check(lib.dvsg_cluster_comm_check(self._h))

    def index_integral(self) -> bool:
        out = ctypes.c_int()
        check(lib.dvsg_index_integral(self._h, ctypes.byref(out)))
        return bool(out.value)

    def set_timing(self, on: bool) -> None:
        check(lib.dvsg_set_timing(self._h, 1 if on else 0))

    def last_timings(self):
        vals = [ctypes.c_float() for _ in range(4)]
        check(lib.dvsg_last_timings(self._h, *[ctypes.byref(v) for v in vals]))
        return {"search_ms": vals[0].value, "assign_ms": vals[1].value,
                "combine_ms": vals[2].value, "total_ms": vals[3].value}

    def last_pipeline_timeline(self, rank: int = 0) -> List[dict]:
        """Measured intervals of the last run_pipeline made with timing on:
        per microbatch h2d (comm lane), search (compute lane), d2h (comm
        lane), ms from the pipeline start -- the measured counterpart of the
        reference's modeled Timeline (simulator.hpp Interval fields)."""
        buf = np.zeros(6 * 16, np.float64)
        n = ctypes.c_int(0)
        check(lib.dvsg_last_pipeline_timeline(self._h, _ptr(buf), 16, ctypes.byref(n)))
        out = []
        for mb in range(n.value):
            t = buf[6 * mb:6 * mb + 6]
            for stage, lane, a, b in (("h2d", "comm", t[0], t[1]), ("search", "compute", t[2], t[3]),
                                      ("d2h", "comm", t[4], t[5])):
                out.append({"rank": rank, "lane": lane, "stage": stage, "microbatch": mb,
                            "start": float(a), "end": float(b)})
        return out


def _sharded_timeline(ctx, rank: int = 0) -> List[dict]:
    buf = np.zeros(3 * 1024, np.float64)
    n = ctypes.c_int(0)
    check(lib.dvsg_last_sharded_timeline(ctx._h, _ptr(buf), 1024, ctypes.byref(n)))
    return [{"rank": rank, "lane": "compute" if buf[3 * i] == 0 else "comm",
             "stage": "xg_step" if buf[3 * i] == 0 else "exchange", "start": float(buf[3 * i + 1]),
             "end": float(buf[3 * i + 2])} for i in range(n.value)]


Context.last_sharded_timeline = _sharded_timeline


TIMELINE_STAGE_ORDER = {"kmeans": 0, "dispatch": 1, "search": 2, "combine": 3}
MEASURED_STAGE_ORDER = {"h2d": 0, "search": 1, "d2h": 2}


def check_timeline(intervals, stage_order=None) -> Optional[str]:
    """check_timeline, simulator.cpp:170-217: no two intervals of one (rank,
    lane) overlap, and every stage of a (rank, microbatch) starts after its
    predecessor ends.  Returns None or the reference's error message.
    stage_order defaults to the measured pipeline's (h2d, search, d2h) when
    the intervals use those names, else the reference's four stages."""
    if stage_order is None:
        stage_order = MEASURED_STAGE_ORDER if any(iv["stage"] in MEASURED_STAGE_ORDER and iv["stage"] != "search"
                                                  for iv in intervals) else TIMELINE_STAGE_ORDER
    lanes = {}
    for iv in intervals:
        if iv["end"] < iv["start"]:
            return f"interval with end < start on rank {iv['rank']}"
        lanes.setdefault((iv["rank"], iv["lane"]), []).append(iv)
    lane_order = {"compute": 0, "comm": 1}
    for (rank, lane) in sorted(lanes, key=lambda kv: (kv[0], lane_order.get(kv[1], 2))):
        ivs = sorted(lanes[(rank, lane)], key=lambda v: (v["start"], v["end"]))
        for a, b in zip(ivs, ivs[1:]):
            if b["start"] < a["end"]:
                return f"overlap on rank {rank} lane {lane} at t={b['start']:.6f}"
    by_stage = {}
    for iv in intervals:
        key = (iv["rank"], iv["microbatch"], stage_order[iv["stage"]])
        if key in by_stage:
            return f"duplicate stage interval for rank {iv['rank']} microbatch {iv['microbatch']}"
        by_stage[key] = iv
    for (rank, mb, s), iv in sorted(by_stage.items()):
        if s == 0:
            continue
        prev = by_stage.get((rank, mb, s - 1))
        if prev is None:
            return f"missing predecessor stage for rank {rank} microbatch {mb}"
        if iv["start"] < prev["end"]:
            return (f"dependency violation: {iv['stage']} of microbatch {mb} starts before "
                    f"{prev['stage']} ends")
    return None


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


# ---------------------------------------------------------------------------
# reference-shaped free functions (graph_index.hpp, simulator.hpp, kmeans.hpp)
# ---------------------------------------------------------------------------
def validate(p: SearchParams) -> None:
    """graph_index.cpp:14-19."""
    if p.iterations < 1 or p.beam_width < 1 or p.k < 1 or p.entry_count < 1:
        raise InvalidArgument(
            "SearchParams: iterations, beam_width, k and entry_count must all be >= 1")


def compute_entry_order(vectors) -> np.ndarray:
    """graph_index.cpp:21-44 (host C++ in libdvsg, exact)."""
    v = _f32(vectors, 2)
    out = np.zeros(v.shape[0], np.uint32)
    check(lib.dvsg_compute_entry_order(_ptr(v), v.shape[0], v.shape[1], _ptr(out)))
    return out


def build_graph(vectors, out_degree: int, global_ids=None, ctx: Optional[Context] = None) -> GraphIndex:
    """graph_index.cpp:46-97 on the GPU (K6)."""
    v = _f32(vectors, 2)
    if v.shape[0] == 0:
        raise InvalidArgument("build_graph: empty partition")
    if out_degree < 1:
        raise InvalidArgument("build_graph: out_degree must be >= 1")
    gids = np.arange(v.shape[0], dtype=np.uint32) if global_ids is None else _u32(global_ids)
    if gids.shape[0] != v.shape[0]:
        raise InvalidArgument(f"build_graph: global id count {gids.shape[0]} != partition size {v.shape[0]}")
    adj = (ctx or default_context()).build_graph(v, out_degree)
    return GraphIndex(v, gids, int(out_degree), adj, compute_entry_order(v))


def _single_graph_ctx(g: GraphIndex, ctx: Optional[Context]) -> Context:
    c = ctx or default_context()
    key = (id(g), g.size())
    if getattr(c, "_single_key", None) != key:
        c.reset()
        c.load_partition(0, g)
        c._single_key = key
    return c


def beam_search_batch(g: GraphIndex, queries, p: SearchParams, ctx: Optional[Context] = None):
    """Batched beam_search_stats over one partition -> (ids, dists, counts, visited)."""
    validate(p)
    if g.size() == 0:
        raise InvalidArgument("beam_search: empty graph")
    c = _single_graph_ctx(g, ctx)
    return c.beam_search(0, queries, p)


def beam_search_stats(g: GraphIndex, query, p: SearchParams, seed: int = 0,
                      ctx: Optional[Context] = None) -> SearchResult:
    """graph_index.hpp:58-59.  The seed is accepted and ignored (graph_index.hpp:55-57)."""
    del seed
    q = _f32(query)
    if q.ndim != 1:
        raise InvalidArgument("beam_search: query must be one vector")
    if q.shape[0] != g.vectors.shape[1]:
        raise InvalidArgument(f"beam_search: query dim {q.shape[0]} != index dim {g.vectors.shape[1]}")
    ids, dists, counts, visited = beam_search_batch(g, q.reshape(1, -1), p, ctx)
    n = int(counts[0])
    return SearchResult([ScoredId(int(ids[0, i]), float(dists[0, i])) for i in range(n)],
                        int(visited[0]))


def beam_search(g: GraphIndex, query, p: SearchParams, seed: int = 0,
                ctx: Optional[Context] = None) -> List[ScoredId]:
    return beam_search_stats(g, query, p, seed, ctx).hits


def visited_count(g: GraphIndex, query, p: SearchParams, ctx: Optional[Context] = None) -> int:
    return beam_search_stats(g, query, p, 0, ctx).visited


def combine_results(partials: Sequence[Sequence[ScoredId]], k: int,
                    ctx: Optional[Context] = None) -> List[ScoredId]:
    """simulator.cpp:219-243 on the GPU (K4)."""
    if k < 1:
        raise InvalidArgument("combine_results: k must be >= 1")
    nparts = len(partials)
    stride = max([len(p) for p in partials] + [1])
    ids = np.zeros((1, max(nparts, 1), stride), np.uint32)
    dists = np.zeros((1, max(nparts, 1), stride), np.float32)
    counts = np.zeros((1, max(nparts, 1)), np.uint32)
    for j, part in enumerate(partials):
        counts[0, j] = len(part)
        for i, s in enumerate(part):
            ids[0, j, i] = s.id
            dists[0, j, i] = s.dist
    if nparts == 0:
        return []
    oi, od, oc = (ctx or default_context()).combine_results(ids, dists, counts, k)
    return [ScoredId(int(oi[0, i]), float(od[0, i])) for i in range(int(oc[0]))]


def assign_top_c(centroids, queries, c: int, ctx: Optional[Context] = None) -> np.ndarray:
    """kmeans.cpp:243-280 on the GPU (K5).  Loads the centroids into ctx."""
    cx = ctx or default_context()
    cents = _f32(centroids, 2)
    q = _f32(queries, 2)
    if q.shape[1] != cents.shape[1]:
        raise InvalidArgument(f"assign_top_c: query dim {q.shape[1]} != centroid dim {cents.shape[1]}")
    cx.reset()
    cx._single_key = None
    cx.set_centroids(cents, None, 1)
    return cx.assign_top_c(q, c)


@dataclass
class KmeansStats:
    """kmeans.hpp:27-30."""
    wcss: np.ndarray
    iterations: int


def kmeans_train(db, clusters: int, max_iters: int, seed: int = 42, ctx: Optional[Context] = None,
                 stats: bool = False):
    """kmeans.cpp:189-241 on the GPU (dvsg_kmeans_train): the reference's
    k-means++ seeding (mt19937_64), Lloyd loop, empty-cluster repair and final
    non-empty check.  -> centroids (clusters x dim), or (centroids, KmeansStats)."""
    cx = ctx or default_context()
    x = _f32(db, 2)
    cents = np.zeros((max(int(clusters), 1), x.shape[1]), np.float32)
    it = ctypes.c_int(0)
    wcss = np.zeros(max(int(max_iters), 1), np.float64)
    check(lib.dvsg_kmeans_train(cx.handle, _ptr(x), x.shape[0], x.shape[1], int(clusters), int(max_iters),
                                ctypes.c_uint64(int(seed)), _ptr(cents), ctypes.byref(it), _ptr(wcss)))
    return (cents, KmeansStats(wcss[:it.value].copy(), it.value)) if stats else cents


def partition_database(db, centroids, ctx: Optional[Context] = None) -> List[np.ndarray]:
    """kmeans.cpp:282-300: per cluster, the ids of its rows in row order."""
    cx = ctx or default_context()
    x = _f32(db, 2)
    cents = _f32(centroids, 2)
    if x.shape[1] != cents.shape[1]:
        raise InvalidArgument("partition_database: dim mismatch")
    lab = np.zeros(x.shape[0], np.uint32)
    check(lib.dvsg_partition_database(cx.handle, _ptr(x), x.shape[0], x.shape[1], _ptr(cents), cents.shape[0],
                                      _ptr(lab)))
    order = np.argsort(lab, kind="stable")
    bounds = np.searchsorted(lab[order], np.arange(cents.shape[0] + 1))
    return [order[bounds[c]:bounds[c + 1]].astype(np.uint32) for c in range(cents.shape[0])]


def build_index(db, clusters: int, out_degree: int, ranks: int = 1, kmeans_iters: int = 25, seed: int = 42,
                ctx: Optional[Context] = None) -> BuiltIndex:
    """index.cpp:43-72: kmeans_train -> place_clusters -> partition_database ->
    one build_graph per cluster (GPU K6 on integer data, exact host rows
    otherwise is the shim's job; this helper needs integer-valued data or an
    approximation-tolerant caller)."""
    cx = ctx or default_context()
    x = _f32(db, 2)
    if clusters < ranks:
        raise InvalidArgument(f"build_index: clusters ({clusters}) must be >= ranks ({ranks})")
    cents = kmeans_train(x, clusters, kmeans_iters, seed, ctx=cx)
    placement = place_clusters(clusters, ranks)
    graphs = []
    for ids in partition_database(x, cents, ctx=cx):
        part = np.ascontiguousarray(x[ids])
        graphs.append(build_graph(part, out_degree, global_ids=ids, ctx=cx))
    return BuiltIndex(cents, placement, ranks, out_degree, graphs)


def place_clusters(clusters: int, ranks: int) -> np.ndarray:
    """router.cpp:28-43: cluster i -> rank i mod R; refuses an empty rank."""
    if ranks < 1:
        raise InvalidArgument("ClusterTopology: ranks and ranks_per_node must be >= 1")
    if clusters < ranks:
        raise InvalidArgument(f"place_clusters: {clusters} clusters over {ranks} ranks would leave a rank empty")
    return (np.arange(clusters) % ranks).astype(np.uint32)


def route(assignment: np.ndarray, cluster_to_rank: np.ndarray, origin_rank: int, ranks: int):
    """router.cpp:52-79: per destination rank, (query, origin, cluster) entries."""
    if origin_rank < 0 or origin_rank >= ranks:
        raise InvalidArgument(f"route: origin rank {origin_rank} outside 0..{ranks - 1}")
    per_rank: List[List[Tuple[int, int, int]]] = [[] for _ in range(ranks)]
    for q, row in enumerate(np.asarray(assignment)):
        for cl in row:
            if cl >= len(cluster_to_rank):
                raise InternalError(f"route: cluster id {cl} outside placement of {len(cluster_to_rank)} clusters")
            per_rank[int(cluster_to_rank[cl])].append((q, origin_rank, int(cl)))
    return per_rank


def run_pipeline(index: BuiltIndex, queries, params: SearchParams, fanout: int, ranks: int,
                 batch_index: int = 0, ctx: Optional[Context] = None,
                 with_vectors: bool = True) -> PipelineResult:
    """simulator.cpp:245-337 functional part, on one GPU."""
    cx = ctx or default_context()
    key = (id(index), index.total_vectors())
    if getattr(cx, "_index_key", None) != key:
        cx.load_index(index)
        cx._index_key = key
        cx._single_key = None
    return cx.run_pipeline(queries, params, fanout, ranks, batch_index, with_vectors)


def save_index(index: BuiltIndex, path: str) -> None:
    """index_file.cpp:88-147 (FNSY v1)."""
    C = index.clusters()
    if C < 1 or len(index.graphs) != C:
        raise InvalidArgument("BuiltIndex: index is not built")
    sizes = [g.size() for g in index.graphs]
    offs = np.zeros(C + 1, np.uint64)
    offs[1:] = np.cumsum(sizes)
    vec = _f32(np.concatenate([g.vectors for g in index.graphs]))
    adj = _u32(np.concatenate([np.asarray(g.adjacency).reshape(-1) for g in index.graphs]))
    gids = _u32(np.concatenate([g.global_ids for g in index.graphs]))
    cents = _f32(index.centroids, 2)
    ctr = _u32(index.cluster_to_rank)
    check(lib.dvsg_save_index_file(str(path).encode(), C, cents.shape[1], int(index.out_degree),
                                   _ptr(cents), _ptr(ctr), int(index.ranks), _ptr(offs), _ptr(vec),
                                   _ptr(adj), _ptr(gids)))


def load_index(path: str, ctx: Optional[Context] = None, rank: int = -1) -> Context:
    """index_file.cpp:149-296: parse FNSY v1 straight into device memory."""
    cx = ctx or default_context()
    cx.load_index_file(path, rank)
    cx._index_key = None
    cx._single_key = None
    return cx
