"""Multi-GPU plumbing (one process per GPU).

Node-sharded search (SURVEY 8e design B): torch.distributed carries only
control-plane data -- the 64-byte CUDA IPC handles of each rank's comm arena
(all_gather_object), the NCCL unique id of the baseline exchange, barriers.
The data path -- candidate ids out, scored keys back -- is the kernels' own
NVLink peer stores (xchg_kernel.cu / shard_kernel.cu), not a collective.
The shard rule is the C-ABI's (dvsg_shard_init): S = ceil(n / R), rank r owns
node ids [r*S, min(n, (r+1)*S)).

Cluster-sharded pipeline (SURVEY 8e design A, the reference's own
run_pipeline semantics across ranks): run_pipeline_distributed below --
cluster i lives on rank placement[i] (router.cpp:38-41), one all-to-all
dispatches the routed (query, cluster) units to their owners and one sends
the results back (NCCL through torch.distributed), the library kernels do
the assignment, the per-partition searches and the combine.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple


def shard_range(n: int, nranks: int, rank: int) -> Tuple[int, int]:
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError(f"shard_range: rank {rank} of {nranks}")
    s = (n + nranks - 1) // nranks
    lo = min(n, s * rank)
    return lo, min(n, lo + s)


def owner_of(node: int, n: int, nranks: int) -> int:
    return node // ((n + nranks - 1) // nranks)


def exchange_handles(handle: bytes, group=None) -> List[bytes]:
    """all_gather the 64-byte IPC handles (rank order)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out: List[Optional[bytes]] = [None] * world
    dist.all_gather_object(out, handle, group=group)
    for r, h in enumerate(out):
        if not isinstance(h, (bytes, bytearray)) or len(h) != 64:
            raise RuntimeError(f"exchange_handles: bad handle from rank {r}")
    return [bytes(h) for h in out]  # type: ignore[arg-type]


def setup_sharded(ctx, rank: int, nranks: int, data, adjacency, entry_order,
                  global_ids=None, group=None, exchange=exchange_handles) -> Tuple[int, int]:
    """Load this rank's shard + the replicated graph, then connect to every
    rank's comm arena.  Returns the owned node range."""
    n = int(data.shape[0])
    lo, hi = shard_range(n, nranks, rank)
    ctx.shard_init(nranks, rank, data[lo:hi], n, adjacency, entry_order, global_ids)
    handles = exchange(ctx.shard_export(), group)
    ctx.shard_connect(handles)
    return lo, hi


def setup_sharded_resident(ctx, rank: int, nranks: int, group=None,
                           exchange=exchange_handles) -> None:
    """Shard the context's resident partition (every rank built the same
    graph) and connect to every rank's comm arena."""
    ctx.shard_init_resident(nranks, rank)
    handles = exchange(ctx.shard_export(), group)
    ctx.shard_connect(handles)


def setup_cluster_comm(ctx, rank: int, world: int, max_queries: int, max_fanout: int, k: int,
                       with_vectors: bool = True, group=None, exchange=exchange_handles) -> None:
    """Arena of the device-initiated cluster exchange (cluster_xchg.cu); ctx
    already holds this rank's partitions and the routing table."""
    ctx.cluster_comm_init(world, rank, max_queries, max_fanout, k, with_vectors)
    ctx.cluster_comm_connect(exchange(ctx.cluster_comm_export(), group))


def run_pipeline_cluster(ctx, d_q, p, fanout: int, with_vectors: bool = True):
    """run_pipeline (simulator.cpp:250-337), cluster-sharded, with the
    dispatch / combine done by the library's own peer-store kernels (K3/K4) --
    no NCCL collective and no host round trip.  Collective: every rank calls
    it for its own batch.  -> torch tensors (ids, dists, counts, vectors or
    None, visited_total as a 1-element int64 tensor), asynchronous on ctx.stream."""
    import torch
    dev = d_q.device
    nq, dim = int(d_q.shape[0]), int(d_q.shape[1])
    k = int(p.k)
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    counts = torch.empty((nq,), dtype=torch.int32, device=dev)
    vecs = torch.zeros((nq, k, dim), dtype=torch.float32, device=dev) if with_vectors else None
    vt = torch.zeros(1, dtype=torch.int64, device=dev)
    torch.cuda.current_stream(dev).synchronize()  # d_q / outputs ready before the library stream uses them
    ctx.run_pipeline_cluster_device(d_q.data_ptr(), nq, dim, p, fanout, ids.data_ptr(), dists.data_ptr(),
                                    counts.data_ptr(), vecs.data_ptr() if with_vectors else 0, vt.data_ptr())
    return ids, dists, counts, vecs, vt


def connect_nccl(ctx, rank: int, group=None) -> None:
    """NCCL communicator for the 'nccl' exchange: rank 0's unique id is
    broadcast over torch.distributed (control plane only)."""
    import torch.distributed as dist
    box = [ctx.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    ctx.nccl_connect(box[0])


def prepare_step(ctx, barrier) -> None:
    """Reset this rank's arena; no rank may launch before every reset is done."""
    ctx.shard_prepare()
    barrier()


def split_even(n: int, parts: int) -> Sequence[Tuple[int, int]]:
    return [(n * i // parts, n * (i + 1) // parts) for i in range(parts)]


def route_to_owners(assign, placement, world: int):
    """router.cpp:52-79 over device tensors: unit u = q * fanout + j is routed
    to rank placement[assign[q, j]] (self-traffic kept).  Returns (order,
    send_counts): units grouped by owner rank (stable), and units per rank."""
    import torch
    owner = placement.index_select(0, assign.reshape(-1).long())
    order = torch.argsort(owner, stable=True)
    return order, torch.bincount(owner, minlength=world)


def run_pipeline_distributed(ctx, d_q, p, fanout: int, placement, world: int, with_vectors: bool = True,
                             group=None):
    """run_pipeline (simulator.cpp:250-337), cluster-sharded across ranks.

    ctx holds the centroids (set_centroids) and the partitions of the clusters
    placed on this rank; d_q is this rank's query batch (torch, nq x dim, on
    ctx's device); placement a device tensor cluster -> rank.  Returns torch
    tensors (ids nq x k, dists, counts, vectors nq x k x dim or None) and the
    batch's visited_total -- identical to a one-GPU run_pipeline over the same
    queries with every cluster resident (tests, bench --mode cluster)."""
    import torch
    import torch.distributed as dist
    dev = d_q.device
    nq, dim = int(d_q.shape[0]), int(d_q.shape[1])
    k, c = int(p.k), int(fanout)
    cs = torch.cuda.ExternalStream(ctx.stream, device=dev)
    with torch.cuda.stream(cs):  # torch ops and library calls share one stream
        assign = torch.empty((nq, c), dtype=torch.int32, device=dev)
        ctx.assign_top_c_device(d_q.data_ptr(), nq, dim, c, assign.data_ptr())
        order, send_counts = route_to_owners(assign, placement, world)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=group)
        sc, rc = send_counts.tolist(), recv_counts.tolist()
        nrecv = int(sum(rc))
        # dispatch: each routed unit carries its query vector and cluster id
        q_send = d_q.index_select(0, torch.div(order, c, rounding_mode="floor"))
        cl_send = assign.reshape(-1).index_select(0, order)
        q_recv = torch.empty((nrecv, dim), dtype=d_q.dtype, device=dev)
        cl_recv = torch.empty((nrecv,), dtype=torch.int32, device=dev)
        dist.all_to_all_single(q_recv, q_send, rc, sc, group=group)
        dist.all_to_all_single(cl_recv, cl_send, rc, sc, group=group)
        # owner: search every received unit in its resident partition
        r_ids = torch.empty((nrecv, k), dtype=torch.int32, device=dev)
        r_d = torch.empty((nrecv, k), dtype=torch.float32, device=dev)
        r_cnt = torch.empty((nrecv,), dtype=torch.int32, device=dev)
        r_vis = torch.empty((nrecv,), dtype=torch.int64, device=dev)
        if nrecv:
            uq = torch.arange(nrecv, dtype=torch.int32, device=dev)
            ctx.search_units_device(q_recv.data_ptr(), nrecv, dim, uq.data_ptr(), cl_recv.data_ptr(), nrecv, p,
                                    r_ids.data_ptr(), r_d.data_ptr(), r_cnt.data_ptr(), r_vis.data_ptr())
        r_vec = None
        if with_vectors:
            r_vec = torch.zeros((nrecv, k, dim), dtype=torch.float32, device=dev)
            if nrecv:
                ctx.gather_vectors_device(r_ids.data_ptr(), r_cnt.data_ptr(), nrecv, k, r_vec.data_ptr())
        # combine all-to-all: results back to the origin, then un-permute
        nu = nq * c

        def back(t, shape):
            out = torch.empty(shape, dtype=t.dtype, device=dev)
            dist.all_to_all_single(out, t, sc, rc, group=group)
            u = torch.empty_like(out)
            u[order] = out
            return u

        u_ids = back(r_ids, (nu, k))
        u_d = back(r_d, (nu, k))
        u_cnt = back(r_cnt, (nu,))
        u_vis = back(r_vis, (nu,))
        ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
        dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
        counts = torch.empty((nq,), dtype=torch.int32, device=dev)
        ctx.combine_results_device(nq, c, u_ids.data_ptr(), u_d.data_ptr(), u_cnt.data_ptr(), k, k,
                                   ids.data_ptr(), dists.data_ptr(), counts.data_ptr())
        vectors = None
        if with_vectors:
            u_vec = back(r_vec, (nu, k, dim)).view(nq, c * k, dim)
            # each final hit comes from exactly one partial slot (clusters are disjoint)
            part_ids = u_ids.view(nq, c * k)
            slot_ok = (torch.arange(k, device=dev)[None, None, :] < u_cnt.view(nq, c, 1)).view(nq, c * k)
            hit_ok = torch.arange(k, device=dev)[None, :] < counts[:, None]
            match = (part_ids[:, None, :] == ids[:, :, None]) & slot_ok[:, None, :]
            src = match.int().argmax(dim=2)
            vectors = torch.gather(u_vec, 1, src[:, :, None].expand(nq, k, dim))
            vectors = torch.where(hit_ok[:, :, None], vectors, torch.zeros_like(vectors))
        visited_total = int(u_vis.sum().item())
    return ids, dists, counts, vectors, visited_total


def run_pipeline_distributed_mb(ctx, comm_ctx, d_q, p, fanout: int, placement, world: int,
                                microbatches: int = 2, with_vectors: bool = True, group=None,
                                timeline: bool = False, rank: int = 0):
    """run_pipeline_distributed with the reference's microbatch schedule made
    real (simulator.cpp:295-297 two_microbatch, replay_schedule :71-168):
    per microbatch kmeans (assign + route) and search run on ctx's stream --
    the compute lane -- while dispatch and combine (the all-to-alls, the
    un-permute and the combine kernel, on comm_ctx's stream) run on the comm
    lane, so microbatch i+1's dispatch overlaps microbatch i's search and
    microbatch i's combine overlaps i+1's search.  comm_ctx is a second
    context on the same device (its stream and kernels only; no index).
    Returns (ids, dists, counts, vectors, visited_total, intervals): the
    intervals are the reference's Timeline fields measured with CUDA events
    (None unless timeline=True) and satisfy check_timeline."""
    import torch
    import torch.distributed as dist
    dev = d_q.device
    nq, dim = int(d_q.shape[0]), int(d_q.shape[1])
    k, c = int(p.k), int(fanout)
    m = max(1, min(int(microbatches), nq))
    edges = [nq * i // m for i in range(m + 1)]
    cs = torch.cuda.ExternalStream(ctx.stream, device=dev)
    xs = torch.cuda.ExternalStream(comm_ctx.stream, device=dev)

    def ev():
        return torch.cuda.Event(enable_timing=timeline)

    marks = {}
    with torch.cuda.stream(xs):  # written on the comm lane (combine)
        ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
        dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
        counts = torch.empty((nq,), dtype=torch.int32, device=dev)
        vectors = torch.zeros((nq, k, dim), dtype=torch.float32, device=dev) if with_vectors else None
    with torch.cuda.stream(cs):  # written on the compute lane (kmeans)
        assign = torch.empty((nq, c), dtype=torch.int32, device=dev)
    plans = []
    # kmeans stage of every microbatch on the compute lane
    with torch.cuda.stream(cs):
        for i in range(m):
            q0, q1 = edges[i], edges[i + 1]
            e0, e1 = ev(), ev()
            e0.record(cs)
            ctx.assign_top_c_device(d_q[q0:q1].data_ptr(), q1 - q0, dim, c, assign[q0:q1].data_ptr())
            order, cnt = route_to_owners(assign[q0:q1], placement, world)
            e1.record(cs)
            marks[(i, "kmeans")] = (e0, e1)
            plans.append((order, cnt))
        send = torch.stack([pl[1] for pl in plans]).t().contiguous()  # world x m
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=group)  # sizes for every microbatch at once
        sc = send.t().tolist()
        rc = recv.t().tolist()
    # dispatch of every microbatch on the comm lane (NCCL runs collectives in
    # issue order, so all dispatches go ahead of the first combine)
    recvd = []
    for i in range(m):
        q0, q1 = edges[i], edges[i + 1]
        order = plans[i][0]
        with torch.cuda.stream(xs):
            xs.wait_event(marks[(i, "kmeans")][1])
            d0, d1 = ev(), ev()
            d0.record(xs)
            nrecv = int(sum(rc[i]))
            q_send = d_q[q0:q1].index_select(0, torch.div(order, c, rounding_mode="floor"))
            cl_send = assign[q0:q1].reshape(-1).index_select(0, order)
            q_recv = torch.empty((nrecv, dim), dtype=d_q.dtype, device=dev)
            cl_recv = torch.empty((nrecv,), dtype=torch.int32, device=dev)
            dist.all_to_all_single(q_recv, q_send, rc[i], sc[i], group=group)
            dist.all_to_all_single(cl_recv, cl_send, rc[i], sc[i], group=group)
            d1.record(xs)
            marks[(i, "dispatch")] = (d0, d1)
            recvd.append((q_recv, cl_recv, nrecv))
    # every search is issued before the first combine: combine_results_device
    # synchronizes the comm stream (unsorted-partial check), which must not
    # hold back the next microbatch's search
    results = []
    for i in range(m):
        q_recv, cl_recv, nrecv = recvd[i]
        with torch.cuda.stream(cs):  # search on the compute lane
            cs.wait_event(marks[(i, "dispatch")][1])
            s0, s1 = ev(), ev()
            s0.record(cs)
            r_ids = torch.empty((nrecv, k), dtype=torch.int32, device=dev)
            r_d = torch.empty((nrecv, k), dtype=torch.float32, device=dev)
            r_cnt = torch.empty((nrecv,), dtype=torch.int32, device=dev)
            r_vis = torch.empty((nrecv,), dtype=torch.int64, device=dev)
            r_vec = torch.zeros((nrecv, k, dim), dtype=torch.float32, device=dev) if with_vectors else None
            if nrecv:
                uq = torch.arange(nrecv, dtype=torch.int32, device=dev)
                ctx.search_units_device(q_recv.data_ptr(), nrecv, dim, uq.data_ptr(), cl_recv.data_ptr(), nrecv, p,
                                        r_ids.data_ptr(), r_d.data_ptr(), r_cnt.data_ptr(), r_vis.data_ptr())
                if with_vectors:
                    ctx.gather_vectors_device(r_ids.data_ptr(), r_cnt.data_ptr(), nrecv, k, r_vec.data_ptr())
            s1.record(cs)
            marks[(i, "search")] = (s0, s1)
            results.append((r_ids, r_d, r_cnt, r_vis, r_vec))
    with torch.cuda.stream(xs):  # the comm lane owns every later read of it
        visited_total = torch.zeros((), dtype=torch.int64, device=dev)
    for i in range(m):
        q0, q1 = edges[i], edges[i + 1]
        n = q1 - q0
        order = plans[i][0]
        r_ids, r_d, r_cnt, r_vis, r_vec = results[i]
        with torch.cuda.stream(xs):  # combine on the comm lane
            xs.wait_event(marks[(i, "search")][1])
            c0, c1 = ev(), ev()
            c0.record(xs)
            nu = n * c

            def back(t, shape):
                out = torch.empty(shape, dtype=t.dtype, device=dev)
                dist.all_to_all_single(out, t, sc[i], rc[i], group=group)
                u = torch.empty_like(out)
                u[order] = out
                return u

            u_ids = back(r_ids, (nu, k))
            u_d = back(r_d, (nu, k))
            u_cnt = back(r_cnt, (nu,))
            u_vis = back(r_vis, (nu,))
            comm_ctx.combine_results_device(n, c, u_ids.data_ptr(), u_d.data_ptr(), u_cnt.data_ptr(), k, k,
                                            ids[q0:q1].data_ptr(), dists[q0:q1].data_ptr(), counts[q0:q1].data_ptr())
            if with_vectors:
                u_vec = back(r_vec, (nu, k, dim)).view(n, c * k, dim)
                part_ids = u_ids.view(n, c * k)
                slot_ok = (torch.arange(k, device=dev)[None, None, :] < u_cnt.view(n, c, 1)).view(n, c * k)
                hit_ok = torch.arange(k, device=dev)[None, :] < counts[q0:q1, None]
                match = (part_ids[:, None, :] == ids[q0:q1, :, None]) & slot_ok[:, None, :]
                src = match.int().argmax(dim=2)
                got = torch.gather(u_vec, 1, src[:, :, None].expand(n, k, dim))
                vectors[q0:q1] = torch.where(hit_ok[:, :, None], got, torch.zeros_like(got))
            visited_total += u_vis.sum()  # stream-ordered on the comm lane
            c1.record(xs)
            marks[(i, "combine")] = (c0, c1)
    torch.cuda.synchronize(dev)
    visited_total = int(visited_total.item())
    intervals = None
    if timeline:
        base = marks[(0, "kmeans")][0]
        lane = {"kmeans": "compute", "search": "compute", "dispatch": "comm", "combine": "comm"}
        intervals = [{"rank": rank, "lane": lane[s], "stage": s, "microbatch": i,
                      "start": base.elapsed_time(a), "end": base.elapsed_time(b)}
                     for (i, s), (a, b) in sorted(marks.items())]
    return ids, dists, counts, vectors, visited_total, intervals
