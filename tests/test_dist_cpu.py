"""CPU: the N>1 host-side logic of the sharded mode, world_size 2 over gloo.

Covers the shard rule (matches dvsg_shard_init's S = ceil(n/R)), the IPC
handle exchange over torch.distributed, and the per-rank setup sequence with
a recording stand-in for the GPU context (no device work here)."""
import os
import socket

import numpy as np
import pytest

from paper_2512_02278_b200.dist import owner_of, setup_sharded, shard_range, split_even


def test_shard_range_covers_ids_exactly_once():
    for n in (1, 7, 8, 1000, 1_000_003):
        for R in (1, 2, 3, 4, 8):
            seen = np.zeros(n, np.int32)
            for r in range(R):
                lo, hi = shard_range(n, R, r)
                seen[lo:hi] += 1
                for v in {lo, hi - 1} if hi > lo else set():
                    assert owner_of(v, n, R) == r
            assert (seen == 1).all()
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_split_even():
    parts = split_even(10, 3)
    assert parts[0][0] == 0 and parts[-1][1] == 10
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


class FakeCtx:
    """Records the calls setup_sharded makes on a dvs.Context."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []

    def shard_init(self, nranks, rank, shard_vectors, n_total, adjacency, entry_order, gids):
        self.calls.append(("init", nranks, rank, shard_vectors.shape[0], n_total))

    def shard_export(self):
        return bytes([self.rank]) * 64

    def shard_connect(self, handles):
        self.calls.append(("connect", [h[0] for h in handles]))


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 1001
        data = np.zeros((n, 4), np.float32)
        adj = np.zeros((n, 2), np.uint32)
        eo = np.arange(n, dtype=np.uint32)
        ctx = FakeCtx(rank)
        lo, hi = setup_sharded(ctx, rank, world, data, adj, eo)
        q.put((rank, lo, hi, ctx.calls))
    finally:
        dist.destroy_process_group()


def test_setup_sharded_two_ranks_gloo():
    import multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    procs = [ctxm.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r, lo, hi, calls = q.get(timeout=120)
        out[r] = (lo, hi, calls)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][:2] == (0, 501) and out[1][:2] == (501, 1001)
    for r in (0, 1):
        calls = out[r][2]
        assert calls[0] == ("init", 2, r, 501 if r == 0 else 500, 1001)
        assert calls[1] == ("connect", [0, 1])  # every rank's handle, in rank order


def test_route_to_owners_matches_router_semantics():
    """router.cpp:52-79 (design A dispatch): every (query, slot) unit goes to
    placement[cluster]; units grouped by owner rank, stable within a rank."""
    import torch
    from paper_2512_02278_b200.dist import route_to_owners
    rng = np.random.default_rng(3)
    nq, fanout, clusters, world = 257, 3, 12, 4
    assign = torch.from_numpy(rng.integers(0, clusters, size=(nq, fanout)).astype(np.int32))
    placement = torch.from_numpy((np.arange(clusters) % world).astype(np.int64))  # place_clusters, router.cpp:38-41
    order, counts = route_to_owners(assign, placement, world)
    owner = (assign.numpy().reshape(-1) % world)
    want = [u for r in range(world) for u in range(nq * fanout) if owner[u] == r]
    assert order.tolist() == want
    assert counts.tolist() == [int((owner == r).sum()) for r in range(world)]
