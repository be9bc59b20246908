"""Multi-GPU plumbing for the node-sharded search (one process per GPU).

torch.distributed carries only control-plane data here: the 64-byte CUDA IPC
handles of each rank's comm arena (all_gather_object) and barriers.  The data
path -- candidate ids out, scored keys back -- is the fused kernel's own
NVLink peer stores (shard_kernel.cu), not a collective.

The shard rule is the C-ABI's (dvsg_shard_init): S = ceil(n / R), rank r owns
node ids [r*S, min(n, (r+1)*S)).
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
