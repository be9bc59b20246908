#!/usr/bin/env python
"""BASELINE configs[4] at N GPUs: batch x beam sweep on the 100M x 96 index
with every rank holding a full replica, then the same sweep node-sharded
(vectors split N ways, NVLink frontier exchange).  Every rank builds the same
graph once.  torchrun --nproc-per-node N scripts/cfg5_sweep_mgpu.py

One JSON line per (layout, beam, batch) on rank 0: whole-job QPS (max-over-
ranks time), recall@10 of rank 0's first 2000 queries, sharded ids identical
to the replica ids on every rank."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2512_02278_b200 as dvs  # noqa: E402
from paper_2512_02278_b200.dist import prepare_step, setup_sharded_resident  # noqa: E402

BEAMS = [(16, 24), (32, 14), (64, 10), (128, 8)]
BATCHES = [10_000, 100_000, 1_000_000]


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    dist.init_process_group("nccl", device_id=dev)
    args = bench.parse(["--nq", str(max(BATCHES))])
    ctx = dvs.Context(local)
    w = bench.build_workload(args, rank, ctx, dev)
    nq = max(BATCHES)
    b = bench.Bufs(torch, nq, 10, args.dim, dev, vectors=False)
    uq = torch.arange(nq, dtype=torch.int32, device=dev)
    up = torch.zeros(nq, dtype=torch.int32, device=dev)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    replica_ids = {}

    def timed(run, pre=lambda: None, reps=1):
        pre()
        run()
        ctx.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = 0.0
        for _ in range(reps):
            pre()
            torch.cuda.synchronize()
            e0.record(stream)
            run()
            e1.record(stream)
            ctx.synchronize()
            ms += e0.elapsed_time(e1)
        t = torch.tensor([ms / reps], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def report(layout, beam, iters, bs, ms, same=None):
        s = min(bs, w.gt.shape[0])
        ids = b.ids[:s].cpu().numpy().view(np.uint32)
        rec = bench.recall_at_k(ids, b.counts[:s].cpu().numpy(), w.gt[:s], 10)
        if rank == 0:
            line = {"layout": layout, "n_gpus": world, "n": args.n, "dim": args.dim, "beam": beam,
                    "iterations": iters, "batch_per_gpu": bs, "qps": bs * world / (ms / 1e3), "ms": ms,
                    "recall_at_10_rank0": round(rec, 4)}
            if same is not None:
                line["ids_identical_to_replica_all_ranks"] = same
            print(json.dumps(line), flush=True)

    for beam, iters in BEAMS:
        p = dvs.SearchParams(iters, beam, 10, beam, accum="f32")
        for bs in BATCHES:
            def run():
                ctx.search_units_device(w.queries.data_ptr(), bs, args.dim, uq.data_ptr(), up.data_ptr(), bs, p,
                                        b.ids.data_ptr(), b.dists.data_ptr(), b.counts.data_ptr(), b.vis.data_ptr())
            ms = timed(run, reps=max(1, min(10, 100_000 // bs)))
            replica_ids[(beam, bs)] = b.ids[:bs].cpu().numpy().copy()
            report("replicas", beam, iters, bs, ms)
    ctx.set_shard_exchange("bulk")
    setup_sharded_resident(ctx, rank, world)
    for beam, iters in BEAMS:
        p = dvs.SearchParams(iters, beam, 10, beam, accum="f32")
        for bs in BATCHES:
            def run():
                ctx.search_sharded_device(w.queries.data_ptr(), bs, args.dim, p, b.ids.data_ptr(),
                                          b.dists.data_ptr(), b.counts.data_ptr(), b.vis.data_ptr())
            ms = timed(run, pre=lambda: prepare_step(ctx, dist.barrier))
            same = torch.tensor([int(np.array_equal(b.ids[:bs].cpu().numpy(), replica_ids[(beam, bs)]))],
                                device=dev)
            dist.all_reduce(same, op=dist.ReduceOp.MIN)
            report("node-sharded", beam, iters, bs, ms, bool(same[0]))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
