"""Cluster-sharded run_pipeline across GPUs (SURVEY 8e design A): parity with
the one-GPU pipeline over the same queries, then timing.

    torchrun --nproc-per-node N scripts/cluster_pipeline_mgpu.py [--rows 1000000]
        [--clusters-per-gpu 2] [--fanout 2] [--nq 100000] [--steps 3]

Every rank builds the same k-means index (synth.build_index, C = N x
clusters-per-gpu, cluster i on rank i mod N), keeps only its own clusters'
partitions for the distributed run, and checks ids / dists / counts / hit
vectors / visited_total against ctx.run_pipeline on a context holding every
cluster.  Rank 0 prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--clusters-per-gpu", type=int, default=2)
    ap.add_argument("--fanout", type=int, default=2)
    ap.add_argument("--nq", type=int, default=100_000)
    ap.add_argument("--check", type=int, default=20_000)
    ap.add_argument("--beam", type=int, default=64)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    import paper_2512_02278_b200 as dvs
    from paper_2512_02278_b200 import synth
    from paper_2512_02278_b200.dist import run_pipeline_distributed

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    t0 = time.time()
    data = synth.sift_like(a.rows, a.dim, 16, seed=1)
    clusters = world * a.clusters_per_gpu
    full = dvs.Context(local)
    index = synth.build_index(full, data, clusters, out_degree=32, ranks=world)
    full.load_index(index)
    ctx = dvs.Context(local)
    ctx.load_index(index, rank=rank)
    placement = torch.from_numpy(index.cluster_to_rank.astype(np.int64)).to(dev)
    queries = synth.sift_like_queries(a.nq, a.dim, 16, data_seed=1, seed=2 + rank)
    p = dvs.SearchParams(6, a.beam, 10, a.beam, accum="f32")
    setup_s = time.time() - t0

    # parity on the first `check` queries
    qc = queries[:a.check]
    want = full.run_pipeline(qc, p, a.fanout, world)
    ids, dists, counts, vecs, vt = run_pipeline_distributed(ctx, torch.from_numpy(qc).to(dev), p, a.fanout,
                                                            placement, world)
    ctx.synchronize()
    cnt = counts.cpu().numpy().view(np.uint32)
    ok = bool(np.array_equal(cnt, want.counts) and vt == want.visited_total)
    gi, gd, gv = ids.cpu().numpy().view(np.uint32), dists.cpu().numpy(), vecs.cpu().numpy()
    for q in range(qc.shape[0]):
        n = int(want.counts[q])
        if not (np.array_equal(gi[q, :n], want.ids[q, :n]) and np.array_equal(gd[q, :n], want.dists[q, :n])
                and np.array_equal(gv[q, :n], want.hit_vectors[q, :n])):
            ok = False
            break
    same = torch.tensor([int(ok)], device=dev)
    dist.all_reduce(same, op=dist.ReduceOp.MIN)

    # timing: the whole distributed pipeline on device-resident queries
    d_q = torch.from_numpy(queries).to(dev)
    for _ in range(2):
        run_pipeline_distributed(ctx, d_q, p, a.fanout, placement, world)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    e0.record(stream)
    vis = 0
    for _ in range(a.steps):
        vis += run_pipeline_distributed(ctx, d_q, p, a.fanout, placement, world)[4]
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # the library's own device-initiated exchange (cluster_xchg.cu: K3 dispatch
    # by peer stores, K1, results back by peer stores, K4 combine; no NCCL, no
    # host round trip)
    from paper_2512_02278_b200.dist import run_pipeline_cluster, setup_cluster_comm
    setup_cluster_comm(ctx, rank, world, a.nq, a.fanout, 10, True)
    nat = run_pipeline_cluster(ctx, torch.from_numpy(qc).to(dev), p, a.fanout)
    ctx.synchronize()
    ctx.cluster_comm_check()
    ok_n = bool(np.array_equal(nat[2].cpu().numpy().view(np.uint32), want.counts)
                and int(nat[4][0]) == want.visited_total
                and np.array_equal(nat[0].cpu().numpy().view(np.uint32), gi)
                and np.array_equal(nat[1].cpu().numpy(), gd) and np.array_equal(nat[3].cpu().numpy(), gv))
    same_n = torch.tensor([int(ok_n)], device=dev)
    dist.all_reduce(same_n, op=dist.ReduceOp.MIN)
    for _ in range(2):
        run_pipeline_cluster(ctx, d_q, p, a.fanout)
    ctx.synchronize()
    dist.barrier()
    n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0.record(stream)
    for _ in range(a.steps):
        run_pipeline_cluster(ctx, d_q, p, a.fanout)
    n1.record(stream)
    ctx.synchronize()
    ctx.cluster_comm_check()
    tn = torch.tensor([n0.elapsed_time(n1)], dtype=torch.float64, device=dev)
    dist.all_reduce(tn, op=dist.ReduceOp.MAX)
    native = {"qps": a.nq * world / (float(tn[0]) / a.steps / 1e3), "ms_per_step": float(tn[0]) / a.steps,
              "identical_to_one_gpu_pipeline_all_ranks": bool(same_n[0]),
              "exchange": "library peer-store dispatch/combine (cluster_xchg.cu), device-side unit counts"}
    # the microbatched schedule (dispatch / combine overlapping search)
    from paper_2512_02278_b200.dist import run_pipeline_distributed_mb
    cctx = dvs.Context(local)
    mb_out = {}
    for mbs in (2, 4):
        r = run_pipeline_distributed_mb(ctx, cctx, torch.from_numpy(qc).to(dev), p, a.fanout, placement, world,
                                        microbatches=mbs)
        ok_mb = bool(np.array_equal(r[2].cpu().numpy().view(np.uint32), want.counts) and r[4] == want.visited_total
                     and np.array_equal(r[0].cpu().numpy().view(np.uint32), gi) and np.array_equal(r[3].cpu().numpy(), gv))
        same_mb = torch.tensor([int(ok_mb)], device=dev)
        dist.all_reduce(same_mb, op=dist.ReduceOp.MIN)
        for _ in range(2):
            run_pipeline_distributed_mb(ctx, cctx, d_q, p, a.fanout, placement, world, microbatches=mbs)
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            run_pipeline_distributed_mb(ctx, cctx, d_q, p, a.fanout, placement, world, microbatches=mbs)
        tt = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        r = run_pipeline_distributed_mb(ctx, cctx, d_q, p, a.fanout, placement, world, microbatches=mbs,
                                        timeline=True, rank=rank)
        tl = r[5]
        msg = dvs.check_timeline(tl, stage_order={"kmeans": 0, "dispatch": 1, "search": 2, "combine": 3})
        span = max(iv["end"] for iv in tl)
        busy = {ln: sum(iv["end"] - iv["start"] for iv in tl if iv["lane"] == ln) for ln in ("compute", "comm")}
        mb_out[str(mbs)] = {"qps": a.nq * world / (float(tt[0]) / a.steps / 1e3),
                            "ms_per_step": float(tt[0]) / a.steps,
                            "identical_to_one_gpu_pipeline_all_ranks": bool(same_mb[0]),
                            "timeline_rank0": {"check_timeline": msg or "ok", "makespan_ms": span,
                                               "compute_busy_ms": busy["compute"], "comm_busy_ms": busy["comm"]}}
        if rank == 0 and mbs == 2:
            with open(os.environ.get("TIMELINE_OUT", "/dev/null"), "w") as f:
                json.dump(tl, f, indent=1)
    # recall on this rank's first 1000 queries
    truth = synth.brute_force_gt(data, queries[:1000], 10, ctx=full)
    rec = synth.recall_at_k(ids.cpu().numpy().view(np.uint32)[:1000], cnt[:1000], truth, 10)
    if rank == 0:
        ms = float(t[0]) / a.steps
        print(json.dumps({
            "mode": "cluster-sharded run_pipeline (design A)", "n_gpus": world, "n": a.rows, "dim": a.dim,
            "clusters": clusters, "fanout": a.fanout, "beam": a.beam, "queries_per_gpu": a.nq,
            "qps": a.nq * world / (ms / 1e3), "ms_per_step": ms, "visited_per_query": vis / a.steps / a.nq,
            "recall_at_10_rank0": round(rec, 4), "identical_to_one_gpu_pipeline_all_ranks": bool(same[0]),
            "checked_queries_per_rank": a.check, "setup_s": round(setup_s, 1),
            "microbatched": mb_out, "native_exchange": native,
            "exchange": "NCCL all_to_all_single (torch.distributed): dispatch of (query, cluster) units, "
                        "results + hit vectors back"}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
