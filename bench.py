#!/usr/bin/env python
"""bench.py -- QPS of the batched graph search at recall@10 >= 0.95 on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dvsg|reference]

One step = one run_pipeline pass (simulator.cpp:245-337 functional part:
assign -> route -> K1 beam search -> combine -> attach hit vectors) over one
batch of 100k synthetic SIFT-like queries against the 1M x 128 kNN-32 graph
(BASELINE.json configs[1] at N=1: the graph in one partition; I=6, w=64,
entry=64, k=10 calibrated to recall@10 >= 0.95 on this data).

`value`  : device-resident queries, CUDA events on the library's stream, L2
           flushed (256 MiB write) before every step, max over ranks.
`e2e`    : the same step through the public host-buffer call
           (dvsg_run_pipeline: pinned host queries in, ids/dists/counts/hit
           vectors out; H2D and D2H inside the timed region).
`roofline`: K1 algorithmic bytes (visited*4d + expanded*4*d_g + 4d per unit,
           SURVEY 8d) / K1 event time, against MEASURED_PEAKS.json hbm_gbs.
`cpu_baseline`: the reference's own run_pipeline (oracle/_ref, compiled from
           /root/reference sources) on a bounded query sample, all host cores.

N > 1 (torchrun, one rank per GPU): each rank holds a full replica of the
index and searches its own 100k-query batch ("replicas": weak scaling); the
sharded frontier-exchange mode is not in this round.
`--impl reference`: rank 0 times the reference CPU path (same config and
metric), other ranks exit 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback (used only without MEASURED_PEAKS.json)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["dvsg", "reference"], default="dvsg")
    ap.add_argument("--n", "--rows", dest="n", type=int, default=1_000_000)
    ap.add_argument("--nq", type=int, default=100_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--rank-latent", type=int, default=16)
    ap.add_argument("--degree", type=int, default=32)
    ap.add_argument("--iterations", type=int, default=6)
    ap.add_argument("--beam", type=int, default=64)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--entry", type=int, default=64)
    ap.add_argument("--accum", choices=["f32", "f64"], default="f32")
    ap.add_argument("--recall-sample", type=int, default=2000)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cache", default="/tmp/dvsg_bench_cache")
    ap.add_argument("--mode", choices=["auto", "replica", "sharded"], default="auto",
                    help="N>1 layout: full index per GPU, or node-sharded vectors with an NVLink "
                         "frontier exchange (auto = replica headline, sharded measured beside it)")
    ap.add_argument("--timeline-out", default=None,
                    help="write the measured e2e pipeline timeline (intervals JSON) here")
    ap.add_argument("--no-nccl-baseline", action="store_true",
                    help="skip the NCCL-exchange baseline measured beside the sharded mode at N>1")
    ap.add_argument("--exchange", choices=["bulk", "fused", "nccl"], default="bulk",
                    help="sharded-mode exchange: bulk-synchronous phases (xchg_kernel.cu) or "
                         "per-CTA round trips (shard_kernel.cu), or the bulk protocol over "
                         "host-driven NCCL send/recv (the measured baseline)")
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class Clocks:
    """nvidia-smi sampler over the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (getattr(self, "out", "") or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
def workload(args, rank: int, ctx):
    """Data + queries + index (graph cached by config under args.cache)."""
    from paper_2512_02278_b200 import synth
    from paper_2512_02278_b200.api import BuiltIndex, GraphIndex, compute_entry_order
    t0 = time.time()
    data = synth.sift_like(args.n, args.dim, args.rank_latent, seed=1)
    queries = synth.sift_like_queries(args.nq, args.dim, args.rank_latent, data_seed=1, seed=2 + rank)
    os.makedirs(args.cache, exist_ok=True)
    tag = f"n{args.n}_d{args.dim}_r{args.rank_latent}_g{args.degree}"
    adj_path = os.path.join(args.cache, f"adj_{tag}.npy")
    eo_path = os.path.join(args.cache, f"eo_{tag}.npy")
    if os.path.isfile(adj_path) and os.path.isfile(eo_path):
        adj, eo = np.load(adj_path), np.load(eo_path)
    else:
        adj = ctx.build_graph(data, args.degree)       # K6, exact on integer data
        eo = compute_entry_order(data)                 # graph_index.cpp:21-44
        tmp = adj_path + f".{os.getpid()}.npy"
        np.save(tmp, adj)
        os.replace(tmp, adj_path)
        tmp = eo_path + f".{os.getpid()}.npy"
        np.save(tmp, eo)
        os.replace(tmp, eo_path)
    gids = np.arange(args.n, dtype=np.uint32)
    cents = data.mean(0, dtype=np.float64).astype(np.float32)[None, :]
    index = BuiltIndex(cents, np.zeros(1, np.uint32), 1, args.degree,
                       [GraphIndex(data, gids, args.degree, adj, eo)])
    log(f"[bench] workload ready in {time.time() - t0:.1f}s")
    return data, queries, index


def recall(data, queries, ids, counts, k):
    from paper_2512_02278_b200 import synth
    truth = synth.brute_force_gt(data, queries, k)
    return synth.recall_at_k(ids, counts, truth, k)


# ---------------------------------------------------------------------------
def reference_arm(args, data, queries, index, nthreads, seconds, min_q=64):
    """Time the reference's own run_pipeline on a bounded sample."""
    from oracle.oracle import Oracle, Ref, have_ref
    kind = "reference" if have_ref() else "port"
    g = index.graphs[0]
    if kind == "reference":
        ref = Ref()
        ridx = ref.index_from_arrays(index.centroids, index.cluster_to_rank, 1, args.degree,
                                     [(g.vectors, g.adjacency, g.global_ids)])

        def run(qs):
            return ridx.run_pipeline(qs, args.iterations, args.beam, args.k, args.entry, 1, 1,
                                     nthreads=nthreads, with_vectors=True)
    else:
        o = Oracle()

        def run(qs):
            return o.run_pipeline(index, qs, args.iterations, args.beam, args.k, args.entry, 1, 1,
                                  nthreads=nthreads, with_vectors=True)
    # size the sample so one pass is ~`seconds` of CPU wall time
    probe = queries[:max(min_q, 2 * nthreads)]
    t0 = time.perf_counter()
    run(probe)
    dt = time.perf_counter() - t0
    per_q = dt / probe.shape[0]
    n = int(min(queries.shape[0], max(probe.shape[0], seconds / max(per_q, 1e-9))))
    return kind, run, n


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference_impl(args, world, rank):
    """--impl reference: rank 0 times the reference CPU implementation."""
    if rank != 0:
        return
    import paper_2512_02278_b200 as dvs
    ctx = dvs.Context(0)  # setup only: builds the shared graph if not cached
    data, queries, index = workload(args, 0, ctx)
    ctx.close()
    nthreads = os.cpu_count() or 1
    kind, run, n = reference_arm(args, data, queries, index, nthreads, args.cpu_seconds)
    sample = queries[:n]
    run(sample[: min(n, 4 * nthreads)])  # warm caches / page in the index
    times = []
    res = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = run(sample)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    qps = n * args.steps / total
    rec = recall(data, sample[: min(n, args.recall_sample)], res[0], res[2], args.k)
    line = {
        "impl": "reference", "metric": "QPS at recall@10>=0.95", "value": qps, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world, rec),
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": nthreads, "kind": kind,
                         "sample": f"{n} of the {args.nq} queries per step, run_pipeline C=1 "
                                   f"(simulator.cpp:245-366) in {nthreads} threads",
                         "cpu_model": cpu_model()},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def timeline_summary(dvs, tl, args):
    """Measured copy/compute timeline of the last e2e step:
    validated with check_timeline (simulator.cpp:170-217 rules), with the
    time both lanes were busy (the overlap the microbatch pipeline buys)."""
    if not tl:
        return None
    if getattr(args, "timeline_out", None):
        with open(args.timeline_out, "w") as f:
            json.dump(tl, f, indent=1)

    def union(ivs):
        out = []
        for a, b in sorted((iv["start"], iv["end"]) for iv in ivs):
            if out and a <= out[-1][1]:
                out[-1][1] = max(out[-1][1], b)
            else:
                out.append([a, b])
        return out

    comp = union([iv for iv in tl if iv["lane"] == "compute"])
    comm = union([iv for iv in tl if iv["lane"] == "comm"])
    both = sum(max(0.0, min(b1, b2) - max(a1, a2)) for a1, b1 in comp for a2, b2 in comm)
    return {"microbatches": 1 + max(iv["microbatch"] for iv in tl), "check_timeline": dvs.check_timeline(tl) or "ok",
            "makespan_ms": max(iv["end"] for iv in tl), "compute_busy_ms": sum(b - a for a, b in comp),
            "copy_busy_ms": sum(b - a for a, b in comm), "overlapped_ms": both,
            "lanes": "comm = h2d + d2h on the copy stream, compute = run_pipeline kernels"}


def workload_config(args, world, rec):
    return {
        "workload": "BASELINE configs[1] at N=1: SIFT-like synthetic 1M x 128 (integer-valued f32, "
                    "rank-16 latent), exact kNN-32 graph in 1 partition, 100k-query batch per GPU, "
                    "top-10, beam 64, I=6, entry 64",
        "n": args.n, "dim": args.dim, "degree": args.degree, "queries_per_step_per_gpu": args.nq,
        "iterations": args.iterations, "beam_width": args.beam, "k": args.k,
        "entry_count": args.entry, "partitions": 1, "accum": args.accum,
        "recall_at_10": None if rec is None else round(rec, 4),
        "l2": "256 MiB buffer written before every timed step",
        "parallelism": (f"node-sharded x{world}: vectors split by id range, adjacency replicated, "
                        f"{args.exchange} NVLink peer-store frontier exchange" if getattr(args, "_sharded", False)
                        else (f"replicas x{world}" if world > 1 else "single GPU")),
        "step": ("node-sharded search (ids + dists)" if getattr(args, "_sharded", False)
                 else "run_pipeline: assign + route + K1 + combine + hit vectors"),
    }


# ---------------------------------------------------------------------------
def measure_sharded(args, dvs, torch, dist, local, rank, world, data, queries, index, p, ids_ref,
                    cnt_ref, flush, dev):
    """K timed steps of the node-sharded search (vectors split across the N
    GPUs, NVLink frontier exchange, --exchange); ids must equal the replica run's."""
    from paper_2512_02278_b200.dist import prepare_step, setup_sharded
    g0 = index.graphs[0]
    ctx = dvs.Context(local)
    try:
        return _measure_sharded(ctx, args, torch, dist, rank, world, data, queries, g0, p, ids_ref,
                                cnt_ref, flush, dev, setup_sharded, prepare_step)
    finally:
        ctx.close()


def _measure_sharded(ctx, args, torch, dist, rank, world, data, queries, g0, p, ids_ref, cnt_ref, flush,
                     dev, setup_sharded, prepare_step):
    ctx.set_shard_exchange(args.exchange)
    setup_sharded(ctx, rank, world, data, g0.adjacency, g0.entry_order, g0.global_ids)
    if args.exchange == "nccl":
        from paper_2512_02278_b200.dist import connect_nccl
        connect_nccl(ctx, rank)
    nq, dim, k = args.nq, args.dim, args.k
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    d_q = torch.from_numpy(queries).to(dev)
    d_ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    d_dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    d_counts = torch.empty((nq,), dtype=torch.int32, device=dev)
    d_vis = torch.empty((nq,), dtype=torch.int64, device=dev)

    def run():
        ctx.search_sharded_device(d_q.data_ptr(), nq, dim, p, d_ids.data_ptr(), d_dists.data_ptr(),
                                  d_counts.data_ptr(), d_vis.data_ptr())

    for _ in range(max(1, args.warmup)):
        prepare_step(ctx, dist.barrier)
        run()
        ctx.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        prepare_step(ctx, dist.barrier)
        ev0[i].record(stream)
        run()
        ev1[i].record(stream)
        stream.synchronize()
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    same = torch.tensor([int(np.array_equal(d_ids.cpu().numpy().view(np.uint32), ids_ref) and
                             np.array_equal(d_counts.cpu().numpy().view(np.uint32), cnt_ref))],
                        dtype=torch.int32, device=dev)
    dist.all_reduce(same, op=dist.ReduceOp.MIN)
    st = ctx.last_search_stats() if args.exchange != "fused" else None
    tl_sum = None
    if args.exchange != "fused":
        # one more (untimed) step with timing on: measured step-kernel vs
        # barrier / NCCL-exchange intervals on the search stream
        ctx.set_timing(True)
        prepare_step(ctx, dist.barrier)
        run()
        ctx.synchronize()
        tl = ctx.last_sharded_timeline(rank)
        ctx.set_timing(False)
        if tl:
            span = max(iv["end"] for iv in tl) - min(iv["start"] for iv in tl)
            comp = sum(iv["end"] - iv["start"] for iv in tl if iv["lane"] == "compute")
            comm = sum(iv["end"] - iv["start"] for iv in tl if iv["lane"] == "comm")
            tl_sum = {"rank": rank, "intervals": len(tl), "span_ms": span, "step_kernels_ms": comp,
                      "barrier_or_exchange_ms": comm, "exchange_share": comm / span if span else None}
    ms = float(t[0])
    xch = None
    if st and st["units"]:
        # bulk protocol, per GPU and step: every remote candidate costs an 8 B
        # request out and an 8 B key back (a uniform id-range shard makes
        # (R-1)/R of the visited vectors remote), each query is copied once to
        # every other rank; HBM side: the same algorithmic bytes as K1
        vis_q = st["visited"] / st["units"]
        xbytes = nq * (vis_q * (world - 1) / world * 16 + (world - 1) * 4 * dim)
        alg = nq * (vis_q * 4 * dim + st["expanded"] / st["units"] * 4 * args.degree + 4 * dim)
        step_s = ms / args.steps / 1e3
        xch = {"bytes_per_step_per_gpu": xbytes, "achieved_gbs": xbytes / step_s / 1e9,
               "nvlink_peak_gbs_per_direction": 900.0, "frac": xbytes / step_s / 1e9 / 900.0,
               "hbm_alg_gbs_per_gpu": alg / step_s / 1e9, "visited_per_query": vis_q}
    return {"value": nq * world * args.steps / (ms / 1e3), "unit": "queries/s",
            "ms_per_step": ms / args.steps, "exchange_roofline": xch, "timeline_rank0": tl_sum,
            "layout": f"vectors node-sharded {world} ways (id ranges), adjacency replicated; " + (
                "bulk-synchronous NVLink peer-store frontier exchange (xchg_kernel.cu)" if args.exchange == "bulk"
                else "bulk protocol, host-driven ncclSend/ncclRecv exchange (baseline)" if args.exchange == "nccl"
                else "fused NVLink peer-store frontier exchange (shard_kernel.cu)"),
            "exchange": args.exchange,
            "ids_identical_to_replica_all_ranks": bool(same[0])}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_impl(args, world, rank)

    import torch
    import paper_2512_02278_b200 as dvs

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        # rank 0 must print exactly one JSON line on stdout: keep NCCL's version
        # banner (NCCL_DEBUG=VERSION/INFO) off stdout
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() in ("VERSION", ""):
            os.environ["NCCL_DEBUG"] = "WARN"
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    mode = args.mode
    if mode == "auto":
        # 1M x 128 (0.64 GB) fits one GPU: replicas are the QPS-optimal layout;
        # the node-sharded mode is measured beside it at N > 1 (DESIGN.md (e))
        mode = "replica"
    sharded = mode == "sharded"
    args._sharded = sharded

    ctx = dvs.Context(local)
    data, queries, index = workload(args, rank, ctx)
    g0 = index.graphs[0]
    if sharded:
        from paper_2512_02278_b200.dist import prepare_step, setup_sharded
        ctx.set_shard_exchange(args.exchange)
        setup_sharded(ctx, rank, world, data, g0.adjacency, g0.entry_order, g0.global_ids)
        if args.exchange == "nccl":
            from paper_2512_02278_b200.dist import connect_nccl
            connect_nccl(ctx, rank)
    else:
        ctx.load_index(index)
    p = dvs.SearchParams(args.iterations, args.beam, args.k, args.entry, accum=args.accum)
    nq, dim, k = args.nq, args.dim, args.k
    dev = torch.device("cuda", local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    d_q = torch.from_numpy(queries).to(dev)
    d_ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    d_dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    d_counts = torch.empty((nq,), dtype=torch.int32, device=dev)
    d_vecs = torch.empty((nq, k, dim), dtype=torch.float32, device=dev)
    d_vis = torch.empty((nq,), dtype=torch.int64, device=dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    torch.cuda.synchronize()

    def pre_step():  # untimed: the sharded arenas must be reset on every rank first
        if sharded:
            prepare_step(ctx, dist.barrier if dist else (lambda: None))

    def step():
        if sharded:
            ctx.search_sharded_device(d_q.data_ptr(), nq, dim, p, d_ids.data_ptr(),
                                      d_dists.data_ptr(), d_counts.data_ptr(), d_vis.data_ptr())
        else:
            ctx.run_pipeline_device(d_q.data_ptr(), nq, dim, p, 1, d_ids.data_ptr(),
                                    d_dists.data_ptr(), d_counts.data_ptr(), d_vecs.data_ptr())

    ctx.set_timing(True)
    for _ in range(args.warmup):
        pre_step()
        step()
        ctx.synchronize()

    # ---- timed region: K steps, L2 flushed before each -------------------------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k1_ms, vis_tot, exp_tot, units_tot = 0.0, 0, 0, 0
    launches0 = ctx.kernel_launches()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            pre_step()
            starts[i].record(stream)
            step()
            ends[i].record(stream)
            st = ctx.last_search_stats()      # syncs the stream
            k1_ms += ctx.last_timings()["search_ms"]
            vis_tot += st["visited"]
            exp_tot += st["expanded"]
            units_tot += st["units"]
        torch.cuda.synchronize()
    launches = ctx.kernel_launches() - launches0
    step_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t_local = torch.tensor([step_ms, k1_ms], dtype=torch.float64, device=dev)
    if dist:
        dist.barrier()
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms, k1_max_ms = float(t_local[0]), float(t_local[1])

    # ---- parity sample + recall (outside timing) ------------------------------------
    ids_h = d_ids.cpu().numpy().view(np.uint32)
    cnt_h = d_counts.cpu().numpy().view(np.uint32)
    rec = None
    shard_parity = None
    if rank == 0:
        s = min(args.recall_sample, nq)
        rec = recall(data, queries[:s], ids_h[:s], cnt_h[:s], k)
        if sharded:  # the sharded traversal must equal the unsharded one exactly
            ref_ctx = dvs.Context(local)
            ref_ctx.load_index(index)
            ri, rd, rc, rv = ref_ctx.beam_search(0, queries[:s], p)
            vis_h = d_vis.cpu().numpy()[:s]
            shard_parity = {"queries": s,
                            "ids_identical": bool(np.array_equal(ri, ids_h[:s]) and np.array_equal(rc, cnt_h[:s])),
                            "visited_identical": bool(np.array_equal(rv.astype(np.int64), vis_h))}
            ref_ctx.close()

    # ---- e2e through the public host-buffer call ------------------------------------
    e2e = None
    if not args.no_e2e and sharded:
        # host queries in (pinned H2D), sharded search, ids/dists/counts out (D2H)
        hq = torch.from_numpy(queries).pin_memory()
        h_ids = torch.empty((nq, k), dtype=torch.int32, pin_memory=True)
        h_dists = torch.empty((nq, k), dtype=torch.float32, pin_memory=True)
        h_counts = torch.empty((nq,), dtype=torch.int32, pin_memory=True)
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            pre_step()
            with torch.cuda.stream(stream):
                ev0[i].record(stream)
                d_q.copy_(hq, non_blocking=True)
                step()
                h_ids.copy_(d_ids, non_blocking=True)
                h_dists.copy_(d_dists, non_blocking=True)
                h_counts.copy_(d_counts, non_blocking=True)
                ev1[i].record(stream)
            stream.synchronize()
        e_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        assert np.array_equal(h_ids.numpy().view(np.uint32), ids_h), "e2e and device paths disagree"
        e2e = {"value": nq * world * args.steps / (float(e_ms[0]) / 1e3), "unit": "queries/s",
               "h2d_bytes_per_step": int(hq.numel() * 4),
               "d2h_bytes_per_step": int((h_ids.numel() + h_dists.numel() + h_counts.numel()) * 4),
               "ms_per_step": float(e_ms[0]) / args.steps,
               "note": "sharded mode returns ids + dists (hit vectors stay on their owner GPUs)"}
    elif not args.no_e2e:
        keep = []

        def pin(shape, dt):
            t = torch.empty(shape, dtype=dt, pin_memory=True)
            keep.append(t)
            return t.numpy()

        hq = pin((nq, dim), torch.float32)
        hq[:] = queries
        out = {"ids": pin((nq, k), torch.int32).view(np.uint32), "dists": pin((nq, k), torch.float32),
               "counts": pin((nq,), torch.int32).view(np.uint32), "vectors": pin((nq, k, dim), torch.float32)}
        ctx.run_pipeline(hq, p, 1, 1, 0, True, out)  # warm
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            ev0[i].record(stream)
            ctx.run_pipeline(hq, p, 1, 1, 0, True, out)
            ev1[i].record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        assert np.array_equal(out["ids"], ids_h) and np.array_equal(out["counts"], cnt_h), \
            "host-buffer and device-pointer paths disagree"
        h2d = hq.nbytes
        d2h = out["ids"].nbytes + out["dists"].nbytes + out["counts"].nbytes + out["vectors"].nbytes + 4 + 8
        e2e = {"value": nq * world * args.steps / (float(e_ms[0]) / 1e3), "unit": "queries/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": float(e_ms[0]) / args.steps,
               "timeline": timeline_summary(dvs, ctx.last_pipeline_timeline(rank), args)}

    # ---- node-sharded mode beside the replica headline (N > 1) -------------------------
    sharded_side = None
    if world > 1 and not sharded and args.mode == "auto":
        # side measurements must not cost the headline line: a failure (raised
        # on every rank alike, e.g. out of memory) is reported in the JSON
        try:
            sharded_side = measure_sharded(args, dvs, torch, dist, local, rank, world, data, queries,
                                           index, p, ids_h, cnt_h, flush, dev)
        except Exception as e:  # noqa: BLE001
            sharded_side = {"error": f"{type(e).__name__}: {e}"}
        if "error" not in sharded_side and args.exchange != "nccl" and not args.no_nccl_baseline:
            # the same protocol over host-driven NCCL send/recv: the measured baseline
            ex = args.exchange
            args.exchange = "nccl"
            try:
                sharded_side["nccl_baseline"] = measure_sharded(
                    args, dvs, torch, dist, local, rank, world, data, queries, index, p, ids_h, cnt_h,
                    flush, dev)
            except Exception as e:  # noqa: BLE001
                sharded_side["nccl_baseline"] = {"error": f"{type(e).__name__}: {e}"}
            finally:
                args.exchange = ex

    # ---- CPU baseline (rank 0, N=1) ---------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            nthreads = os.cpu_count() or 1
            kind, run, n = reference_arm(args, data, queries, index, nthreads, args.cpu_seconds)
            t0 = time.perf_counter()
            r = run(queries[:n])
            dt = time.perf_counter() - t0
            same = np.array_equal(r[0], ids_h[:n]) and np.array_equal(r[2], cnt_h[:n])
            cpu = {"value": n / dt, "unit": "queries/s", "cores": nthreads, "kind": kind,
                   "sample": f"first {n} of the {nq} step queries, run_pipeline C=1, {nthreads} threads",
                   "cpu_model": cpu_model(), "ids_identical_to_gpu": bool(same)}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "queries/s", "cores": 0, "kind": "unavailable",
                   "sample": f"failed: {ex}"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_kind = peaks()
    d4 = 4 * dim
    alg_bytes = vis_tot * d4 + exp_tot * 4 * args.degree + units_tot * d4
    achieved = alg_bytes / args.steps / (k1_max_ms / args.steps / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.isfile(tpath):
        try:
            tj = json.load(open(tpath))
            if tj.get("config_key") == f"n{args.n}_q{nq}_w{args.beam}_I{args.iterations}_{args.accum}":
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    value = nq * world * args.steps / (total_ms / 1e3)
    line = {
        "metric": "QPS at recall@10>=0.95", "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(args, world, rec),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": ("dvsg::search_kernel (K1)" if not getattr(args, "_sharded", False) else
                                ("dvsg::xg_step (bulk exchange)" if args.exchange == "bulk"
                                 else "dvsg::xg_step (bulk protocol, NCCL exchange)" if args.exchange == "nccl"
                                 else "dvsg::search_sharded_kernel (fused exchange)")),
                     "k1_ms_per_step": k1_max_ms / args.steps,
                     "alg_bytes_per_step": alg_bytes / args.steps,
                     "visited_per_query": vis_tot / max(units_tot, 1),
                     "expanded_per_query": exp_tot / max(units_tot, 1)},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "sharded_parity_vs_unsharded": shard_parity,
        "sharded_mode": sharded_side,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
