#!/usr/bin/env python
"""bench.py -- QPS of the batched graph search at recall@10 >= 0.95 on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dvsg|reference]
                    [--workload cfg3|cfg1|cfg4]

Workloads (BASELINE.json configs):
  cfg3 (default) -- configs[2], the north-star config: Deep-like synthetic
        100M x 96 (integer-valued f32, rank-16 latent), degree-32 graph built
        on the GPU (cluster-restricted kNN + CAGRA-style rank pruning and
        reverse edges, paper_2512_02278_b200/ivf.py), 1M-query batch per GPU
        per step, top-10, beam 16, I=24, entry 16 (calibrated: recall@10
        >= 0.95 against brute-force ground truth on a 2,000-query sample).
  cfg1 -- configs[1] at N=1: 1M x 128, exact kNN-32 graph, 100k queries, I=6.
  cfg4 -- configs[3]: text-embedding-like 10M x 768 float, inner product,
        top-100, beam 256, I=16, 100k queries per GPU (f64 parity mode).

One step = one run_pipeline pass (simulator.cpp:245-337, functional part:
assign -> route -> K1 beam search -> combine -> attach hit vectors) over one
batch of queries.  At N > 1 (torchrun, one rank per GPU; `--gpus N` alone
self-launches torchrun) the headline is the north-star layout: the index's
vectors node-sharded across the N GPUs with the NVLink frontier exchange
(xchg_kernel.cu), each rank the origin of its own 1M-query batch (weak
scaling); full-replica searches are measured beside it.

`value`     : device-resident queries, CUDA events on the library's stream,
              max over ranks.  The 38 GB index is far larger than L2 and a
              256 MiB buffer is written before every step.
`e2e`       : the same step through the public host-buffer call
              (dvsg_run_pipeline): pinned host queries in, ids / dists /
              counts / hit vectors out, H2D and D2H inside the timed region;
              `e2e.pageable` repeats it with ordinary (pageable) numpy buffers.
`roofline`  : K1 algorithmic bytes (visited*4d + expanded*4*d_g + 4d per unit,
              SURVEY 8d) / K1 event time, against MEASURED_PEAKS.json hbm_gbs;
              `traffic` = ncu dram__bytes of K1 on the same config
              (profiles/k1_traffic.json; ncu cannot run inside the timed run).
`accum_modes`, `storage_u8`: side measurements of the same search (f64 /
              f32c accumulation; K1 on a byte copy of the rows) with their
              ids compared to the headline's.
`cpu_baseline`: the reference's own run_pipeline (oracle/_ref, compiled from
              /root/reference sources) on a bounded query sample, all host cores.
`--impl reference`: rank 0 times the reference's run_pipeline on the same
              graph (built on the GPU by a separate setup process that writes
              it to /dev/shm, so the timing process maps no libdvsg code).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback (used only without MEASURED_PEAKS.json)
METRIC = "QPS at recall@10>=0.95"

WORKLOADS = {
    "cfg3": dict(n=100_000_000, dim=96, nq=1_000_000, iterations=24, beam=16, entry=16, k=10, degree=32,
                 graph="ivf",
                 desc="BASELINE configs[2]: Deep-like synthetic 100M x 96 (integer-valued f32, rank-16 "
                      "latent), degree-32 graph (GPU-built: cluster-restricted kNN + CAGRA-style rank "
                      "pruning / reverse edges) in 1 partition, 1M-query batch per GPU, top-10, beam 16, "
                      "I=24, entry 16"),
    "cfg4": dict(n=10_000_000, dim=768, nq=100_000, iterations=16, beam=256, entry=256, k=100, degree=32,
                 graph="ivf", metric="ip", rank_latent=32, accum="f64",
                 desc="BASELINE configs[3]: text-embedding-like synthetic 10M x 768 (float, rank-32 latent, "
                      "L2-normalised), inner product, GPU-built degree-32 graph in 1 partition, 100k-query batch "
                      "per GPU, top-100, beam 256, I=16, entry 256, f64 parity-mode distances"),
    "cfg1": dict(n=1_000_000, dim=128, nq=100_000, iterations=6, beam=64, entry=64, k=10, degree=32,
                 graph="exact",
                 desc="BASELINE configs[1] at N=1: SIFT-like synthetic 1M x 128 (integer-valued f32, "
                      "rank-16 latent), exact kNN-32 graph in 1 partition, 100k-query batch per GPU, "
                      "top-10, beam 64, I=6, entry 64"),
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["dvsg", "reference", "reference-setup"], default="dvsg")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg3")
    ap.add_argument("--n", "--rows", dest="n", type=int, default=None)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--dim", type=int, default=None)
    ap.add_argument("--rank-latent", type=int, default=None)
    ap.add_argument("--degree", type=int, default=None)
    ap.add_argument("--iterations", type=int, default=None)
    ap.add_argument("--beam", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--entry", type=int, default=None)
    ap.add_argument("--accum", choices=["f32", "f64", "f32c"], default=None)
    ap.add_argument("--probe", type=int, default=8, help="cfg3 graph build: clusters probed per row")
    ap.add_argument("--cluster-size", type=int, default=1024, help="cfg3 graph build: rows per cluster")
    ap.add_argument("--keep", type=int, default=12,
                    help="cfg3 graph build: pruned forward edges per row (the rest are reverse edges)")
    ap.add_argument("--recall-sample", type=int, default=2000)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-step-seconds", type=float, default=5.0,
                    help="--impl reference: CPU seconds per timed step (sample size)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-modes", action="store_true", help="skip the f64 / f32c side measurement")
    ap.add_argument("--cache", default="/tmp/dvsg_bench_cache")
    ap.add_argument("--ref-out", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--mode", choices=["auto", "replica", "sharded"], default="auto",
                    help="N>1 layout: auto = node-sharded headline with replicas measured beside it")
    ap.add_argument("--timeline-out", default=None,
                    help="write the measured e2e pipeline timeline (intervals JSON) here")
    ap.add_argument("--no-nccl-baseline", action="store_true",
                    help="skip the NCCL-exchange baseline measured beside the sharded mode at N>1")
    ap.add_argument("--exchange", choices=["bulk", "fused", "nccl"], default="bulk",
                    help="sharded-mode exchange: bulk-synchronous phases (xchg_kernel.cu), per-CTA "
                         "round trips (shard_kernel.cu), or the bulk protocol over host-driven NCCL "
                         "send/recv (the measured baseline)")
    a = ap.parse_args(argv)
    wl = dict(dict(rank_latent=16, accum="f32", metric="l2"), **WORKLOADS[a.workload])
    for key, v in wl.items():
        if key in ("graph", "desc"):
            continue
        if getattr(a, key, None) is None:
            setattr(a, key, v)
    a.graph = wl["graph"]
    return a


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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def sha256_bytes(a: np.ndarray) -> str:
    h = hashlib.sha256()
    mv = memoryview(np.ascontiguousarray(a)).cast("B")
    step = 1 << 28
    for b in range(0, len(mv), step):
        h.update(mv[b:b + step])
    return h.hexdigest()


def recall_at_k(ids, counts, truth, k):
    """recall_at_k, topk.cpp:32-49, averaged over queries."""
    tot = 0.0
    for q in range(truth.shape[0]):
        tot += len(set(ids[q, :int(counts[q])].tolist()) & set(truth[q, :k].tolist())) / k
    return tot / truth.shape[0]


# ---------------------------------------------------------------------------
class Workload:
    """The index resident in `ctx`, this rank's queries on the device, and
    the ground truth of the recall sample."""

    def __init__(self):
        self.info = {}
        self.graph_sha256 = None


def build_cfg3(args, rank, ctx, dev, gt_rows=None):
    """Data, graph and queries of the cfg3 workload, all built on the GPU
    (setup, never timed)."""
    import torch
    from paper_2512_02278_b200 import ivf
    t0 = time.time()
    dpad = (args.dim + 3) // 4 * 4
    if args.metric == "ip":
        x = ivf.embedding_like_device(args.n, args.dim, rank=args.rank_latent, seed=3, device=dev)
    else:
        x = ivf.sift_like_device(args.n, args.dim, args.rank_latent, seed=1, device=dev, dpad=dpad)
    info = ivf.build_graph_ivf(ctx, x, degree=args.degree, cluster_size=args.cluster_size, probe=args.probe,
                               dim=args.dim, optimize=True, keep=args.keep,
                               tensor_cores=args.metric == "l2", log=log)  # byte data: tcgen05 K7 is exact
    del x
    info.pop("perm")
    torch.cuda.empty_cache()
    pv, pa, _, _, n = ctx.partition_view_device(0)
    vec = ivf.device_view(pv, (n, dpad), torch.float32, dev)
    # the routing table of a 1-partition index (C = 1): fp64 mean -> f32
    acc = torch.zeros(dpad, dtype=torch.float64, device=dev)
    for b in range(0, n, 1 << 24):
        acc += vec[b:b + (1 << 24)].double().sum(0)
    cent = (acc / n).float()[:args.dim].cpu().numpy()[None, :]
    ctx.set_centroids(cent, np.zeros(1, np.uint32), 1)
    s = min(args.recall_sample, args.nq) if gt_rows is None else gt_rows
    if args.metric == "ip":
        q = ivf.embedding_like_device(args.nq, args.dim, rank=args.rank_latent, seed=4 + rank, basis_seed=3,
                                      device=dev)
        gt = ivf.topk_ip_device(vec, q[:s].contiguous(), args.k)
    else:
        q = ivf.sift_like_queries_device(args.nq, args.dim, args.rank_latent, data_seed=1, seed=2 + rank,
                                         device=dev)
        vb = ivf.to_bf16(ctx, vec)  # ground truth on the tensor cores (exact on byte data)
        gt, _ = ivf.brute_force_topk(ctx, vec, ivf.row_norms(ctx, vec), q[:s].contiguous(), args.k, db_bf16=vb)
        del vb
    w = Workload()
    w.queries = q
    w.gt = gt.cpu().numpy()
    w.centroid = cent
    w.vec = vec
    w.adj = ivf.device_view(pa, (n, args.degree), torch.int32, dev)
    w.info = {k: v for k, v in info.items()}
    w.info["setup_s"] = time.time() - t0
    log(f"[bench] {args.workload} workload ready in {w.info['setup_s']:.1f}s")
    return w


def build_cfg1(args, rank, ctx, dev, gt_rows=None):
    """The round-1 workload: numpy SIFT-like data, exact K6 graph (cached)."""
    import torch
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
        for path, arr in ((adj_path, adj), (eo_path, eo)):
            tmp = path + f".{os.getpid()}.npy"
            np.save(tmp, arr)
            os.replace(tmp, path)
    gids = np.arange(args.n, dtype=np.uint32)
    cents = data.mean(0, dtype=np.float64).astype(np.float32)[None, :]
    index = BuiltIndex(cents, np.zeros(1, np.uint32), 1, args.degree, [GraphIndex(data, gids, args.degree, adj, eo)])
    ctx.load_index(index)
    s = min(args.recall_sample, args.nq) if gt_rows is None else gt_rows
    w = Workload()
    w.queries = torch.from_numpy(queries).to(dev)
    w.gt = synth.brute_force_gt(data, queries[:s], args.k, ctx=ctx)
    w.centroid = cents
    w.host = (data, adj)
    w.info = {"graph": "exact kNN (K6)", "setup_s": time.time() - t0}
    log(f"[bench] cfg1 workload ready in {w.info['setup_s']:.1f}s")
    return w


def build_workload(args, rank, ctx, dev, gt_rows=None):
    return (build_cfg1 if args.workload == "cfg1" else build_cfg3)(args, rank, ctx, dev, gt_rows)


def host_index(w):
    """(vectors n x dim, adjacency n x d) numpy copies of the resident index."""
    if hasattr(w, "host"):
        return w.host
    vec = w.vec[:, :w.centroid.shape[1]].cpu().numpy() if w.vec.shape[1] != w.centroid.shape[1] \
        else w.vec.cpu().numpy()
    adj = w.adj.cpu().numpy().view(np.uint32)
    return vec, adj


def workload_config(args, world, rec, w=None, sharded=False):
    cfg = {
        "workload": WORKLOADS[args.workload]["desc"],
        "n": args.n, "dim": args.dim, "degree": args.degree, "queries_per_step_per_gpu": args.nq,
        "iterations": args.iterations, "beam_width": args.beam, "k": args.k,
        "entry_count": args.entry, "partitions": 1, "accum": args.accum,
        "recall_at_10": None if rec is None else round(rec, 4),
        "recall_sample": args.recall_sample,
        "l2": ("index and gathers far larger than L2 (38.4 GB vectors, random rows); 256 MiB buffer "
               "written before every timed step") if args.workload == "cfg3" else
              "256 MiB buffer written before every timed step",
        "parallelism": (f"node-sharded x{world}: vectors split by id range, adjacency replicated, "
                        f"{args.exchange} NVLink peer-store frontier exchange" if sharded
                        else (f"replicas x{world}" if world > 1 else "single GPU")),
        "step": ("node-sharded search (ids + dists)" if sharded
                 else "run_pipeline: assign + route + K1 + combine + hit vectors"),
    }
    if w is not None:
        g = {k: v for k, v in w.info.items() if k not in ("perm",)}
        if w.graph_sha256:
            g["adjacency_sha256"] = w.graph_sha256
        cfg["graph"] = g
    return cfg


# ---------------------------------------------------------------------------
def reference_setup(args):
    """--impl reference-setup (a separate process): build the workload on the
    GPU exactly as the dvsg arm does and write the arrays the reference arm
    needs to args.ref_out; the reference process itself maps no libdvsg."""
    import torch
    import paper_2512_02278_b200 as dvs
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    ctx = dvs.Context(0)
    nq_ref = min(args.nq, 100_000)
    w = build_workload(args, 0, ctx, dev)
    vec, adj = host_index(w)
    out = args.ref_out
    np.save(os.path.join(out, "vectors.npy"), vec)
    np.save(os.path.join(out, "adjacency.npy"), adj)
    np.save(os.path.join(out, "centroid.npy"), w.centroid)
    np.save(os.path.join(out, "queries.npy"), w.queries[:nq_ref, :args.dim].cpu().numpy())
    np.save(os.path.join(out, "gt.npy"), w.gt)
    meta = {"adjacency_sha256": sha256_bytes(adj), "graph": {k: v for k, v in w.info.items()}}
    with open(os.path.join(out, "meta.json"), "w") as f:
        json.dump(meta, f)
    ctx.close()


def ref_index(vec, adj, centroid, degree, metric="l2"):
    """The reference's own BuiltIndex over these arrays (oracle/_ref: the
    unmodified reference sources; compute_entry_order is the reference's).
    Inner product has no reference implementation (SPEC.md: L2 only): the
    oracle's restatement (dist = -dot, same tie rules) stands in ("port")."""
    from oracle.oracle import Oracle, Ref, have_ref
    n = vec.shape[0]
    gids = np.arange(n, dtype=np.uint32)
    if metric == "ip":
        o = Oracle()
        return "port", (o, (vec, gids, adj, o.compute_entry_order(vec)))
    if have_ref():
        return "reference", Ref().index_from_arrays(centroid, np.zeros(1, np.uint32), 1, degree,
                                                    [(vec, adj, gids)])
    from paper_2512_02278_b200.api import BuiltIndex, GraphIndex
    return "port", (Oracle(), BuiltIndex(centroid, np.zeros(1, np.uint32), 1, degree,
                                         [GraphIndex(vec, gids, degree, adj, None)]))


def ref_runner(kind, idx, args, nthreads):
    if kind == "reference":
        def run(qs):
            return idx.run_pipeline(qs, args.iterations, args.beam, args.k, args.entry, 1, 1,
                                    nthreads=nthreads, with_vectors=True)
    elif args.metric == "ip":
        o, (vec, gids, adj, eo) = idx

        def run(qs):  # C = 1: run_pipeline is one beam search per query (simulator.cpp:317-324)
            ids, dists, counts, vis = o.beam_search(vec, gids, adj, eo, qs, args.iterations, args.beam, args.k,
                                                    args.entry, metric=1, nthreads=nthreads)
            return ids, dists, counts, None, int(vis.sum())
    else:
        o, bi = idx

        def run(qs):
            return o.run_pipeline(bi, qs, args.iterations, args.beam, args.k, args.entry, 1, 1,
                                  nthreads=nthreads, with_vectors=True)
    return run


def size_sample(run, queries, seconds, nthreads, min_q=64):
    probe = queries[:max(min_q, 2 * nthreads)]
    t0 = time.perf_counter()
    run(probe)
    per_q = (time.perf_counter() - t0) / probe.shape[0]
    return int(min(queries.shape[0], max(probe.shape[0], seconds / max(per_q, 1e-9))))


def run_reference_impl(args, world, rank):
    """--impl reference: rank 0 times the reference CPU implementation (the
    graph comes from a separate setup process through /dev/shm)."""
    if rank != 0:
        return
    t0 = time.time()
    base = "/dev/shm" if os.path.isdir("/dev/shm") else None
    out = tempfile.mkdtemp(prefix="dvsg_ref_", dir=base)
    try:
        cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference-setup", "--ref-out", out,
               "--workload", args.workload, "--n", str(args.n), "--nq", str(args.nq), "--dim", str(args.dim),
               "--rank-latent", str(args.rank_latent), "--degree", str(args.degree),
               "--probe", str(args.probe), "--cluster-size", str(args.cluster_size), "--keep", str(args.keep),
               "--k", str(args.k), "--recall-sample", str(args.recall_sample), "--cache", args.cache,
               "--iterations", str(args.iterations), "--beam", str(args.beam), "--entry", str(args.entry)]
        env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
        subprocess.run(cmd, check=True, env=env, stdout=sys.stderr)
        vec = np.load(os.path.join(out, "vectors.npy"), mmap_mode="r")
        adj = np.load(os.path.join(out, "adjacency.npy"), mmap_mode="r")
        centroid = np.load(os.path.join(out, "centroid.npy"))
        queries = np.load(os.path.join(out, "queries.npy"))
        gt = np.load(os.path.join(out, "gt.npy"))
        meta = json.load(open(os.path.join(out, "meta.json")))
        kind, idx = ref_index(np.ascontiguousarray(vec) if args.metric == "ip" else vec,
                              np.ascontiguousarray(adj) if args.metric == "ip" else adj, centroid, args.degree,
                              args.metric)
        del vec, adj
    finally:
        shutil.rmtree(out, ignore_errors=True)
    setup_s = time.time() - t0
    nthreads = os.cpu_count() or 1
    run = ref_runner(kind, idx, args, nthreads)
    n = size_sample(run, queries, args.ref_step_seconds, nthreads)
    n = max(n, min(gt.shape[0], queries.shape[0]))
    sample = queries[:n]
    for _ in range(min(args.warmup, 1)):
        run(sample[:min(n, 4 * nthreads)])  # page the index in
    times = []
    res = None
    for _ in range(args.steps):
        t1 = time.perf_counter()
        res = run(sample)
        times.append(time.perf_counter() - t1)
    total = sum(times)
    qps = n * args.steps / total
    s = min(gt.shape[0], n)
    rec = recall_at_k(res[0][:s, :10], np.minimum(res[2][:s], 10), gt[:s, :10], 10)
    cfg = workload_config(args, world, rec)
    if args.k != 10:
        cfg[f"recall_at_{args.k}"] = round(recall_at_k(res[0][:s], res[2][:s], gt[:s], args.k), 4)
    cfg["graph"] = dict(meta["graph"], adjacency_sha256=meta["adjacency_sha256"])
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": nthreads, "kind": kind,
                         "sample": f"{n} of the {args.nq} queries per step, run_pipeline C=1 "
                                   f"(simulator.cpp:245-366) in {nthreads} threads",
                         "cpu_model": cpu_model(), "setup_s": setup_s},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
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


class Bufs:
    def __init__(self, torch, nq, k, dim, dev, vectors=True):
        self.ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
        self.dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
        self.counts = torch.empty((nq,), dtype=torch.int32, device=dev)
        self.vis = torch.empty((nq,), dtype=torch.int64, device=dev)
        self.vecs = torch.empty((nq, k, dim), dtype=torch.float32, device=dev) if vectors else None


def timed_steps(args, torch, ctx, stream, step, flush, dist, local, pre_step=lambda: None, stats=True):
    """W warm-up steps, then K timed steps (CUDA events on the library stream,
    L2 flushed before each).  -> (total ms, K1 ms, visited, expanded, units,
    launches, clocks summary)"""
    for _ in range(args.warmup):
        pre_step()
        step()
        ctx.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k1_ms, vis, exp, units = 0.0, 0, 0, 0
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
            if stats:
                st = ctx.last_search_stats()      # syncs the stream
                k1_ms += ctx.last_timings()["search_ms"]
                vis += st["visited"]
                exp += st["expanded"]
                units += st["units"]
            else:
                stream.synchronize()
        torch.cuda.synchronize()
    launches = ctx.kernel_launches() - launches0
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([ms, k1_ms], dtype=torch.float64, device=flush.device)
    if dist:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0]), float(t[1]), vis, exp, units, launches, clk.summary()


def e2e_pinned(args, torch, dvs, ctx, w, p, ids_h, cnt_h, flush, dist, world, rank):
    nq, dim, k = args.nq, args.dim, args.k
    keep = []

    def pin(shape, dt):
        t = torch.empty(shape, dtype=dt, pin_memory=True)
        keep.append(t)
        return t.numpy()

    hq = pin((nq, dim), torch.float32)
    hq[:] = w.queries[:, :dim].cpu().numpy()
    wv = args.workload != "cfg4"  # hit vectors (off at cfg4: 30.7 GB per step)
    out = {"ids": pin((nq, k), torch.int32).view(np.uint32), "dists": pin((nq, k), torch.float32),
           "counts": pin((nq,), torch.int32).view(np.uint32)}
    if wv:
        out["vectors"] = pin((nq, k, dim), torch.float32)
    ctx.run_pipeline(hq, p, 1, 1, 0, wv, out)  # warm
    stream = torch.cuda.ExternalStream(ctx.stream, device=flush.device)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        ev0[i].record(stream)
        ctx.run_pipeline(hq, p, 1, 1, 0, wv, out)
        ev1[i].record(stream)
    torch.cuda.synchronize()
    e_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))], dtype=torch.float64,
                        device=flush.device)
    if dist:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    assert np.array_equal(out["ids"], ids_h) and np.array_equal(out["counts"], cnt_h), \
        "host-buffer and device-pointer paths disagree"
    h2d = hq.nbytes
    d2h = sum(v.nbytes for v in out.values()) + 4 + 8
    e2e = {"value": nq * world * args.steps / (float(e_ms[0]) / 1e3), "unit": "queries/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": float(e_ms[0]) / args.steps, "host_buffers": "pinned",
           "timeline": timeline_summary(dvs, ctx.last_pipeline_timeline(rank), args)}
    # the drop-in caller of INTEGRATION.md passes ordinary (pageable) memory
    qp = np.array(hq)
    outp = {kk: np.zeros_like(v) for kk, v in out.items()}
    ctx.run_pipeline(qp, p, 1, 1, 0, wv, outp)
    reps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(reps):
        ctx.run_pipeline(qp, p, 1, 1, 0, wv, outp)
    dt = (time.perf_counter() - t0) / reps
    e2e["pageable"] = {"value": nq / dt, "unit": "queries/s", "ms_per_step": 1e3 * dt, "steps": reps,
                       "timing": "host wall clock around dvsg_run_pipeline (synchronous call)",
                       "ids_identical": bool(np.array_equal(outp["ids"], ids_h))}
    return e2e


def accum_modes(args, torch, dvs, ctx, w, ids_h, cnt_h, dev):
    """QPS of the same search in the f64 parity mode and the compensated f32
    mode, and whether their ids equal the headline's (verdict r1 #5)."""
    nq = args.nq
    b = Bufs(torch, nq, args.k, args.dim, dev, vectors=False)
    uq = torch.arange(nq, dtype=torch.int32, device=dev)
    up = torch.zeros(nq, dtype=torch.int32, device=dev)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    out = {}
    for mode in ("f64", "f32c"):
        p = dvs.SearchParams(args.iterations, args.beam, args.k, args.entry, metric=args.metric, accum=mode)
        torch.cuda.synchronize()

        def run():
            ctx.search_units_device(w.queries.data_ptr(), nq, args.dim, uq.data_ptr(), up.data_ptr(), nq, p,
                                    b.ids.data_ptr(), b.dists.data_ptr(), b.counts.data_ptr(), b.vis.data_ptr())
        run()
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        ctx.synchronize()
        ms = e0.elapsed_time(e1)
        same = bool(np.array_equal(b.ids.cpu().numpy().view(np.uint32), ids_h) and
                    np.array_equal(b.counts.cpu().numpy().view(np.uint32), cnt_h))
        out[mode] = {"value": nq / (ms / 1e3), "unit": "queries/s", "ms_per_search": ms,
                     "ids_identical_to_headline": same, "step": "K1 search only"}
    return out


def u8_storage(args, torch, ctx, stream, step, flush, dist, local, b, ids_h, cnt_h, f32_total_ms):
    """Side measurement (not the headline): the same run_pipeline step with K1
    gathering a byte copy of the rows (dvsg_set_vector_storage U8; the byte-
    valued synthetic data converts exactly), same W/K, L2 flush and events.
    The reference stores fp32, so the headline stays on fp32 rows."""
    import paper_2512_02278_b200 as dvs
    try:
        ctx.set_vector_storage("u8")
    except dvs.InvalidArgument as ex:
        return {"value": None, "note": f"not byte-valued data: {ex}"}
    try:
        total_ms, k1_ms, vis, exp, units, launches, clocks = timed_steps(args, torch, ctx, stream, step, flush,
                                                                         dist, local, stats=False)
        same = bool(np.array_equal(b.ids.cpu().numpy().view(np.uint32), ids_h) and
                    np.array_equal(b.counts.cpu().numpy().view(np.uint32), cnt_h))
    finally:
        ctx.set_vector_storage("f32")
    return {"value": args.nq * args.steps / (total_ms / 1e3), "unit": "queries/s",
            "ms_per_step": total_ms / args.steps, "speedup_vs_f32_rows": f32_total_ms / total_ms,
            "ids_identical_to_headline": same, "bytes_per_row": args.dim,
            "note": "K1 reads a uint8 copy of the rows (a quarter of the gather bytes); every coordinate of the "
                    "synthetic data is an integer in [0, 255], so distances are bit-identical; side measurement, "
                    "the headline reads fp32 rows like the reference"}


def cpu_baseline(args, w, ids_h, cnt_h, dists_h):
    nthreads = os.cpu_count() or 1
    t0 = time.time()
    vec, adj = host_index(w)
    kind, idx = ref_index(vec, adj, w.centroid, args.degree, args.metric)
    if w.graph_sha256 is None:
        w.graph_sha256 = sha256_bytes(adj)
    del vec, adj
    setup_s = time.time() - t0
    run = ref_runner(kind, idx, args, nthreads)
    qh = w.queries[:, :args.dim].cpu().numpy()
    n = size_sample(run, qh, args.cpu_seconds, nthreads)
    t1 = time.perf_counter()
    r = run(qh[:n])
    dt = time.perf_counter() - t1
    same_ids = np.array_equal(r[0], ids_h[:n]) and np.array_equal(r[2], cnt_h[:n])
    same_q = int(sum(np.array_equal(r[0][i, :r[2][i]], ids_h[i, :cnt_h[i]]) for i in range(n)))
    rel = np.abs(r[1] - dists_h[:n]) / np.maximum(np.abs(r[1]), 1e-30)
    return {"value": n / dt, "unit": "queries/s", "cores": nthreads, "kind": kind,
            "sample": f"first {n} of the {args.nq} step queries, run_pipeline C=1, {nthreads} threads",
            "cpu_model": cpu_model(), "ids_identical_to_gpu": bool(same_ids),
            "queries_identical": same_q, "max_rel_dist_diff": float(rel.max()) if n else None,
            "setup_s": setup_s}


# ---------------------------------------------------------------------------
def sharded_measure(args, torch, dvs, dist, ctx, w, rank, world, local, flush, ids_ref, cnt_ref, dev):
    """K timed steps of the node-sharded search (this rank keeps 1/N of the
    vectors; NVLink frontier exchange); ids must equal the replica run's."""
    from paper_2512_02278_b200.dist import connect_nccl, prepare_step, setup_sharded_resident
    ctx.set_shard_exchange(args.exchange)
    setup_sharded_resident(ctx, rank, world)
    if args.exchange == "nccl":
        connect_nccl(ctx, rank)
    nq, dim = args.nq, args.dim
    p = dvs.SearchParams(args.iterations, args.beam, args.k, args.entry, metric=args.metric, accum=args.accum)
    b = Bufs(torch, nq, args.k, dim, dev, vectors=False)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    def step():
        ctx.search_sharded_device(w.queries.data_ptr(), nq, dim, p, b.ids.data_ptr(), b.dists.data_ptr(),
                                  b.counts.data_ptr(), b.vis.data_ptr())

    ms, _, _, _, _, launches, clk = timed_steps(args, torch, ctx, stream, step, flush, dist, local,
                                                pre_step=lambda: prepare_step(ctx, dist.barrier), stats=False)
    st = ctx.last_search_stats() if args.exchange != "fused" else None
    same = torch.tensor([int(np.array_equal(b.ids.cpu().numpy().view(np.uint32), ids_ref) and
                             np.array_equal(b.counts.cpu().numpy().view(np.uint32), cnt_ref))],
                        dtype=torch.int32, device=dev)
    dist.all_reduce(same, op=dist.ReduceOp.MIN)
    tl_sum = None
    if args.exchange != "fused":
        ctx.set_timing(True)
        prepare_step(ctx, dist.barrier)
        step()
        ctx.synchronize()
        tl = ctx.last_sharded_timeline(rank)
        ctx.set_timing(False)
        if tl:
            span = max(iv["end"] for iv in tl) - min(iv["start"] for iv in tl)
            comp = sum(iv["end"] - iv["start"] for iv in tl if iv["lane"] == "compute")
            comm = sum(iv["end"] - iv["start"] for iv in tl if iv["lane"] == "comm")
            tl_sum = {"rank": rank, "intervals": len(tl), "span_ms": span, "step_kernels_ms": comp,
                      "barrier_or_exchange_ms": comm, "exchange_share": comm / span if span else None}
    # e2e through the public call: pinned host queries in, ids / dists / counts out
    hq = torch.from_numpy(w.queries[:, :dim].cpu().numpy()).pin_memory()
    h_ids = torch.empty((nq, args.k), dtype=torch.int32, pin_memory=True)
    h_dists = torch.empty((nq, args.k), dtype=torch.float32, pin_memory=True)
    h_counts = torch.empty((nq,), dtype=torch.int32, pin_memory=True)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    dq = torch.empty_like(w.queries)
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        prepare_step(ctx, dist.barrier)
        with torch.cuda.stream(stream):
            ev0[i].record(stream)
            dq.copy_(hq, non_blocking=True)
            ctx.search_sharded_device(dq.data_ptr(), nq, dim, p, b.ids.data_ptr(), b.dists.data_ptr(),
                                      b.counts.data_ptr(), b.vis.data_ptr())
            h_ids.copy_(b.ids, non_blocking=True)
            h_dists.copy_(b.dists, non_blocking=True)
            h_counts.copy_(b.counts, non_blocking=True)
            ev1[i].record(stream)
        stream.synchronize()
    e_ms = torch.tensor([sum(a.elapsed_time(c) for a, c in zip(ev0, ev1))], dtype=torch.float64, device=dev)
    dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e = {"value": nq * world * args.steps / (float(e_ms[0]) / 1e3), "unit": "queries/s",
           "h2d_bytes_per_step": int(hq.numel() * 4),
           "d2h_bytes_per_step": int((h_ids.numel() + h_dists.numel() + h_counts.numel()) * 4),
           "ms_per_step": float(e_ms[0]) / args.steps, "host_buffers": "pinned",
           "ids_identical": bool(np.array_equal(h_ids.numpy().view(np.uint32), ids_ref)),
           "note": "sharded mode returns ids + dists (hit vectors stay on their owner GPUs)"}
    xch = None
    if st and st["units"]:
        vis_q = st["visited"] / st["units"]
        dpad = (dim + 3) // 4 * 4
        xbytes = nq * (vis_q * (world - 1) / world * 16 + (world - 1) * 4 * dim)
        alg = nq * (vis_q * 4 * dpad + st["expanded"] / st["units"] * 4 * args.degree + 4 * dpad)
        step_s = ms / args.steps / 1e3
        xch = {"bytes_per_step_per_gpu": xbytes, "achieved_gbs": xbytes / step_s / 1e9,
               "nvlink_peak_gbs_per_direction": 900.0, "frac": xbytes / step_s / 1e9 / 900.0,
               "hbm_alg_gbs_per_gpu": alg / step_s / 1e9, "visited_per_query": vis_q}
    return {"value": nq * world * args.steps / (ms / 1e3), "unit": "queries/s",
            "ms_per_step": ms / args.steps, "exchange_roofline": xch, "timeline_rank0": tl_sum,
            "gpu_launches": int(launches), "clocks": clk,
            "layout": f"vectors node-sharded {world} ways (id ranges), adjacency replicated; " + (
                "bulk-synchronous NVLink peer-store frontier exchange (xchg_kernel.cu)" if args.exchange == "bulk"
                else "bulk protocol, host-driven ncclSend/ncclRecv exchange (baseline)" if args.exchange == "nccl"
                else "fused NVLink peer-store frontier exchange (shard_kernel.cu)"),
            "exchange": args.exchange, "ids_identical_to_replica_all_ranks": bool(same[0]), "e2e": e2e}


def self_launch(args):
    """`--gpus N` without torchrun: relaunch this command under torchrun."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if args.impl == "reference-setup":
        return reference_setup(args)
    if env_world is None and args.gpus > 1 and args.impl == "dvsg":
        sys.exit(self_launch(args))
    world = int(env_world or "1")
    if args.impl == "dvsg" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        # rank 0 times the CPU reference; the line carries the N of the run
        # (torchrun's WORLD_SIZE, or --gpus when launched without torchrun)
        return run_reference_impl(args, max(world, args.gpus), rank)

    import torch
    import paper_2512_02278_b200 as dvs

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        # rank 0 must print exactly one JSON line on stdout: keep NCCL's banner off stdout
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() in ("VERSION", ""):
            os.environ["NCCL_DEBUG"] = "WARN"
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    sharded = world > 1 and args.mode in ("auto", "sharded")

    ctx = dvs.Context(local)
    w = build_workload(args, rank, ctx, dev)
    p = dvs.SearchParams(args.iterations, args.beam, args.k, args.entry, metric=args.metric, accum=args.accum)
    nq, dim, k = args.nq, args.dim, args.k
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    with_vectors = args.workload != "cfg4"  # 100k x 100 x 768 hit vectors would be 30.7 GB per step
    b = Bufs(torch, nq, k, dim, dev, vectors=with_vectors)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    torch.cuda.synchronize()

    def step():
        ctx.run_pipeline_device(w.queries.data_ptr(), nq, dim, p, 1, b.ids.data_ptr(), b.dists.data_ptr(),
                                b.counts.data_ptr(), b.vecs.data_ptr() if with_vectors else 0)

    # ---- the replica / single-GPU run_pipeline (headline at N = 1) ----------------
    ctx.set_timing(True)
    total_ms, k1_ms, vis_tot, exp_tot, units_tot, launches, clocks = timed_steps(
        args, torch, ctx, stream, step, flush, dist, local)
    ctx.set_timing(False)
    ids_h = b.ids.cpu().numpy().view(np.uint32)
    cnt_h = b.counts.cpu().numpy().view(np.uint32)
    dists_h = b.dists.cpu().numpy()
    s = w.gt.shape[0]
    rec = recall_at_k(ids_h[:s, :10], np.minimum(cnt_h[:s], 10), w.gt[:, :10], 10)  # the metric's recall@10
    rec_k = recall_at_k(ids_h[:s], cnt_h[:s], w.gt, k)
    replica = {"value": nq * world * args.steps / (total_ms / 1e3), "unit": "queries/s",
               "ms_per_step": total_ms / args.steps, "recall_at_10": round(rec, 4)}

    ctx.set_timing(True)  # per-microbatch events of the e2e pipeline (measured timeline)
    e2e = None if args.no_e2e or sharded else e2e_pinned(args, torch, dvs, ctx, w, p, ids_h, cnt_h, flush,
                                                         dist, world, rank)
    ctx.set_timing(False)
    modes = None if args.no_modes or sharded else accum_modes(args, torch, dvs, ctx, w, ids_h, cnt_h, dev)
    storage_u8 = None
    if not args.no_modes and not sharded and args.dim <= 256:
        storage_u8 = u8_storage(args, torch, ctx, stream, step, flush, dist, local, b, ids_h, cnt_h, total_ms)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args, w, ids_h, cnt_h, dists_h)
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "queries/s", "cores": 0, "kind": "unavailable",
                   "sample": f"failed: {type(ex).__name__}: {ex}"}
    elif rank == 0 and args.workload != "cfg1" and w.graph_sha256 is None:
        w.graph_sha256 = sha256_bytes(w.adj.cpu().numpy())

    # ---- N > 1: the node-sharded north-star layout is the headline ------------------
    shard = None
    if sharded:
        try:
            shard = sharded_measure(args, torch, dvs, dist, ctx, w, rank, world, local, flush, ids_h, cnt_h, dev)
        except Exception as ex:  # noqa: BLE001
            shard = {"error": f"{type(ex).__name__}: {ex}"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_kind = peaks()
    dpad = (dim + 3) // 4 * 4
    alg_bytes = vis_tot * 4 * dpad + exp_tot * 4 * args.degree + units_tot * 4 * dpad
    achieved = alg_bytes / args.steps / (k1_ms / args.steps / 1e3) / 1e9
    traffic, tsrc = None, None
    tpath = os.path.join(ROOT, "profiles", "k1_traffic.json")
    key = f"{args.workload}_n{args.n}_q{nq}_w{args.beam}_I{args.iterations}_{args.accum}"
    if os.path.isfile(tpath):
        try:
            tj = json.load(open(tpath))
            ent = tj.get(key) if isinstance(tj, dict) else None
            if ent:
                traffic, tsrc = ent.get("dram_bytes_per_launch"), ent.get("source")
        except Exception:
            traffic = None
    headline = shard if (sharded and shard and "error" not in shard) else None
    value = headline["value"] if headline else nq * world * args.steps / (total_ms / 1e3)
    ms_step = headline["ms_per_step"] if headline else total_ms / args.steps
    eff_accum = args.accum if args.accum != "f32" or ctx.index_integral() else "f64/f32c (upgraded)"
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": eff_accum, "data": "synthetic",
        "config": dict(workload_config(args, world, rec, w, sharded=bool(headline)),
                       **({f"recall_at_{k}": round(rec_k, 4)} if k != 10 else {})),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": tsrc,
                     "peak_kind": peak_kind, "kernel": "dvsg::search_kernel (K1)",
                     "k1_ms_per_step": k1_ms / args.steps, "alg_bytes_per_step": alg_bytes / args.steps,
                     "visited_per_query": vis_tot / max(units_tot, 1),
                     "expanded_per_query": exp_tot / max(units_tot, 1),
                     "k1_share_of_step": k1_ms / total_ms if total_ms else None},
        "cpu_baseline": cpu, "e2e": headline["e2e"] if headline else e2e, "gpu_launches": int(headline["gpu_launches"] if headline else launches),
        "accum_modes": modes,
        "storage_u8": storage_u8,
        "clocks": headline["clocks"] if headline else clocks,
    }
    if world > 1:
        line["replicas"] = replica
        line["sharded_mode"] = shard
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
