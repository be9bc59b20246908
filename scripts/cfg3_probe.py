#!/usr/bin/env python
"""Build a SIFT-/Deep-like n x d index on the GPU (ivf.build_graph_ivf) and
sweep (iterations, beam) for recall@10 / QPS -- calibration of the cfg3
(100M x 96) bench workload.  One JSON line per setting on stdout."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_02278_b200 as dvs  # noqa: E402
from paper_2512_02278_b200 import ivf  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=96)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--nq", type=int, default=100_000)
    ap.add_argument("--gt", type=int, default=2000)
    ap.add_argument("--cluster-size", type=int, default=1024)
    ap.add_argument("--probe", type=int, default=8)
    ap.add_argument("--sweep", default="6x64,8x64,10x64,8x96,10x96,12x96,10x128,12x128")
    ap.add_argument("--accum", default="f32")
    ap.add_argument("--keep", type=int, default=16)
    ap.add_argument("--no-optimize", action="store_true")
    ap.add_argument("--tc", action="store_true", help="K7 on the tensor cores")
    args = ap.parse_args()
    dev = "cuda:0"
    ctx = dvs.Context(0)
    t0 = time.time()
    x = ivf.sift_like_device(args.n, args.dim, args.rank, seed=1, device=dev)
    torch.cuda.synchronize()
    log(f"[probe] data {args.n}x{args.dim} in {time.time() - t0:.1f}s")
    info = ivf.build_graph_ivf(ctx, x, degree=32, cluster_size=args.cluster_size, probe=args.probe,
                               dim=args.dim, optimize=not args.no_optimize, keep=args.keep,
                               tensor_cores=args.tc, log=log)
    del x
    torch.cuda.empty_cache()
    pv, pa, pg, pe, n = ctx.partition_view_device(0)
    dpad = (args.dim + 3) // 4 * 4
    vec = ivf.device_view(pv, (n, dpad), torch.float32, dev)
    q = ivf.sift_like_queries_device(args.nq, args.dim, args.rank, data_seed=1, seed=2, device=dev)
    t1 = time.time()
    vn = ivf.row_norms(ctx, vec)
    gt_ids, _ = ivf.brute_force_topk(ctx, vec, vn, q[:args.gt].contiguous(), 10)
    gt = gt_ids.cpu().numpy()
    log(f"[probe] ground truth for {args.gt} queries in {time.time() - t1:.1f}s")
    mem = torch.cuda.mem_get_info()
    log(f"[probe] free {mem[0] / 1e9:.1f} GB of {mem[1] / 1e9:.1f}")
    nq, k = args.nq, 10
    d_ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    d_dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    d_counts = torch.empty((nq,), dtype=torch.int32, device=dev)
    d_vis = torch.empty((nq,), dtype=torch.int64, device=dev)
    uq = torch.arange(nq, dtype=torch.int32, device=dev)
    up = torch.zeros(nq, dtype=torch.int32, device=dev)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    for s in args.sweep.split(","):
        parts = [int(v) for v in s.split("x")]
        it, w = parts[0], parts[1]
        ent = parts[2] if len(parts) > 2 else w
        p = dvs.SearchParams(it, w, k, ent, accum=args.accum)
        torch.cuda.synchronize()

        def run():
            ctx.search_units_device(q.data_ptr(), nq, args.dim, uq.data_ptr(), up.data_ptr(), nq, p,
                                    d_ids.data_ptr(), d_dists.data_ptr(), d_counts.data_ptr(),
                                    d_vis.data_ptr())
        run()
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        ctx.synchronize()
        ms = e0.elapsed_time(e1)
        ids = d_ids[:args.gt].cpu().numpy().view(np.uint32).astype(np.int64)
        cnt = d_counts[:args.gt].cpu().numpy()
        rec = np.mean([len(set(ids[i, :cnt[i]].tolist()) & set(gt[i].tolist())) / 10 for i in range(args.gt)])
        vis = float(d_vis.double().mean())
        alg = (vis * 4 * dpad + it * w * 128 + 4 * dpad) * nq
        line = {"n": args.n, "dim": args.dim, "iters": it, "beam": w, "entry": ent, "recall@10": round(float(rec), 4),
                "qps": nq / (ms / 1e3), "ms": ms, "visited": vis, "alg_gbs": alg / (ms / 1e3) / 1e9,
                "accum": args.accum, "keep": args.keep, "build": {k2: v for k2, v in info.items() if k2 != "perm"}}
        print(json.dumps(line), flush=True)
        log(f"[probe] I={it} w={w} E={ent}: recall {rec:.4f}, {nq / (ms / 1e3):,.0f} QPS, visited {vis:.0f}")
    ctx.close()


if __name__ == "__main__":
    main()
